// Microbenchmark: tcgen05.mma kind::f16 issue-to-completion rate for the
// operand layouts the scan uses (no swizzle vs 128B swizzle, N = 64/128/256).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2605_17415_b200/csrc scripts/mma_bench.cu -o /tmp/mma_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace ivftq;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr, uint32_t sbo) {
  // K-major, SWIZZLE_128B (layout type 2 at bits 61-63), LBO ignored (1)
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

template <int N, bool SW>
__global__ void bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < (128 + N) * 128; i += blockDim.x) ((uint16_t*)smem)[i] = 0x3c00;
  if (tid < 32) sm100::tmem_alloc(&tslot, 256);
  if (tid == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::mbar_fence_init();
  }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t a = sm100::smem_u32(smem), b = a + 128 * 128 * 2;
  const uint32_t idesc = sm100::idesc_f16_f32(128, N);
  if (tid == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int s = 0; s < 8; ++s) {  // K = 128 in 8 steps
        uint64_t ad, bd;
        if (SW) {
          ad = desc_sw128(a + (s >> 2) * 128 * 128 + (s & 3) * 32, 1024);
          bd = desc_sw128(b + (s >> 2) * N * 128 + (s & 3) * 32, 1024);
        } else {
          ad = sm100::smem_desc(a + s * 2 * 128 * 16, 128 * 16, 128);
          bd = sm100::smem_desc(b + s * 2 * N * 16, N * 16, 128);
        }
        sm100::mma_f16(tmem, ad, bd, idesc, (it | s) ? 1u : 0u);
      }
    }
    sm100::mma_commit(&bar);
    sm100::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (tid < 32) sm100::tmem_dealloc(tmem, 256);
}

// A operand from TMEM (.ts form): columns [256, 256 + 64) hold A (K = 128 as
// 8 K-steps x 8 columns), accumulator at column 0 (N <= 256).
template <int N>
__global__ void bench_ts(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < N * 128; i += blockDim.x) ((uint16_t*)smem)[i] = 0x3c00;
  if (tid < 32) sm100::tmem_alloc(&tslot, 512);
  if (tid == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::mbar_fence_init();
  }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t b = sm100::smem_u32(smem);
  const uint32_t idesc = sm100::idesc_f16_f32(128, N);
  if (tid == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int s = 0; s < 8; ++s) {
        uint64_t bd = sm100::smem_desc(b + s * 2 * N * 16, N * 16, 128);
        sm100::mma_f16_ts(tmem, tmem + 256 + s * 8, bd, idesc, (it | s) ? 1u : 0u);
      }
    }
    sm100::mma_commit(&bar);
    sm100::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (tid < 32) sm100::tmem_dealloc(tmem, 512);
}

// Same MMA stream while other warps load the machine: mode 1 = 8 warps
// streaming 16-byte shared-memory stores + loads, mode 2 = 4 warps reading
// TMEM (tcgen05.ld 32 columns) in a loop, mode 3 = both.
template <int N>
__global__ void bench_ts_busy(int iters, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < N * 128; i += blockDim.x) ((uint16_t*)smem)[i] = 0x3c00;
  if (tid < 32) sm100::tmem_alloc(&tslot, 512);
  if (tid == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::mbar_fence_init();
    done = 0;
  }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t b = sm100::smem_u32(smem);
  const uint32_t idesc = sm100::idesc_f16_f32(128, N);
  unsigned char* scratch = smem + N * 128 * 2;
  if (warp == 0) {
    if (tid == 0) {
      long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        for (int s = 0; s < 8; ++s) {
          uint64_t bd = sm100::smem_desc(b + s * 2 * N * 16, N * 16, 128);
          sm100::mma_f16_ts(tmem, tmem + 256 + s * 8, bd, idesc, (it | s) ? 1u : 0u);
        }
      }
      sm100::mma_commit(&bar);
      sm100::mbar_wait(&bar, 0);
      long long t1 = clock64();
      out[blockIdx.x] = (unsigned long long)(t1 - t0);
      done = 1;
    }
  } else if (warp >= 1 && warp <= 8) {
    if (mode & 1) {
      uint4* p = (uint4*)scratch + (warp - 1) * 32 * 16 + (tid & 31);
      uint4 v = make_uint4(tid, 1, 2, 3);
      while (!done) {
        for (int i = 0; i < 16; ++i) {
          p[i * 32] = v;
          v.x += ((volatile uint4*)p)[((i + 5) & 15) * 32].y;
        }
      }
      if (v.x == 12345) out[148 + tid] = v.x;
    }
  } else if (warp >= 9 && warp <= 12) {
    if (mode & 2) {
      uint32_t acc = 0;
      const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 384;
      while (!done) {
        uint32_t r[32];
        sm100::tmem_ld32(ta, r);
        sm100::tmem_ld_wait();
        acc += r[0] + r[31];
      }
      if (acc == 12345) out[148 + tid] = acc;
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (tid < 32) sm100::tmem_dealloc(tmem, 512);
}

template <int N>
void run_ts_busy(int mode) {
  unsigned long long* d;
  cudaMalloc(&d, (148 + 1024) * 8);
  int iters = 2000;
  size_t smem = N * 128 * 2 + 8 * 32 * 16 * 16 + 1024;
  cudaFuncSetAttribute(bench_ts_busy<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bench_ts_busy<N><<<148, 13 * 32, smem>>>(iters, mode, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = (double)h[0] / (iters * 8);
  printf("ts busy mode %d N=%3d: %7.1f cycles/MMA  (%s)\n", mode, N, cyc, cudaGetErrorString(e));
  cudaFree(d);
}


// Dependent-accumulate latency: the same .ts MMA stream spread round-robin
// over CH independent accumulators (columns c*N), 18 MMAs per "tile".
template <int N, int CH>
__global__ void bench_ts_chains(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  for (int i = tid; i < N * 128; i += blockDim.x) ((uint16_t*)smem)[i] = 0x3c00;
  if (tid < 32) sm100::tmem_alloc(&tslot, 512);
  if (tid == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::mbar_fence_init();
  }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t b = sm100::smem_u32(smem);
  const uint32_t idesc = sm100::idesc_f16_f32(128, N);
  if (tid == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int s = 0; s < 6; ++s) {
        uint64_t bd = sm100::smem_desc(b + s * 2 * N * 16, N * 16, 128);
#pragma unroll
        for (int c = 0; c < CH; ++c)
          sm100::mma_f16_ts(tmem + c * N, tmem + 384 + s * 8 + (c % 2) * 48, bd, idesc, (it | s) ? 1u : 0u);
      }
    }
    sm100::mma_commit(&bar);
    sm100::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (tid < 32) sm100::tmem_dealloc(tmem, 512);
}
template <int N, int CH>
void run_chains() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  int iters = 2000;
  size_t smem = N * 128 * 2 + 1024;
  cudaFuncSetAttribute(bench_ts_chains<N, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bench_ts_chains<N, CH><<<148, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = (double)h[0] / (iters * 6 * CH);
  printf("ts chains=%d N=%3d: %7.1f cycles/MMA (floor %d)  (%s)\n", CH, N, cyc, N / 2, cudaGetErrorString(e));
  cudaFree(d);
}

// TMEM read rate: NW warps per lane quadrant loop over tcgen05.ld x32 (+wait)
// of the accumulator columns, alone (mma = 0) or under a continuous N=80 .ts
// MMA stream (mma = 1). Reports cycles per x32 load per warp and B/clk/SM.
template <int NW, int DEPTH>
__global__ void bench_ldtm(int iters, int mma, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5;
  constexpr int N = 80;
  for (int i = tid; i < N * 128; i += blockDim.x) ((uint16_t*)smem)[i] = 0x3c00;
  if (tid < 32) sm100::tmem_alloc(&tslot, 512);
  if (tid == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::mbar_fence_init();
    done = 0;
  }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t b = sm100::smem_u32(smem);
  const uint32_t idesc = sm100::idesc_f16_f32(128, N);
  if (warp == 0) {
    if (tid == 0 && mma) {
      int it = 0;
      while (!done) {
        for (int s = 0; s < 6; ++s) {
          uint64_t bd = sm100::smem_desc(b + s * 2 * N * 16, N * 16, 128);
          sm100::mma_f16_ts(tmem + (it & 1) * 128, tmem + 384 + s * 8, bd, idesc, s ? 1u : 0u);
        }
        ++it;
        if ((it & 15) == 0) {
          sm100::mma_commit(&bar);
          sm100::mbar_wait(&bar, ((it >> 4) - 1) & 1);
        }
      }
    }
  } else if (warp >= 4 && warp < 4 + 4 * NW) {
    uint32_t acc = 0;
    const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    __syncwarp();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint32_t r[DEPTH][32];
#pragma unroll
      for (int x = 0; x < DEPTH; ++x) sm100::tmem_ld32(ta + ((it + x) & 3) * 32, r[x]);
      sm100::tmem_ld_wait();
#pragma unroll
      for (int x = 0; x < DEPTH; ++x) acc += r[x][0] + r[x][31];
    }
    long long t1 = clock64();
    if ((tid & 31) == 0) out[blockIdx.x * 32 + warp] = (unsigned long long)(t1 - t0);
    if (acc == 12345) out[148 * 32 + tid] = acc;
    __syncwarp();
    if (warp == 4 && (tid & 31) == 0) { __nanosleep(2000); done = 1; }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (tid < 32) sm100::tmem_dealloc(tmem, 512);
}
template <int NW, int DEPTH>
void run_ldtm(int mma) {
  unsigned long long* d;
  cudaMalloc(&d, (148 * 32 + 1024) * 8);
  cudaMemset(d, 0, (148 * 32 + 1024) * 8);
  int iters = 2000;
  size_t smem = 80 * 128 * 2 + 1024;
  cudaFuncSetAttribute(bench_ldtm<NW, DEPTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bench_ldtm<NW, DEPTH><<<148, (4 + 4 * NW) * 32, smem>>>(iters, mma, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[32];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = (double)h[4] / (iters * DEPTH);
  printf("ldtm x32: %d warps/quadrant, %d in flight, mma=%d: %7.1f cycles per load per warp, %6.1f B/clk/SM (%s)\n",
         NW, DEPTH, mma, cyc, 4096.0 * 4 * NW / cyc, cudaGetErrorString(e));
  cudaFree(d);
}

template <int N>
void run_ts() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  int iters = 2000;
  size_t smem = N * 128 * 2 + 1024;
  cudaFuncSetAttribute(bench_ts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bench_ts<N><<<148, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = (double)h[0] / (iters * 8);
  printf("%-14s N=%3d: %7.1f cycles/MMA  %7.0f flop/cyc/SM  (%s)\n", "ts(A in TMEM)", N, cyc,
         2.0 * 128 * N * 16 / cyc, cudaGetErrorString(e));
  cudaFree(d);
}

template <int N, bool SW>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  int iters = 2000;
  size_t smem = (128 + N) * 128 * 2 + 1024;
  cudaFuncSetAttribute(bench<N, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bench<N, SW><<<148, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = (double)h[0] / (iters * 8);
  double flops = 2.0 * 128 * N * 16 / cyc;  // per SM per cycle
  printf("%-14s N=%3d: %7.1f cycles/MMA  %7.0f flop/cyc/SM  (%s)\n", name, N, cyc, flops,
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int m = 0; m < 2; ++m) { run_ldtm<1, 1>(m); run_ldtm<1, 2>(m); run_ldtm<2, 1>(m); run_ldtm<2, 2>(m); run_ldtm<4, 1>(m); }
  run<64, false>("noswizzle");
  run<128, false>("noswizzle");
  run<256, false>("noswizzle");
  run<64, true>("swizzle128");
  run<128, true>("swizzle128");
  run<256, true>("swizzle128");
  run_ts<64>();
  run_ts<128>();
  run_ts<256>();
  run_chains<32, 1>(); run_chains<32, 2>(); run_chains<32, 3>(); run_chains<48, 1>(); run_chains<80, 1>(); run_chains<80, 2>(); run_chains<80, 3>();
  run_chains<96, 1>(); run_chains<96, 2>(); run_chains<128, 1>(); run_chains<128, 2>(); run_chains<16,1>(); run_chains<16,4>(); run_chains<64,1>(); run_chains<64,2>();
  for (int m = 0; m < 4; ++m) run_ts_busy<64>(m);
  for (int m = 0; m < 4; ++m) run_ts_busy<128>(m);
  return 0;
}
