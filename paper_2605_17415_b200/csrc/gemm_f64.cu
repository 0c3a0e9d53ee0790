// FP64 CUDA-core GEMMs of the hot path (v1 numerics anchor).
//
//   coarse scores  S = qn . C^T   (index.py:436, f64 with f32 centroids upcast)
//   assignment     argmax_l <xn, c_l>, ties -> lowest l (partition.py:52-55)
//   rotation       Y = r . R^T    (rotation.py:40)
//
// All three are float64 in the reference, so they run as DFMA here: each
// output is a sequential k-order FMA chain, which differs from OpenBLAS only
// in rounding order (~1 ulp of f64), far below every decision margin measured
// in SURVEY.md §7 (min coarse gap 7e-8). Tile 64x64x16, 256 threads, each
// thread a 4x4 register tile at stride 16 (conflict-free shared reads).
#include "common.cuh"

namespace ivftq {

constexpr int TM = 64, TN = 64, TK = 16, PAD = 65;

template <typename TB>
__device__ __forceinline__ void gemm_tile(const double* __restrict__ A,
                                          const TB* __restrict__ B, int64_t M, int N,
                                          int K, int64_t m0, int n0, double (&As)[TK][PAD],
                                          double (&Bs)[TK][PAD], double (&acc)[4][4]) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k0 = 0; k0 < K; k0 += TK) {
#pragma unroll
    for (int it = 0; it < (TM * TK) / 256; ++it) {
      int i = threadIdx.x + it * 256;
      int r = i >> 4, kk = i & 15;
      int64_t gm = m0 + r;
      int gk = k0 + kk;
      As[kk][r] = (gm < M && gk < K) ? A[gm * K + gk] : 0.0;
      int gn = n0 + r;
      Bs[kk][r] = (gn < N && gk < K) ? (double)B[(int64_t)gn * K + gk] : 0.0;
    }
    __syncthreads();
    int kmax = min(TK, K - k0);
    for (int kk = 0; kk < kmax; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
}

template <typename TB, typename TC>
__global__ void __launch_bounds__(256)
gemm_nt_kernel(const double* __restrict__ A, const TB* __restrict__ B, int64_t M, int N,
               int K, TC* __restrict__ C) {
  __shared__ double As[TK][PAD];
  __shared__ double Bs[TK][PAD];
  double acc[4][4];
  int64_t m0 = (int64_t)blockIdx.x * TM;
  int n0 = blockIdx.y * TN;
  gemm_tile<TB>(A, B, M, N, K, m0, n0, As, Bs, acc);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gn = n0 + tx + 16 * j;
      if (gn < N) C[gm * N + gn] = (TC)acc[i][j];
    }
  }
}

// 128x128 tiles, 8x8 outputs per thread (rows ty+16i, cols tx+16j): half the
// shared-memory operand traffic per DFMA of the 64x64 kernel, which was
// shared-memory-bound at ~42 % of the FP64 pipe. The k loop keeps the same
// sequential FMA chain from 0.0 per output, so results are bit-identical.
// Next K-slab prefetched into registers while the current one computes.
constexpr int BM2 = 128, BN2 = 128, BK2 = 8, PAD2 = 132;

template <typename TB, typename TC>
__global__ void __launch_bounds__(256)
gemm_nt_big_kernel(const double* __restrict__ A, const TB* __restrict__ B, int64_t M, int N, int K,
                   TC* __restrict__ C) {
  __shared__ double As[2][BK2][PAD2];
  __shared__ double Bs[2][BK2][PAD2];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * BM2;
  const int n0 = blockIdx.y * BN2;
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  double ra[4], rb[4];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int i = threadIdx.x + it * 256;
      const int r = i >> 3, kk = i & 7;
      const int64_t gm = m0 + r;
      const int gn = n0 + r, gk = k0 + kk;
      ra[it] = (gm < M && gk < K) ? A[gm * K + gk] : 0.0;
      rb[it] = (gn < N && gk < K) ? (double)B[(int64_t)gn * K + gk] : 0.0;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int i = threadIdx.x + it * 256;
      As[buf][i & 7][i >> 3] = ra[it];
      Bs[buf][i & 7][i >> 3] = rb[it];
    }
  };
  fetch(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += BK2) {
    const bool more = k0 + BK2 < K;
    if (more) fetch(k0 + BK2);
    const int kmax = min(BK2, K - k0);
    for (int kk = 0; kk < kmax; ++kk) {
      double a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
    }
    if (more) {
      stash(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn < N) C[gm * N + gn] = (TC)acc[i][j];
    }
  }
}

// One block owns 64 rows and sweeps every centroid tile, keeping a running
// (max, argmax) per row; ties resolve to the lowest list id like np.argmax.
__global__ void __launch_bounds__(256)
assign_kernel(const double* __restrict__ A, const float* __restrict__ B, int64_t M, int N,
              int K, int32_t* __restrict__ out) {
  __shared__ double As[TK][PAD];
  __shared__ double Bs[TK][PAD];
  __shared__ double rv[TM][17];
  __shared__ int ri[TM][17];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  int64_t m0 = (int64_t)blockIdx.x * TM;
  double best[4];
  int bidx[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { best[i] = -INFINITY; bidx[i] = 0x7fffffff; }
  double acc[4][4];
  for (int n0 = 0; n0 < N; n0 += TN) {
    gemm_tile<float>(A, B, M, N, K, m0, n0, As, Bs, acc);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gn = n0 + tx + 16 * j;
      if (gn >= N) continue;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double v = acc[i][j];
        if (v > best[i] || (v == best[i] && gn < bidx[i]) || bidx[i] == 0x7fffffff) {
          best[i] = v;
          bidx[i] = gn;
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    rv[ty + 16 * i][tx] = best[i];
    ri[ty + 16 * i][tx] = bidx[i];
  }
  __syncthreads();
  if (threadIdx.x < TM) {
    int r = threadIdx.x;
    double bv = rv[r][0];
    int bi = ri[r][0];
    for (int t = 1; t < 16; ++t) {
      double v = rv[r][t];
      int ix = ri[r][t];
      if (ix == 0x7fffffff) continue;
      if (bi == 0x7fffffff || v > bv || (v == bv && ix < bi)) { bv = v; bi = ix; }
    }
    if (m0 + r < M) out[m0 + r] = bi;
  }
}

}  // namespace ivftq

using namespace ivftq;

extern "C" int ivftq_gemm_nt(const double* A, const void* B, int b_dtype, int64_t M, int N,
                             int K, void* C, int c_dtype, void* stream) {
  if (M < 0 || N < 0 || K < 1) {
    set_error("gemm_nt: bad shape");
    return IVFTQ_ERR_ARG;
  }
  if (M == 0 || N == 0) return 0;
  if ((N + TN - 1) / TN > 65535) {
    set_error("gemm_nt: N=%d too large", N);
    return IVFTQ_ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  // measured: the 128x128 kernel wins only for tall, narrow products (the
  // ingest rotation, 250k x 128 x 128: 490 vs 534 us); for the coarse
  // 10k x 1024 x 128 its one-block-per-SM occupancy loses (184 vs 167 us)
  if (M >= 65536 && N >= BN2 / 2 && N <= 256) {
    dim3 g2((unsigned)((M + BM2 - 1) / BM2), (N + BN2 - 1) / BN2);
    if (b_dtype == IVFTQ_F32 && c_dtype == IVFTQ_F64)
      gemm_nt_big_kernel<float, double><<<g2, 256, 0, s>>>(A, (const float*)B, M, N, K, (double*)C);
    else if (b_dtype == IVFTQ_F64 && c_dtype == IVFTQ_F64)
      gemm_nt_big_kernel<double, double><<<g2, 256, 0, s>>>(A, (const double*)B, M, N, K, (double*)C);
    else if (b_dtype == IVFTQ_F64 && c_dtype == IVFTQ_F32)
      gemm_nt_big_kernel<double, float><<<g2, 256, 0, s>>>(A, (const double*)B, M, N, K, (float*)C);
    else if (b_dtype == IVFTQ_F32 && c_dtype == IVFTQ_F32)
      gemm_nt_big_kernel<float, float><<<g2, 256, 0, s>>>(A, (const float*)B, M, N, K, (float*)C);
    else {
      set_error("gemm_nt: bad dtypes");
      return IVFTQ_ERR_ARG;
    }
    return check_launch("gemm_nt_big");
  }
  dim3 grid((unsigned)((M + TM - 1) / TM), (N + TN - 1) / TN);
  if (b_dtype == IVFTQ_F32 && c_dtype == IVFTQ_F64)
    gemm_nt_kernel<float, double><<<grid, 256, 0, s>>>(A, (const float*)B, M, N, K, (double*)C);
  else if (b_dtype == IVFTQ_F64 && c_dtype == IVFTQ_F64)
    gemm_nt_kernel<double, double><<<grid, 256, 0, s>>>(A, (const double*)B, M, N, K, (double*)C);
  else if (b_dtype == IVFTQ_F64 && c_dtype == IVFTQ_F32)
    gemm_nt_kernel<double, float><<<grid, 256, 0, s>>>(A, (const double*)B, M, N, K, (float*)C);
  else if (b_dtype == IVFTQ_F32 && c_dtype == IVFTQ_F32)
    gemm_nt_kernel<float, float><<<grid, 256, 0, s>>>(A, (const float*)B, M, N, K, (float*)C);
  else {
    set_error("gemm_nt: bad dtypes");
    return IVFTQ_ERR_ARG;
  }
  return check_launch("gemm_nt");
}

extern "C" int ivftq_assign(const double* xn, const float* centroids, int64_t n, int n_lists,
                            int dim, int32_t* list_out, void* stream) {
  if (n_lists < 1 || dim < 1) {
    set_error("assign: bad arguments");
    return IVFTQ_ERR_ARG;
  }
  if (n == 0) return 0;
  unsigned grid = (unsigned)((n + TM - 1) / TM);
  assign_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(xn, centroids, n, n_lists, dim,
                                                         list_out);
  return check_launch("assign");
}
