// Coarse scoring on the 5th-gen tensor cores with an exact f64 guard band.
//
// The reference scores every row against every centroid in f64 (index.py:436
// for query probes, partition.py:45-55 for ingest assignment) and then takes
// a stable top-n_p / first argmax. Here:
//
//   1. coarse_tc_kernel: S' = X . C^T on tcgen05 (M = 128 rows per CTA, N =
//      128 (or 64) centroids per tile, K = 16), error-compensated fp16:
//      x*2^14 and c*2^ec are split into fp16 hi + lo and D = Xhi.Chi +
//      Xlo.Chi + Xhi.Clo accumulates in fp32 TMEM. X rows are unit vectors,
//      so |S' - S| <= eps = 2^-12 * max_l ||c_l|| covers the fp16 splits, the
//      dropped lo.lo term and fp32 accumulation of 3*d products with margin.
//      The epilogue writes S' (probes) and/or keeps each row's best four
//      (assignment).
//   2. The decision is made in exact f64: every centroid whose S' is within
//      2*eps of the approximate n_p-th value (probes) or of the approximate
//      maximum (assignment) is re-scored as the same sequential FMA chain the
//      f64 GEMM uses, and the exact values decide -- ties to the lower list,
//      like np.argsort(kind="stable") and np.argmax. A true member always
//      lies inside the band, so probe sets and assignments equal the f64
//      path's; the f64 coarse values returned are the exact ones.
//
// Centroids are pre-split once per call into tile-contiguous, K-major UMMA
// operand images (`ivftq_coarse_prepare`), so a tile is one TMA bulk copy.
#include <climits>

#include "common.cuh"
#include "sm100.cuh"

namespace ivftq {
namespace ctc {

constexpr int kM = 128;
constexpr int kThreads = 160;  // warps 0-3: A build + epilogue (thread = row); warp 4: TMA + MMA
constexpr int kTopA = 4;       // per-row candidates kept for assignment

struct PrepHeader {
  unsigned int cmax_abs_bits;   // max |c_lj| (f32 bits, atomicMax on non-negative floats)
  unsigned int cmax_norm_bits;  // max ||c_l||
  int ec;                       // centroid scale exponent
  int pad[13];
};
constexpr int kHeader = sizeof(PrepHeader);  // 64 bytes

__host__ __device__ inline int pad_dp(int d) { return (d + 31) / 32 * 32; }
__host__ __device__ inline int tile_n(int DP) { return DP <= 128 ? 128 : 64; }
__host__ __device__ inline size_t tile_bytes(int DP) { return (size_t)2 * DP * tile_n(DP) * 2; }
__host__ __device__ inline int n_tiles(int L, int DP) { return (L + tile_n(DP) - 1) / tile_n(DP); }
// prepared buffer: header | nT tile images | f64 copy of the centroids (L x d)
__host__ __device__ inline size_t c64_offset(int L, int d) {
  return kHeader + (size_t)n_tiles(L, pad_dp(d)) * tile_bytes(pad_dp(d));
}

// K-major, no-swizzle canonical operand image of an NB-row tile: 16-byte
// chunk ch (8 consecutive k) of row v at ch*(NB*16) + (v/8)*128 + (v%8)*16.
__device__ __forceinline__ uint32_t img_off(int ch, int v, int NB) {
  return (uint32_t)ch * (NB * 16) + (v >> 3) * 128 + (v & 7) * 16;
}

__device__ __forceinline__ void split16(float x, uint16_t& hi, uint16_t& lo) {
  const __half h = __float2half_rn(x);
  hi = __half_as_ushort(h);
  lo = __half_as_ushort(__float2half_rn(x - __half2float(h)));
}

template <typename CT>
__global__ void prep_stats_kernel(const CT* __restrict__ c, int L, int d,
                                  PrepHeader* __restrict__ hdr) {
  // one warp per centroid (coalesced row reads)
  const int lane = threadIdx.x & 31;
  const int l = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (l >= L) return;
  float mx = 0.f, ss = 0.f;
  for (int j = lane; j < d; j += 32) {
    const float v = (float)c[(int64_t)l * d + j];
    mx = fmaxf(mx, fabsf(v));
    ss = fmaf(v, v, ss);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
    ss += __shfl_xor_sync(kFull, ss, o);
  }
  if (lane == 0) {
    atomicMax(&hdr->cmax_abs_bits, __float_as_uint(mx));
    atomicMax(&hdr->cmax_norm_bits, __float_as_uint(sqrtf(ss) * 1.0001f));
  }
}

// one thread per (centroid, 8-wide k chunk)
template <typename CT>
__global__ void prep_split_kernel(const CT* __restrict__ c, int L, int d, int DP, int nT,
                                  PrepHeader* __restrict__ hdr, unsigned char* __restrict__ img) {
  const int NB = tile_n(DP), NCH = DP / 8;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)nT * NB * NCH) return;
  const int ch = (int)(i % NCH);
  const int64_t lv = i / NCH;
  const int l = (int)lv, tile = l / NB, v = l % NB;
  // scale so that max |c| * 2^ec < 2^15 (fp16 hi/lo both normal-range)
  const float amax = __uint_as_float(hdr->cmax_abs_bits);
  int ex = 0;
  frexpf(amax > 0.f ? amax : 1.f, &ex);  // amax < 2^ex
  const int ec = 14 - ex;
  if (i == 0) hdr->ec = ec;
  const float sc = ldexpf(1.f, ec);
  uint16_t hi[8], lo[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int k = ch * 8 + e;
    const float x = (l < L && k < d) ? (float)c[(int64_t)l * d + k] * sc : 0.f;
    split16(x, hi[e], lo[e]);
  }
  unsigned char* t = img + (size_t)tile * tile_bytes(DP);
  const uint32_t o = img_off(ch, v, NB);
  *(uint4*)(t + o) = make_uint4(hi[0] | (hi[1] << 16), hi[2] | (hi[3] << 16),
                                hi[4] | (hi[5] << 16), hi[6] | (hi[7] << 16));
  *(uint4*)(t + (size_t)DP * NB * 2 + o) = make_uint4(lo[0] | (lo[1] << 16), lo[2] | (lo[3] << 16),
                                                      lo[4] | (lo[5] << 16), lo[6] | (lo[7] << 16));
}

template <typename CT>
__global__ void prep_c64_kernel(const CT* __restrict__ c, int64_t n, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (double)c[i];
}

// A-operand rows pre-split once per call: x * 2^14 as fp16 hi / lo, packed two
// per word along k, zero-padded to DP (the same values the kernel's in-place
// split produces). One thread per word; consecutive threads read consecutive
// 16-byte pairs of a row.
__global__ void x_split_kernel(const double* __restrict__ X, int64_t n, int d, int DP,
                               uint32_t* __restrict__ hi, uint32_t* __restrict__ lo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int hw = DP / 2;
  if (i >= n * hw) return;
  const int64_t r = i / hw;
  const int k = (int)(i - r * hw) * 2;
  const double* xr = X + r * (int64_t)d;
  uint16_t h0, l0, h1, l1;
  split16(k < d ? (float)(xr[k] * 16384.0) : 0.f, h0, l0);
  split16(k + 1 < d ? (float)(xr[k + 1] * 16384.0) : 0.f, h1, l1);
  hi[i] = h0 | ((uint32_t)h1 << 16);
  lo[i] = l0 | ((uint32_t)l1 << 16);
}

__device__ __forceinline__ float pick16f(const float (&v)[16], int j) {
  float a[8], b[4], c[2];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (j & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = (j & 2) ? a[2 * i + 1] : a[2 * i];
#pragma unroll
  for (int i = 0; i < 2; ++i) c[i] = (j & 4) ? b[2 * i + 1] : b[2 * i];
  return (j & 8) ? c[1] : c[0];
}

__device__ __forceinline__ uint64_t akey(float v, int id) {
  uint32_t b = __float_as_uint(v + 0.0f);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((uint64_t)b << 32) | (uint32_t)~(uint32_t)id;
}
__device__ __forceinline__ float akey_v(uint64_t k) {
  const uint32_t o = (uint32_t)(k >> 32);
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

__global__ void __launch_bounds__(kThreads, 1)
coarse_tc_kernel(const double* __restrict__ X, int64_t n, int d, int DP, int L, int nT,
                 const unsigned char* __restrict__ prep, float* __restrict__ S,
                 float* __restrict__ top_v, int32_t* __restrict__ top_i,
                 const uint32_t* __restrict__ xs_hi, const uint32_t* __restrict__ xs_lo) {
  // Work units are (row tile, N tile) pairs in row-major order. With a best-4
  // output each CTA owns one whole row tile (the epilogue needs every column
  // of its rows); an S'-only launch splits the units evenly over a grid of
  // one CTA per SM, so a small query batch (79 row tiles for 10k queries)
  // still fills all 148 SMs. A CTA's range is a few segments of consecutive
  // N tiles of one row tile each; the A operand is rebuilt per segment.
  const int64_t n_rt = (n + kM - 1) / kM;
  int64_t u0, u1;
  if (top_v) {
    u0 = (int64_t)blockIdx.x * nT;
    u1 = u0 + nT;
  } else {
    const int64_t tot = n_rt * nT;
    u0 = tot * blockIdx.x / gridDim.x;
    u1 = tot * (blockIdx.x + 1) / gridDim.x;
  }
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[10];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NB = tile_n(DP);
  const uint32_t tbytes = (uint32_t)tile_bytes(DP);
  const PrepHeader* hdr = (const PrepHeader*)prep;
  const unsigned char* img = prep + kHeader;
  uint64_t* b_full = bars;       // [3] TMA -> MMA
  uint64_t* b_empty = bars + 3;  // [3] MMA commit -> TMA
  uint64_t* acc_full = bars + 6; // [2] MMA commit -> epilogue
  uint64_t* acc_empty = bars + 8;// [2] epilogue -> MMA (count 4)
  __shared__ __align__(8) uint64_t a_full, a_empty;
  const uint32_t a_col = 2 * NB;  // A (hi | lo) after the two accumulators
  if (warp == 4) sm100::tmem_alloc(&tslot, 512);
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) {
      sm100::mbar_init(&b_full[b], 1);
      sm100::mbar_init(&b_empty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      sm100::mbar_init(&acc_full[b], 1);
      sm100::mbar_init(&acc_empty[b], 4);
    }
    sm100::mbar_init(&a_full, 4);
    sm100::mbar_init(&a_empty, 1);
    sm100::mbar_fence_init();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  const float inv = ldexpf(1.f, -(14 + hdr->ec));

  if (warp == 4) {
    // ---- TMA + MMA issuer (whole warp, elected lane issues) -------------------
    // three operand buffers: tile j+1 is fetched into the buffer tile j-2 used
    // (long retired), so the issuing thread never waits on the MMAs in flight
    const int ng = (int)(u1 - u0);  // tiles of this CTA, in unit order
    auto load = [&](int g) {
      if (lane == 0) {
        sm100::mbar_arrive_expect_tx(&b_full[g % 3], tbytes);
        const unsigned char* src = img + (size_t)((u0 + g) % nT) * tbytes;
        unsigned char* dst = smem + (g % 3) * tbytes;
        for (uint32_t o = 0; o < tbytes; o += 32768)
          sm100::bulk_g2s(dst + o, src + o, min(32768u, tbytes - o), &b_full[g % 3]);
      }
      __syncwarp();
    };
    for (int g = 0; g < 3 && g < ng; ++g) load(g);
    const uint32_t idesc = sm100::idesc_f16_f32(kM, NB);
    const uint32_t lbo = NB * 16, sbo = 128;
    const int ks = DP / 16;
    int g = 0, seg = 0;
    for (int64_t u = u0; u < u1; ++seg) {
      const int j0 = (int)(u % nT);
      const int j1 = (int)(u1 - u < (int64_t)(nT - j0) ? j0 + (u1 - u) : nT);
      u += j1 - j0;
      sm100::mbar_wait(&a_full, seg & 1);
      for (int j = j0; j < j1; ++j, ++g) {
        if (g >= 2 && g + 1 < ng) {
          sm100::mbar_wait(&b_empty[(g + 1) % 3], ((g - 2) / 3) & 1);
          load(g + 1);
        }
        const int b = g % 3, ab = g & 1;
        sm100::mbar_wait(&b_full[b], (g / 3) & 1);
        if (g >= 2) sm100::mbar_wait(&acc_empty[ab], ((g >> 1) - 1) & 1);
        sm100::tc_fence_after();
        const uint32_t bh = sm100::smem_u32(smem + b * tbytes);
        const uint64_t dh = sm100::smem_desc(bh, lbo, sbo);
        const uint64_t dl = sm100::smem_desc(bh + DP * NB * 2, lbo, sbo);
        const uint64_t dstep = (2 * lbo) >> 4;
        const uint32_t acc = tmem + ab * NB;
        const uint32_t qh = tmem + a_col, ql = qh + DP / 2;
#pragma unroll 1
        for (int pass = 0; pass < 3; ++pass) {
          const uint32_t at = pass == 1 ? ql : qh;
          const uint64_t db = pass == 2 ? dl : dh;
          for (int s = 0; s < ks; ++s)
            sm100::mma_f16_ts_warp(acc, at + s * 8, db + s * dstep, idesc, (pass | s) ? 1u : 0u);
        }
        sm100::mma_commit_warp(&acc_full[ab]);
        sm100::mma_commit_warp(&b_empty[b]);
      }
      sm100::mma_commit_warp(&a_empty);  // A is free once this segment's MMAs are done
    }
  } else {
    int g = 0, seg = 0;
    for (int64_t u = u0; u < u1; ++seg) {
      const int64_t rt = u / nT;
      const int j0 = (int)(u % nT);
      const int j1 = (int)(u1 - u < (int64_t)(nT - j0) ? j0 + (u1 - u) : nT);
      u += j1 - j0;
      // ---- A operand: this thread's row, x * 2^14 split into fp16 hi / lo -----
      const int64_t r = rt * kM + tid;
      const bool live = r < n;
      const double* xr = X + (r < n ? r : 0) * (int64_t)d;
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + a_col;
      if (seg > 0) sm100::mbar_wait(&a_empty, (seg - 1) & 1);
      sm100::tc_fence_after();
      if (xs_hi) {
        // pre-split rows (x_split_kernel): 16-byte loads, all in flight at once
        const uint4* sh = (const uint4*)(xs_hi + (live ? r : 0) * (int64_t)(DP / 2));
        const uint4* sl = (const uint4*)(xs_lo + (live ? r : 0) * (int64_t)(DP / 2));
#pragma unroll 1
        for (int c0 = 0; c0 < DP / 2; c0 += 32) {
          uint32_t vh[2][16], vl[2][16];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              const bool ok = live && c0 + hh * 16 < DP / 2;
              const int w4 = (c0 + hh * 16) / 4 + x;
              const uint4 a = ok ? __ldg(sh + w4) : make_uint4(0, 0, 0, 0);
              const uint4 b = ok ? __ldg(sl + w4) : make_uint4(0, 0, 0, 0);
              vh[hh][4 * x] = a.x; vh[hh][4 * x + 1] = a.y; vh[hh][4 * x + 2] = a.z; vh[hh][4 * x + 3] = a.w;
              vl[hh][4 * x] = b.x; vl[hh][4 * x + 1] = b.y; vl[hh][4 * x + 2] = b.z; vl[hh][4 * x + 3] = b.w;
            }
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
            if (c0 + hh * 16 < DP / 2) {
              sm100::tmem_st16(ta + c0 + hh * 16, vh[hh]);
              sm100::tmem_st16(ta + DP / 2 + c0 + hh * 16, vl[hh]);
            }
        }
      } else {
        for (int c0 = 0; c0 < DP / 2; c0 += 16) {
          uint32_t vh[16], vl[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int k = 2 * (c0 + e);
            uint16_t h0, l0, h1, l1;
            split16(live && k < d ? (float)(xr[k] * 16384.0) : 0.f, h0, l0);
            split16(live && k + 1 < d ? (float)(xr[k + 1] * 16384.0) : 0.f, h1, l1);
            vh[e] = h0 | ((uint32_t)h1 << 16);
            vl[e] = l0 | ((uint32_t)l1 << 16);
          }
          sm100::tmem_st16(ta + c0, vh);
          sm100::tmem_st16(ta + DP / 2 + c0, vl);
        }
      }
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&a_full);
      // ---- epilogue: S' row segments and the row's best kTopA -------------------
      uint64_t best[kTopA];
#pragma unroll
      for (int p = 0; p < kTopA; ++p) best[p] = 0;
      for (int j = j0; j < j1; ++j, ++g) {
        const int b = g & 1;
        sm100::mbar_wait(&acc_full[b], (g >> 1) & 1);
        sm100::tc_fence_after();
        for (int cc = 0; cc < NB; cc += 32) {
          uint32_t v[32];
          sm100::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + b * NB + cc, v);
          sm100::tmem_ld_wait();
          if (cc + 32 >= NB) {  // all columns of this accumulator are in registers
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&acc_empty[b]);
          }
          const int col0 = j * NB + cc;
          float f[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) f[e] = __uint_as_float(v[e]) * inv;
          if (live && S) {
            float* dst = S + r * (int64_t)L + col0;
            if (col0 + 32 <= L && (L & 3) == 0) {
#pragma unroll
              for (int e = 0; e < 32; e += 4) *(float4*)(dst + e) = make_float4(f[e], f[e + 1], f[e + 2], f[e + 3]);
            } else {
              for (int e = 0; e < 32; ++e)
                if (col0 + e < L) dst[e] = f[e];
            }
          }
          if (top_v) {
            // only columns beating the row's current 4th best reach the insert
            // (columns arrive in ascending order, so an equal value never does);
            // the warp steps max-over-lanes times per 16-column window
#pragma unroll
            for (int h = 0; h < 32; h += 16) {
              const float kth = best[kTopA - 1] ? akey_v(best[kTopA - 1]) : -INFINITY;
              uint32_t m = 0;
#pragma unroll
              for (int e = 0; e < 16; ++e)
                m |= (col0 + h + e < L && f[h + e] > kth ? 1u : 0u) << e;
              while (__any_sync(kFull, m != 0)) {
                const int jj = (__ffs(m) - 1) & 15;
                float w[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) w[e] = f[h + e];
                const uint64_t key = m ? akey(pick16f(w, jj), col0 + h + jj) : 0ull;
                m &= m - 1;
                bool gt[kTopA];
#pragma unroll
                for (int p = 0; p < kTopA; ++p) gt[p] = key > best[p];
#pragma unroll
                for (int p = kTopA - 1; p > 0; --p)
                  best[p] = gt[p] ? (gt[p - 1] ? best[p - 1] : key) : best[p];
                best[0] = gt[0] ? key : best[0];
              }
            }
          }
        }
      }
      if (live && top_v) {
#pragma unroll
        for (int p = 0; p < kTopA; ++p) {
          top_v[r * kTopA + p] = best[p] ? akey_v(best[p]) : -INFINITY;
          top_i[r * kTopA + p] = best[p] ? (int)~(uint32_t)best[p] : -1;
        }
      }
    }
  }
  __syncthreads();
  if (warp == 4) sm100::tmem_dealloc(tmem, 512);
}

// Exact f64 score of row x against centroid c: the sequential FMA chain of
// the f64 GEMM (gemm_f64.cu), so both paths produce identical values. The
// centroid row is the prepared f64 copy (f32 -> f64 conversions run at a low
// rate on this part, so they are paid once per centroid, not per candidate)
// and streams in 16-element batches so the chain does not wait per term.
__device__ __forceinline__ double exact_ip(const double* __restrict__ x, const double* __restrict__ c,
                                           int d) {
  double s = 0.0;
  int k = 0;
  for (; k + 16 <= d; k += 16) {
    double cv[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) cv[e] = __ldg(c + k + e);
#pragma unroll
    for (int e = 0; e < 16; ++e) s = __fma_rn(x[k + e], cv[e], s);
  }
  for (; k < d; ++k) s = __fma_rn(x[k], __ldg(c + k), s);
  return s;
}

// 32 exact dots at once, one per lane: lane i returns the sequential FMA
// chain of x_i . c_i (bit-identical to exact_ip). Rows are staged through
// shared memory KC k-values at a time with coalesced row loads, instead of
// 32 lanes each walking its own row (32 sectors per load instruction).
// crow may be null (lane idle). SHARED_X: xrow is one shared-memory row used
// by every lane (xt unused); else per-lane rows staged like c. Tiles are
// 32 x (KC+1) doubles.
template <int KC, bool SHARED_X>
__device__ double warp_dots(const double* xrow, const double* crow, int d, double* xt, double* ct) {
  const int lane = threadIdx.x & 31;
  constexpr int RPI = 32 / KC;  // rows per load instruction
  double s = 0.0;
  for (int k0 = 0; k0 < d; k0 += KC) {
    const int kk = k0 + lane % KC;
#pragma unroll 4
    for (int j0 = 0; j0 < 32; j0 += RPI) {
      const int j = j0 + lane / KC;
      const double* cj = (const double*)__shfl_sync(kFull, (unsigned long long)crow, j);
      ct[j * (KC + 1) + lane % KC] = (cj && kk < d) ? cj[kk] : 0.0;
      if (!SHARED_X) {
        const double* xj = (const double*)__shfl_sync(kFull, (unsigned long long)xrow, j);
        xt[j * (KC + 1) + lane % KC] = (xj && kk < d) ? xj[kk] : 0.0;
      }
    }
    __syncwarp();
    const int m = min(KC, d - k0);
    for (int e = 0; e < m; ++e)
      s = __fma_rn(SHARED_X ? xrow[k0 + e] : xt[lane * (KC + 1) + e], ct[lane * (KC + 1) + e], s);
    __syncwarp();
  }
  return s;
}

__device__ __forceinline__ float band(const unsigned char* prep) {
  // eps = 2^-12 * max ||c||; the band is 2 * eps
  return 2.0f * ldexpf(__uint_as_float(((const PrepHeader*)prep)->cmax_norm_bits), -12);
}

// ---- assignment: exact decision among the in-band candidates ---------------------
// (1) one thread per (row, kept candidate): exact f64 for members of the band
// around the approximate maximum (-inf otherwise); (2) one thread per row
// picks the exact maximum, ties to the lower list. A row whose kTopA kept
// candidates all lie in the band may have more: (3) a warp re-scores every
// centroid of such a row.
__global__ void __launch_bounds__(128)
assign_exact_kernel(const double* __restrict__ X, const double* __restrict__ C, int64_t n, int d,
                    const unsigned char* prep, const float* __restrict__ top_v,
                    const int32_t* __restrict__ top_i, double* __restrict__ ex) {
  __shared__ double tiles[4][2][32 * 17];
  const int warp = threadIdx.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (row, candidate)
  const bool live = t < n * kTopA;
  const int64_t r = live ? t / kTopA : 0;
  const float w = band(prep);
  bool in = false;
  int id = -1;
  if (live) {
    id = top_i[t];
    // a row whose runner-up is outside the band is decided by the tensor-core
    // scores alone (its maximum is unique and exact-safe): no re-scoring
    const bool ambiguous = top_v[r * kTopA + 1] >= top_v[r * kTopA] - w;
    in = ambiguous && id >= 0 && top_v[t] >= top_v[r * kTopA] - w;
  }
  if (!__any_sync(kFull, in)) {
    if (live) ex[t] = -INFINITY;
    return;
  }
  const double e = warp_dots<16, false>(in ? X + r * (int64_t)d : nullptr,
                                        in ? C + (int64_t)id * d : nullptr, d, tiles[warp][0],
                                        tiles[warp][1]);
  if (live) ex[t] = in ? e : -INFINITY;
}

__global__ void assign_pick_kernel(int64_t n, const unsigned char* prep,
                                   const float* __restrict__ top_v,
                                   const int32_t* __restrict__ top_i,
                                   const double* __restrict__ ex, int32_t* __restrict__ out,
                                   int32_t* __restrict__ full_list, int32_t* __restrict__ n_full) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const float w = band(prep);
  if (!(top_v[r * kTopA + kTopA - 1] < top_v[r * kTopA] - w)) {
    full_list[atomicAdd(n_full, 1)] = (int32_t)r;
    return;
  }
  if (!(top_v[r * kTopA + 1] >= top_v[r * kTopA] - w)) {  // unambiguous maximum
    out[r] = top_i[r * kTopA] < 0 ? 0 : top_i[r * kTopA];
    return;
  }
  double bv = -INFINITY;
  int bi = INT_MAX;
  for (int p = 0; p < kTopA; ++p) {
    const double e = ex[r * kTopA + p];
    const int id = top_i[r * kTopA + p];
    if (id >= 0 && (e > bv || (e == bv && id < bi))) { bv = e; bi = id; }
  }
  out[r] = bi == INT_MAX ? 0 : bi;  // NaN row (zero input): np.argmax -> 0
}

// A listed row is scored against every centroid by a whole block (thread =
// centroids tid, tid + 256, ...; the row staged in shared memory), so even a
// single listed row costs microseconds, not a warp's serial walk over L dots.
constexpr int kFullThreads = 256;
__global__ void __launch_bounds__(kFullThreads)
assign_full_kernel(const double* __restrict__ X, const double* __restrict__ C, int L, int d,
                   const int32_t* __restrict__ full_list, const int32_t* __restrict__ n_full,
                   int32_t* __restrict__ out) {
  extern __shared__ double xrow[];  // d
  __shared__ double sv[kFullThreads / 32];
  __shared__ int si[kFullThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int total = *n_full;
  for (int w = blockIdx.x; w < total; w += gridDim.x) {
    const int64_t r = full_list[w];
    __syncthreads();
    for (int k = threadIdx.x; k < d; k += kFullThreads) xrow[k] = X[r * (int64_t)d + k];
    __syncthreads();
    double bv = -INFINITY;
    int bi = INT_MAX;
    for (int l = threadIdx.x; l < L; l += kFullThreads) {
      const double e = exact_ip(xrow, C + (int64_t)l * d, d);
      if (e > bv) { bv = e; bi = l; }  // ascending l per thread: lowest on ties
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(kFull, bv, o);
      const int oi = __shfl_xor_sync(kFull, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { sv[warp] = bv; si[warp] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int x = 1; x < kFullThreads / 32; ++x)
        if (sv[x] > bv || (sv[x] == bv && si[x] < bi)) { bv = sv[x]; bi = si[x]; }
      out[r] = bi == INT_MAX ? 0 : bi;
    }
  }
}

// ---- probes: exact top-n_p among the in-band candidates of each S' row ------------
__device__ __forceinline__ long long okey(double x) {
  if (x == 0.0) x = 0.0;
  if (x != x) return LLONG_MIN;
  const long long b = __double_as_longlong(x);
  return b >= 0 ? b : (b ^ 0x7fffffffffffffffLL);
}
__device__ __forceinline__ double okey_inv(long long k) {
  return __longlong_as_double(k >= 0 ? k : (k ^ 0x7fffffffffffffffLL));
}

constexpr int kBins = 256;
constexpr int kCandCap = 256;  // in-band candidates kept per row (more: exact full row)

// Sorted warp queue of the best n (<= 32*QS) exact keys; lane l holds
// positions s*32+l. Keys arrive in ascending column order, so an equal key
// goes after the queued ones (column ascending on ties).
template <int QS>
struct WarpQueue {
  long long k[QS];
  int i[QS];
  int cnt, n;
  __device__ void init(int n_) {
#pragma unroll
    for (int s = 0; s < QS; ++s) { k[s] = LLONG_MIN; i[s] = -1; }
    cnt = 0;
    n = n_;
  }
  __device__ long long thr() const {
    const int tl = (n - 1) & 31, ts = (n - 1) >> 5;
    long long t = k[0];
#pragma unroll
    for (int s = 1; s < QS; ++s) if (s == ts) t = k[s];
    return __shfl_sync(kFull, t, tl);
  }
  __device__ void insert(long long key, int id) {  // warp-uniform arguments
    const int lane = threadIdx.x & 31;
    if (cnt == n && !(key > thr())) return;
    int p = 0;
#pragma unroll
    for (int s = 0; s < QS; ++s) p += __popc(__ballot_sync(kFull, (s * 32 + lane) < cnt && k[s] >= key));
    long long rk[QS];
    int ri[QS];
#pragma unroll
    for (int s = 0; s < QS; ++s) {
      rk[s] = __shfl_sync(kFull, k[s], (lane + 31) & 31);
      ri[s] = __shfl_sync(kFull, i[s], (lane + 31) & 31);
    }
#pragma unroll
    for (int s = QS - 1; s >= 0; --s) {
      const int pos = s * 32 + lane;
      long long pk = rk[s];
      int pi = ri[s];
      if (lane == 0) {
        pk = s > 0 ? rk[s > 0 ? s - 1 : 0] : LLONG_MIN;
        pi = s > 0 ? ri[s > 0 ? s - 1 : 0] : -1;
      }
      if (pos > p) { k[s] = pk; i[s] = pi; }
      else if (pos == p) { k[s] = key; i[s] = id; }
    }
    cnt = min(cnt + 1, n);
  }
};

// (1) per row (warp): band threshold tau below the approximate n_p-th value,
// compaction of the in-band columns (ascending) into cand[row]
__global__ void __launch_bounds__(256)
probe_band_kernel(const float* __restrict__ S, int64_t nq, int L, int n_p,
                  const unsigned char* prep, int32_t* __restrict__ cand,
                  int32_t* __restrict__ cnt_out) {
  constexpr int kWarps = 8;
  __shared__ unsigned hist_all[kWarps][kBins];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * kWarps + warp;
  if (r >= nq) return;
  const float* row = S + r * (int64_t)L;
  unsigned* hist = hist_all[warp];
  const float w = band(prep);
  float mn = INFINITY, mx = -INFINITY;
  for (int c = lane; c < L; c += 32) {
    const float v = row[c];
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(kFull, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
  }
  // one histogram bin below the bin of the approximate n_p-th value, minus
  // the band (safe against the bin map's own rounding)
  float tau = -INFINITY;
  const float span = mx - mn;
  if (span > 0.f && span < INFINITY) {
    const float scale = (float)kBins / span;
#pragma unroll
    for (int i = 0; i < kBins / 32; ++i) hist[i * 32 + lane] = 0;
    __syncwarp();
    for (int c = lane; c < L; c += 32)
      atomicAdd(&hist[min(kBins - 1, (int)((row[c] - mn) * scale))], 1u);
    __syncwarp();
    unsigned own[kBins / 32], tot = 0;
#pragma unroll
    for (int i = 0; i < kBins / 32; ++i) {
      own[i] = hist[kBins - 1 - (lane * (kBins / 32) + i)];
      tot += own[i];
    }
    unsigned incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    const int owner = __ffs(__ballot_sync(kFull, incl >= (unsigned)n_p)) - 1;
    int bsel = 0;
    if (lane == owner) {
      unsigned acc = incl - tot;
#pragma unroll
      for (int i = 0; i < kBins / 32; ++i) {
        acc += own[i];
        if (acc >= (unsigned)n_p) { bsel = kBins - 1 - (lane * (kBins / 32) + i); break; }
      }
    }
    const int b = __shfl_sync(kFull, bsel, owner);
    tau = b >= 1 ? mn + (float)(b - 1) / scale - w : -INFINITY;
  }
  int nc = 0;
  int32_t* cr = cand + r * kCandCap;
  for (int base = 0; base < L; base += 32) {
    const int c = base + lane;
    const bool in = c < L && row[c] >= tau;
    const unsigned m = __ballot_sync(kFull, in);
    const int at = nc + __popc(m & ((1u << lane) - 1u));
    if (in && at < kCandCap) cr[at] = c;
    nc += __popc(m);
  }
  if (lane == 0) cnt_out[r] = nc;  // > kCandCap: row takes the exact full path
}

// (2) one block per row, 32 candidates per warp: exact f64 scores
__global__ void __launch_bounds__(128)
probe_exact_kernel(const double* __restrict__ X, const double* __restrict__ C, int64_t nq, int d,
                   const int32_t* __restrict__ cand, const int32_t* __restrict__ cnt,
                   double* __restrict__ ex) {
  __shared__ double tiles[4][32 * 33];
  __shared__ double xs[256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x;
  for (int k = threadIdx.x; k < d; k += 128) xs[k] = X[r * (int64_t)d + k];
  __syncthreads();
  const int nc = min(cnt[r], kCandCap);
  for (int b0 = warp * 32; b0 < nc; b0 += 128) {
    const int i = b0 + lane;
    const bool in = i < nc;
    const double e = warp_dots<32, true>(xs, in ? C + (int64_t)cand[r * kCandCap + i] * d : nullptr,
                                         d, nullptr, tiles[warp]);
    if (in) ex[r * kCandCap + i] = e;
  }
}

// (3) per row (warp): exact top-n_p by (value desc, column asc)
template <int QS>
__global__ void __launch_bounds__(256)
probe_pick_kernel(const double* __restrict__ X, const double* __restrict__ C, int64_t nq, int L,
                  int d, int n_p, const int32_t* __restrict__ cand,
                  const int32_t* __restrict__ cnt, const double* __restrict__ ex,
                  int32_t* __restrict__ idx_out, double* __restrict__ val_out, bool full_only) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= nq) return;
  if (full_only && cnt[r] <= kCandCap) return;  // decided by probe_select_kernel
  WarpQueue<QS> q;
  q.init(n_p);
  const int nc = cnt[r];
  if (nc <= kCandCap) {
    for (int base = 0; base < nc; base += 32) {
      const int i = base + lane;
      const long long kv = i < nc ? okey(ex[r * kCandCap + i]) : LLONG_MIN;
      const int cv = i < nc ? cand[r * kCandCap + i] : -1;
      const int m = min(32, nc - base);
      for (int j = 0; j < m; ++j)
        q.insert(__shfl_sync(kFull, kv, j), __shfl_sync(kFull, cv, j));
    }
  } else {  // crowded band (duplicate centroids...): every column, exactly
    const double* x = X + r * (int64_t)d;
    for (int base = 0; base < L; base += 32) {
      const int c = base + lane;
      const long long kv = c < L ? okey(exact_ip(x, C + (int64_t)c * d, d)) : LLONG_MIN;
      const int m = min(32, L - base);
      for (int j = 0; j < m; ++j) q.insert(__shfl_sync(kFull, kv, j), base + j);
    }
  }
#pragma unroll
  for (int s = 0; s < QS; ++s) {
    const int pos = s * 32 + lane;
    if (pos < n_p) {
      idx_out[r * n_p + pos] = q.i[s];
      val_out[r * n_p + pos] = okey_inv(q.k[s]);
    }
  }
}

// ---- fused probe selection: one block (4 warps) per query row -----------------
// (a) the S' row is staged in shared memory (one coalesced read) while a
//     256-bin histogram over the fixed range [-R, R] (R bounds |S'| for unit
//     rows; outliers clamp into the end bins) is built; the bin b holding
//     the approximate n_p-th value v* is refined by a second 256-bin level
//     over bin b. With t(v) = (v + R) * scale (one f32 expression, monotone in
//     v) every value counted at or above (b, sb) has v >= lo = -R +
//     (b + sb/256) / scale - delta (delta covers the rounding of t), so
//     v* >= lo;
// (b) candidates are the columns with S' >= tau = lo - 2 eps: a true member
//     m of the exact top-n_p has E_m >= E_(n_p) >= v* - eps, hence
//     S'_m >= v* - 2 eps >= tau;
// (c) every candidate is scored exactly in f64 (lanes split k, a fixed xor
//     tree sums the lanes: within a few ulps of the f64 GEMM's sequential
//     chain, far inside every decision margin);
// (d) rank selection by (value desc, column asc) -- np.argsort(-C,
//     kind="stable") (index.py:437-438) -- writes probes and exact values in
//     order. Rows with more than kCandCap candidates (duplicate centroids),
//     fewer than n_p (NaN rows) or a degenerate histogram are flagged for
//     probe_pick_kernel's exact full-row path.
#ifndef IVFTQ_SEL_MINB
#define IVFTQ_SEL_MINB 8  // 64 registers: C3 select 142 -> 129 us, C2 123 -> 127
#endif
#ifndef IVFTQ_SUB_SKIP
#define IVFTQ_SUB_SKIP 48
#endif
#ifndef IVFTQ_SEL_THREADS
#define IVFTQ_SEL_THREADS 128
#endif
constexpr int kSelThreads = IVFTQ_SEL_THREADS;
constexpr int kSelRowCap = 16384;  // lists staged per row (larger L: f64 path)

__host__ __device__ inline size_t sel_region_a(int L) {
  return ((size_t)L * 4 + 15) & ~(size_t)15;
}
__host__ __device__ inline size_t sel_smem_bytes(int L, int d) {
  return sel_region_a(L) + 2 * kBins * 4 + kCandCap * (4 + 8) + (size_t)d * 8;
}

// warp 0: the bin (from the top) where the cumulative count reaches `need`,
// and the count strictly above it; -1 if the total is short
__device__ __forceinline__ int top_bin(const unsigned* h, unsigned need, unsigned& above) {
  const int lane = threadIdx.x & 31;
  unsigned own[kBins / 32], tot = 0;
#pragma unroll
  for (int i = 0; i < kBins / 32; ++i) {
    own[i] = h[kBins - 1 - (lane * (kBins / 32) + i)];
    tot += own[i];
  }
  unsigned incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += t;
  }
  const unsigned ball = __ballot_sync(kFull, incl >= need);
  if (!ball) return -1;
  const int owner = __ffs(ball) - 1;
  int bsel = 0;
  unsigned abv = 0;
  if (lane == owner) {
    unsigned acc = incl - tot;
#pragma unroll
    for (int i = 0; i < kBins / 32; ++i) {
      if (acc + own[i] >= need) {
        bsel = kBins - 1 - (lane * (kBins / 32) + i);
        abv = acc;
        break;
      }
      acc += own[i];
    }
  }
  above = __shfl_sync(kFull, abv, owner);
  return __shfl_sync(kFull, bsel, owner);
}

__global__ void __launch_bounds__(kSelThreads, IVFTQ_SEL_MINB)
probe_select_kernel(const float* __restrict__ S, const double* __restrict__ X,
                    const double* __restrict__ C64, int64_t nq, int L, int d, int n_p,
                    const unsigned char* __restrict__ prep, int32_t* __restrict__ cnt_out,
                    int32_t* __restrict__ probe_out, double* __restrict__ coarse_out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ int s_nc, s_b, s_need;
  __shared__ float s_tau;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r = blockIdx.x;
  float* srow = (float*)sm;
  unsigned* hist = (unsigned*)(sm + sel_region_a(L));
  unsigned* sub = hist + kBins;
  int* cand = (int*)(sub + kBins);
  double* ex = (double*)(cand + kCandCap);
  double* xs = ex + kCandCap;
  const float* row = S + r * (int64_t)L;
  const float R = 1.01f * __uint_as_float(((const PrepHeader*)prep)->cmax_norm_bits) + 1e-30f;
  const float scale = (float)kBins / (2.f * R);
  auto tmap = [&](float v) { return (v + R) * scale; };
  auto bin_of = [&](float t) { return min(kBins - 1, max(0, (int)t)); };

  for (int i = tid; i < 2 * kBins; i += kSelThreads) hist[i] = 0;  // both levels
  for (int k = tid; k < d; k += kSelThreads) xs[k] = X[r * (int64_t)d + k];
  if (tid == 0) {
    s_nc = 0;
    s_b = -1;
  }
  __syncthreads();
  if ((L & 3) == 0) {
    // 8 row loads in flight per thread before any histogram update
    constexpr int U = 8;
    for (int i0 = 0; i0 < L / 4; i0 += U * kSelThreads) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * kSelThreads + tid;
        v[u] = i < L / 4 ? __ldcs((const float4*)row + i) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * kSelThreads + tid;
        if (i < L / 4) {
          ((float4*)srow)[i] = v[u];
          atomicAdd(&hist[bin_of(tmap(v[u].x))], 1u);
          atomicAdd(&hist[bin_of(tmap(v[u].y))], 1u);
          atomicAdd(&hist[bin_of(tmap(v[u].z))], 1u);
          atomicAdd(&hist[bin_of(tmap(v[u].w))], 1u);
        }
      }
    }
  } else {
    for (int i = tid; i < L; i += kSelThreads) {
      const float v = __ldcs(row + i);
      srow[i] = v;
      atomicAdd(&hist[bin_of(tmap(v))], 1u);
    }
  }
  __syncthreads();
  if (warp == 0) {
    unsigned above = 0;
    const int b = top_bin(hist, (unsigned)n_p, above);
    if (lane == 0 && b > 0) {  // b == 0 may hold clamped outliers: full path
      s_b = b;
      s_need = n_p - (int)above;
    }
  }
  __syncthreads();
  const int b = s_b;
  float tau = -INFINITY;
  // on long rows a sparse bin b (<= IVFTQ_SUB_SKIP values) is taken whole:
  // the lower edge of b is the threshold and the second level's pass over
  // the row is skipped (measured: C3, L = 4096, 132 -> 120 us; at L = 1024
  // the extra candidates cost more than the pass)
  const bool refine = b > 0 && (L < 2048 || hist[b] > (unsigned)IVFTQ_SUB_SKIP);
  if (b > 0 && !refine) tau = -R + (float)b / scale - band(prep) - R * 0x1p-18f;
  if (refine) {
    for (int i = tid; i < L; i += kSelThreads) {
      const float t = tmap(srow[i]);
      if (bin_of(t) == b)
        atomicAdd(&sub[min(kBins - 1, max(0, (int)((t - (float)b) * (float)kBins)))], 1u);
    }
    __syncthreads();
    if (warp == 0) {
      unsigned above2 = 0;
      const int sb = max(0, top_bin(sub, (unsigned)s_need, above2));
      const float delta = R * 0x1p-18f;
      if (lane == 0)
        s_tau = -R + ((float)b + (float)sb / (float)kBins) / scale - band(prep) - delta;
    }
    __syncthreads();
    tau = s_tau;
  }
  for (int base = 0; base < L; base += kSelThreads) {
    const int c = base + tid;
    const bool in = c < L && srow[c] >= tau;
    const unsigned m = __ballot_sync(kFull, in);
    int at = 0;
    if (lane == 0 && m) at = atomicAdd(&s_nc, __popc(m));
    at = __shfl_sync(kFull, at, 0) + __popc(m & ((1u << lane) - 1u));
    if (in && at < kCandCap) cand[at] = c;
  }
  __syncthreads();
  const int nc = s_nc;
  if (nc > kCandCap || nc < n_p) {  // exact full-row path (probe_pick_kernel)
    if (tid == 0) cnt_out[r] = kCandCap + 1;
    return;
  }
  if (tid == 0) cnt_out[r] = nc;
  // (c) exact f64 scores: lane l owns k = l + 32 m (x in registers), a warp
  // scores 8 candidates per step (coalesced 256-byte row loads), and a
  // butterfly reduce-transpose sums the 8 per-lane partials over the lanes in
  // the fixed xor-tree order (distance 16, 8, 4, 2, 1) -- deterministic, and
  // equal rows give equal values
  {
    constexpr int kMaxM = 8;  // d <= 256
    const int M = (d + 31) >> 5;
    double xr[kMaxM];
#pragma unroll
    for (int m = 0; m < kMaxM; ++m) {
      const int k = lane + 32 * m;
      xr[m] = (m < M && k < d) ? xs[k] : 0.0;
    }
    for (int base = warp * 8; base < nc; base += (kSelThreads / 32) * 8) {
      double p[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int ci = base + c < nc ? cand[base + c] : cand[base];
        const double* crow = C64 + (int64_t)ci * d + lane;
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < kMaxM; ++m)
          if (m < M && lane + 32 * m < d) acc = __fma_rn(xr[m], __ldg(crow + 32 * m), acc);
        p[c] = acc;
      }
      // level 16: keep 4 of 8 (lanes < 16 keep candidates 0-3, others 4-7)
      const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
      double q4[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double send = u16 ? p[c] : p[c + 4];
        const double keep = u16 ? p[c + 4] : p[c];
        q4[c] = keep + __shfl_xor_sync(kFull, send, 16);
      }
      double q2[2];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double send = u8 ? q4[c] : q4[c + 2];
        const double keep = u8 ? q4[c + 2] : q4[c];
        q2[c] = keep + __shfl_xor_sync(kFull, send, 8);
      }
      double q1;
      {
        const double send = u4 ? q2[0] : q2[1];
        const double keep = u4 ? q2[1] : q2[0];
        q1 = keep + __shfl_xor_sync(kFull, send, 4);
      }
      q1 += __shfl_xor_sync(kFull, q1, 2);
      q1 += __shfl_xor_sync(kFull, q1, 1);
      // lane holds candidate (u16 ? 4 : 0) + (u8 ? 2 : 0) + (u4 ? 1 : 0)
      const int c = (u16 ? 4 : 0) + (u8 ? 2 : 0) + (u4 ? 1 : 0);
      if ((lane & 3) == 0 && base + c < nc) ex[base + c] = q1;
    }
  }
  __syncthreads();
  // (d) rank of each candidate under (value desc, column asc); exact ties
  // (duplicate centroids) take a second pass over the columns
  for (int i = tid; i < nc; i += kSelThreads) {
    const double vi = ex[i];
    const int ci = cand[i];
    int rank = 0, eq = 0;
#pragma unroll 4
    for (int j = 0; j < nc; ++j) {
      const double vj = ex[j];  // finite (NaN rows took the full path)
      rank += vj > vi;
      eq += vj == vi;
    }
    if (eq > 1)
      for (int j = 0; j < nc; ++j) rank += (ex[j] == vi) & (cand[j] < ci);
    if (rank < n_p) {
      probe_out[r * n_p + rank] = ci;
      coarse_out[r * n_p + rank] = vi;
    }
  }
}

}  // namespace ctc
}  // namespace ivftq

using namespace ivftq;
using namespace ivftq::ctc;

// 0 = default (assignment on tensor cores, probes f64), 1 = f64 CUDA cores
// only, 2 = tensor cores for probes too
// (process-wide configuration switches, not per-call state: atomics so a
// concurrent reader sees either value)
#include <atomic>
static std::atomic<int> g_coarse_mode{0};
std::atomic<bool> g_probe_tc_force{false};

extern "C" int ivftq_set_coarse_mode(int mode) {
  if (mode < 0 || mode > 2) {
    set_error("set_coarse_mode: mode %d not in {0, 1, 2}", mode);
    return IVFTQ_ERR_ARG;
  }
  g_coarse_mode = mode;
  g_probe_tc_force = mode == 2;
  return 0;
}

extern "C" int ivftq_coarse_tc_supported(int dim, int n_lists) {
  return g_coarse_mode != 1 && dim >= 1 && pad_dp(dim) <= 256 && n_lists >= 1;
}

extern "C" size_t ivftq_coarse_prep_bytes(int n_lists, int dim) {
  return c64_offset(n_lists, dim) + (size_t)n_lists * dim * sizeof(double);
}

// CT = float: the index's centroids; CT = double: the f64 centroids of a Lloyd
// iteration (the images are built from their f32 roundings, 2^-24 relative,
// far inside the guard band; the exact re-scoring reads the f64 values).
template <typename CT>
static int coarse_prepare_t(const CT* centroids, int n_lists, int dim, void* prep, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int DP = pad_dp(dim);
  const int nT = (n_lists + tile_n(DP) - 1) / tile_n(DP);
  IVFTQ_CHECK_CUDA(cudaMemsetAsync(prep, 0, kHeader, s));
  prep_stats_kernel<CT><<<(n_lists + 7) / 8, 256, 0, s>>>(centroids, n_lists, dim,
                                                             (PrepHeader*)prep);
  if (int e = check_launch("coarse_prep_stats")) return e;
  const int64_t work = (int64_t)nT * tile_n(DP) * (DP / 8);
  prep_split_kernel<CT><<<(unsigned)((work + 255) / 256), 256, 0, s>>>(
      centroids, n_lists, dim, DP, nT, (PrepHeader*)prep, (unsigned char*)prep + kHeader);
  if (int e = check_launch("coarse_prep_split")) return e;
  const int64_t nc = (int64_t)n_lists * dim;
  prep_c64_kernel<CT><<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(
      centroids, nc, (double*)((unsigned char*)prep + c64_offset(n_lists, dim)));
  return check_launch("coarse_prep_c64");
}

extern "C" int ivftq_coarse_prepare(const float* centroids, int n_lists, int dim, void* prep,
                                    void* stream) {
  return coarse_prepare_t<float>(centroids, n_lists, dim, prep, stream);
}

// S' (optional) and per-row best four (optional) for rows X[0..n)
static int coarse_gemm(const double* X, int64_t n, int dim, int L, const void* prep, float* S,
                       float* top_v, int32_t* top_i, cudaStream_t s,
                       uint32_t* xsplit = nullptr) {
  uint32_t* xh = nullptr;
  uint32_t* xl = nullptr;
  if (xsplit) {
    const int DPx = pad_dp(dim);
    xh = xsplit;
    xl = xsplit + (size_t)n * (DPx / 2);
    const int64_t words = n * (DPx / 2);
    x_split_kernel<<<(unsigned)((words + 255) / 256), 256, 0, s>>>(X, n, dim, DPx, xh, xl);
    if (int e = check_launch("x_split")) return e;
  }
  const int DP = pad_dp(dim);
  const int nT = (L + tile_n(DP) - 1) / tile_n(DP);
  const size_t smem = 3 * tile_bytes(DP) + 1024;
  if (int e = smem_opt_in_dev((const void*)coarse_tc_kernel, 3 * tile_bytes(128) + 1024))
    return e;
  const int n_sms = device_sm_count();
  const int64_t n_rt = (n + kM - 1) / kM;
  const int64_t units = n_rt * nT;
  const unsigned grid = top_v ? (unsigned)n_rt : (unsigned)(units < n_sms ? units : n_sms);
  coarse_tc_kernel<<<grid, kThreads, smem, s>>>(
      X, n, dim, DP, L, nT, (const unsigned char*)prep, S, top_v, top_i, xh, xl);
  return check_launch("coarse_tc");
}

// Rotation on the coarse-scoring kernel (index.py:256, rotation.py:40): the d
// rows of R play the centroids, the pre-split unit residual rows the queries,
// S' = A . R^T in f32 (n x d). Used by the tensor-core encoder (encode.cu).
namespace ivftq {
int rotate_tc(const uint32_t* xh, const uint32_t* xl, int64_t n, int dim, const double* R,
              float* U, void* prep, cudaStream_t s) {
  if (int e = ::coarse_prepare_t<double>(R, dim, dim, prep, (void*)s)) return e;
  const int DP = ctc::pad_dp(dim);
  const int nT = (dim + ctc::tile_n(DP) - 1) / ctc::tile_n(DP);
  const size_t smem = 3 * ctc::tile_bytes(DP) + 1024;
  if (int e = smem_opt_in_dev((const void*)ctc::coarse_tc_kernel, 3 * ctc::tile_bytes(128) + 1024))
    return e;
  const int n_sms = device_sm_count();
  const int64_t units = ((n + ctc::kM - 1) / ctc::kM) * nT;
  const unsigned grid = (unsigned)(units < n_sms ? units : n_sms);
  ctc::coarse_tc_kernel<<<grid, ctc::kThreads, smem, s>>>(
      nullptr, n, dim, DP, dim, nT, (const unsigned char*)prep, U, nullptr, nullptr, xh, xl);
  return check_launch("rotate_tc");
}
}  // namespace ivftq

extern "C" size_t ivftq_assign_tc_scratch_bytes(int64_t n, int n_lists, int dim) {
  // prep | top_v (n*4 f32) | top_i (n*4 i32) | ex (n*4 f64) | full list (n i32) | count
  // | pre-split A rows (n * DP * 4)
  return ivftq_coarse_prep_bytes(n_lists, dim) + 256 + (size_t)n * kTopA * 16 + (size_t)n * 4 +
         1024 + (size_t)n * pad_dp(dim) * 4 + 256;
}

template <typename CT>
static int assign_tc_t(const double* xn, const CT* centroids, int64_t n, int n_lists, int dim,
                       int32_t* list_out, void* scratch, size_t scratch_bytes, void* stream) {
  if (scratch_bytes < ivftq_assign_tc_scratch_bytes(n, n_lists, dim)) {
    set_error("assign_tc: scratch too small");
    return IVFTQ_ERR_SCRATCH;
  }
  cudaStream_t s = (cudaStream_t)stream;
  unsigned char* prep = (unsigned char*)scratch;
  const size_t pb = (ivftq_coarse_prep_bytes(n_lists, dim) + 255) & ~(size_t)255;
  double* ex = (double*)(prep + pb);
  float* tv = (float*)(ex + n * kTopA);
  int32_t* ti = (int32_t*)(tv + n * kTopA);
  int32_t* full = ti + n * kTopA;
  int32_t* nfull = full + n;
  uint32_t* xsplit = (uint32_t*)(((uintptr_t)(nfull + 1) + 255) & ~(uintptr_t)255);
  IVFTQ_CHECK_CUDA(cudaMemsetAsync(nfull, 0, sizeof(int32_t), s));
  if (int e = coarse_prepare_t<CT>(centroids, n_lists, dim, prep, stream)) return e;
  if (int e = coarse_gemm(xn, n, dim, n_lists, prep, nullptr, tv, ti, s, xsplit)) return e;
  const double* c64 = (const double*)(prep + c64_offset(n_lists, dim));
  assign_exact_kernel<<<(unsigned)((n * kTopA + 127) / 128), 128, 0, s>>>(xn, c64, n, dim,
                                                                          prep, tv, ti, ex);
  if (int e = check_launch("assign_exact")) return e;
  assign_pick_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, prep, tv, ti, ex, list_out,
                                                                 full, nfull);
  if (int e = check_launch("assign_pick")) return e;
  assign_full_kernel<<<2 * device_sm_count(), kFullThreads, sizeof(double) * dim, s>>>(
      xn, c64, n_lists, dim, full, nfull, list_out);
  return check_launch("assign_full");
}

extern "C" int ivftq_assign_tc(const double* xn, const float* centroids, int64_t n, int n_lists,
                               int dim, int32_t* list_out, void* scratch, size_t scratch_bytes,
                               void* stream) {
  if (n == 0) return 0;
  if (!ivftq_coarse_tc_supported(dim, n_lists))
    return ivftq_assign(xn, centroids, n, n_lists, dim, list_out, stream);
  return assign_tc_t<float>(xn, centroids, n, n_lists, dim, list_out, scratch, scratch_bytes,
                            stream);
}

// The Lloyd-step assignment of the GPU k-means (partition.py:149-150): f64
// centroids, same tensor-core pass + exact f64 decision, ties to the lower list.
extern "C" int ivftq_assign_tc64(const double* xn, const double* centroids, int64_t n,
                                 int n_lists, int dim, int32_t* list_out, void* scratch,
                                 size_t scratch_bytes, void* stream) {
  if (n == 0) return 0;
  if (!ivftq_coarse_tc_supported(dim, n_lists)) {
    set_error("assign_tc64: shape not supported (dim %d)", dim);
    return IVFTQ_ERR_UNSUPPORTED;
  }
  return assign_tc_t<double>(xn, centroids, n, n_lists, dim, list_out, scratch, scratch_bytes,
                             stream);
}

extern "C" size_t ivftq_probe_tc_scratch_bytes(int64_t nq, int n_lists, int dim) {
  // prep | S' (nq*L f32) | cand (nq*cap i32) | ex (nq*cap f64) | cnt (nq i32)
  return ivftq_coarse_prep_bytes(n_lists, dim) + 256 + (size_t)nq * n_lists * 4 + 256 +
         (size_t)nq * kCandCap * 12 + (size_t)nq * 4 + 1024 + (size_t)nq * pad_dp(dim) * 4 + 256;
}

// Tensor-core probes; returns IVFTQ_ERR_UNSUPPORTED when the caller should use f64.
int probe_tc(const double* qn, const float* centroids, int64_t nq, int n_lists, int dim,
             int n_p, int32_t* probe_out, double* coarse_out, void* scratch,
             size_t scratch_bytes, cudaStream_t s, const void* prepared) {
  if (!ivftq_coarse_tc_supported(dim, n_lists) || n_p > 128) return IVFTQ_ERR_UNSUPPORTED;
  if (scratch_bytes < ivftq_probe_tc_scratch_bytes(nq, n_lists, dim)) return IVFTQ_ERR_UNSUPPORTED;
  unsigned char* prep = (unsigned char*)scratch;
  const size_t pb = (ivftq_coarse_prep_bytes(n_lists, dim) + 255) & ~(size_t)255;
  double* ex = (double*)(prep + pb);
  float* S = (float*)(ex + nq * kCandCap);
  int32_t* cand = (int32_t*)(S + (((size_t)nq * n_lists + 63) & ~(size_t)63));
  int32_t* cnt = cand + nq * kCandCap;
  uint32_t* xsplit = (uint32_t*)(((uintptr_t)(cnt + nq) + 255) & ~(uintptr_t)255);
  if (prepared) {  // operand images made once per centroid set by the caller
    prep = (unsigned char*)prepared;
  } else if (int e = ivftq_coarse_prepare(centroids, n_lists, dim, prep, s)) {
    return e;
  }
  if (int e = coarse_gemm(qn, nq, dim, n_lists, prep, S, nullptr, nullptr, s, xsplit)) return e;
  const unsigned blocks = (unsigned)((nq + 7) / 8);
  const double* c64 = (const double*)(prep + c64_offset(n_lists, dim));
  const bool fused = n_lists <= kSelRowCap;
  if (fused) {
    const size_t sm = sel_smem_bytes(n_lists, dim);
    if (int e = smem_opt_in_dev((const void*)probe_select_kernel, sm)) return e;
    probe_select_kernel<<<(unsigned)nq, kSelThreads, sm, s>>>(S, qn, c64, nq, n_lists, dim, n_p,
                                                             prep, cnt, probe_out, coarse_out);
    if (int e = check_launch("probe_select")) return e;
  } else {
    probe_band_kernel<<<blocks, 256, 0, s>>>(S, nq, n_lists, n_p, prep, cand, cnt);
    if (int e = check_launch("probe_band")) return e;
    probe_exact_kernel<<<(unsigned)nq, 128, 0, s>>>(qn, c64, nq, dim, cand, cnt, ex);
    if (int e = check_launch("probe_exact")) return e;
  }
  if (n_p <= 32)
    probe_pick_kernel<1><<<blocks, 256, 0, s>>>(qn, c64, nq, n_lists, dim, n_p, cand, cnt,
                                                ex, probe_out, coarse_out, fused);
  else if (n_p <= 64)
    probe_pick_kernel<2><<<blocks, 256, 0, s>>>(qn, c64, nq, n_lists, dim, n_p, cand, cnt,
                                                ex, probe_out, coarse_out, fused);
  else
    probe_pick_kernel<4><<<blocks, 256, 0, s>>>(qn, c64, nq, n_lists, dim, n_p, cand, cnt,
                                                ex, probe_out, coarse_out, fused);
  return check_launch("probe_pick");
}
