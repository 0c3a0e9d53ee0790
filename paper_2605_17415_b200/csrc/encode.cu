// Ingest-side kernels: normalisation, residual + binary16 norm, Lloyd-Max
// quantize + bit-pack, list-store append / relayout / export.
//
// Reference: IvfTqIndex._encode_batch (index.py:231-267), add_batch
// (index.py:286-310), ScalarQuantizer.quantize (lloydmax.py:129-144).
// Every f64 operation that the reference performs elementwise (normalise,
// subtract, divide, f16 rounding, boundary compares) is reproduced with the
// same IEEE operations in the same order, so those stages are bit-exact; only
// the GEMMs (assign, rotate) differ in summation order from OpenBLAS.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace ivftq {

constexpr int kRowTile = 32;     // rows staged per block
constexpr int kRowThreads = 128;

// 16 rows per block: one lane group of 8 per row in a single pass, and 4x the
// blocks of the 32-row tile for a 10k-query batch (latency-bound otherwise)
constexpr int kNormRows = 16;

template <typename T>
__global__ void __launch_bounds__(kRowThreads)
normalize_kernel(const T* __restrict__ x, int64_t n, int d, double* __restrict__ xn,
                 unsigned long long* bad) {
  extern __shared__ double sm[];  // kNormRows * (d+1)
  __shared__ double nrm[kNormRows];
  const int ld = d + 1;
  int64_t row0 = (int64_t)blockIdx.x * kNormRows;
  int rows = (int)(n - row0 < kNormRows ? n - row0 : kNormRows);
  for (int i = threadIdx.x; i < rows * d; i += blockDim.x) {
    int r = i / d, c = i - r * d;
    sm[r * ld + c] = (double)x[(row0 + r) * d + c];
  }
  __syncthreads();
  // 8 lanes per row (whole lane groups iterate together: rows is uniform)
  for (int r = threadIdx.x >> 3; r < ((rows + 3) & ~3); r += kRowThreads / 8) {
    const int rr = r < rows ? r : 0;
    const double s = pw_sumsq_lane8(sm + rr * ld, d);
    if ((threadIdx.x & 7) == 0 && r < rows) {
      const double nr = __dsqrt_rn(s);
      nrm[r] = nr;
      if (!(nr >= 1e-12) && !(nr != nr)) atomicMin(bad, (unsigned long long)(row0 + r));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < rows * d; i += blockDim.x) {
    int r = i / d, c = i - r * d;
    xn[(row0 + r) * d + c] = __ddiv_rn(sm[r * ld + c], nrm[r]);
  }
}

// Rows of 8 <= d <= 128 without shared-memory staging: eight lanes per row,
// lane j owns numpy's pairwise accumulator r_j (elements j, j+8, ...: 64-byte
// segments per load step, all of a lane's loads in flight at once), the three
// xor shuffles form ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and the d % 8 tail is
// added in order, exactly as pw_sumsq_lane8 / numpy do.
constexpr int kDirectMax = 128;
template <typename T>
__global__ void __launch_bounds__(256)
normalize_direct_kernel(const T* __restrict__ x, int64_t n, int d, double* __restrict__ xn,
                        unsigned long long* bad) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gid >> 3;
  const int j = (int)(gid & 7);
  const bool live = row < n;
  const T* xr = x + (live ? row : n - 1) * (int64_t)d;
  const int lim = d - (d % 8), cnt = lim >> 3;
  double v[kDirectMax / 8];
#pragma unroll
  for (int i = 0; i < kDirectMax / 8; ++i) v[i] = i < cnt ? (double)xr[j + 8 * i] : 0.0;
  double r = sq(v[0]);
#pragma unroll
  for (int i = 1; i < kDirectMax / 8; ++i)
    if (i < cnt) r = add(r, sq(v[i]));
  const unsigned gm = 0xffu << (threadIdx.x & 24);
  r = add(r, __shfl_xor_sync(gm, r, 1));
  r = add(r, __shfl_xor_sync(gm, r, 2));
  r = add(r, __shfl_xor_sync(gm, r, 4));
  double tail = lim + j < d ? (double)xr[lim + j] : 0.0;
  for (int i = lim; i < d; ++i) r = add(r, sq(__shfl_sync(gm, tail, (threadIdx.x & 24) + i - lim)));
  const double nr = __dsqrt_rn(r);
  if (!live) return;
  if (j == 0 && !(nr >= 1e-12) && !(nr != nr)) atomicMin(bad, (unsigned long long)row);
  double* out = xn + row * (int64_t)d;
#pragma unroll
  for (int i = 0; i < kDirectMax / 8; ++i)
    if (i < cnt) out[j + 8 * i] = __ddiv_rn(v[i], nr);
  if (lim + j < d) out[lim + j] = __ddiv_rn(tail, nr);
}

__global__ void init_i64(int64_t* p, int64_t v) { *p = v; }

__global__ void __launch_bounds__(kRowThreads)
residual_kernel(const double* __restrict__ xn, const float* __restrict__ cent,
                const int32_t* __restrict__ lids, int64_t n, int d, int flat,
                double* __restrict__ out, uint16_t* __restrict__ norm_out) {
  extern __shared__ double sm[];
  const int ld = d + 1;
  int64_t row0 = (int64_t)blockIdx.x * kRowTile;
  int rows = (int)(n - row0 < kRowTile ? n - row0 : kRowTile);
  for (int i = threadIdx.x; i < rows * d; i += blockDim.x) {
    int r = i / d, c = i - r * d;
    double v = xn[(row0 + r) * d + c];
    if (!flat) v = __dsub_rn(v, (double)cent[(int64_t)lids[row0 + r] * d + c]);
    sm[r * ld + c] = v;
    out[(row0 + r) * d + c] = v;
  }
  __syncthreads();
  for (int r = threadIdx.x >> 3; r < ((rows + 3) & ~3); r += kRowThreads / 8) {
    const int rr = r < rows ? r : 0;
    const double s = pw_sumsq_lane8(sm + rr * ld, d);
    if ((threadIdx.x & 7) == 0 && r < rows) norm_out[row0 + r] = d2h_bits(__dsqrt_rn(s));
  }
}

// bin = #interior boundaries <= v (upper-bin on ties), sign = v >= centroid.
__device__ __forceinline__ uint32_t quant_field(double v, const double* bnd,
                                                const double* qc, int levels) {
  int lo = 0, hi = levels - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (bnd[mid] <= v) lo = mid; else hi = mid - 1;
  }
  return ((uint32_t)lo << 1) | (v >= qc[lo] ? 1u : 0u);
}

__global__ void __launch_bounds__(kRowThreads)
quantize_pack_kernel(const double* __restrict__ rot, const uint16_t* __restrict__ norms,
                     int64_t n, int d, int bits, int use_sign,
                     const double* __restrict__ boundaries, const double* __restrict__ qcent,
                     uint32_t* __restrict__ words) {
  extern __shared__ double sm[];
  __shared__ double nrm[kRowTile];
  __shared__ double bnd[257];
  __shared__ double qc[256];
  const int levels = 1 << bits;
  const int fb = field_bits(bits, use_sign), fpw = fields_per_word(fb);
  const int W = words_per_vec(d, fb);
  const int ld = d + 1;
  for (int i = threadIdx.x; i <= levels; i += blockDim.x) bnd[i] = boundaries[i];
  for (int i = threadIdx.x; i < levels; i += blockDim.x) qc[i] = qcent[i];
  int64_t row0 = (int64_t)blockIdx.x * kRowTile;
  int rows = (int)(n - row0 < kRowTile ? n - row0 : kRowTile);
  for (int i = threadIdx.x; i < rows * d; i += blockDim.x) {
    int r = i / d, c = i - r * d;
    sm[r * ld + c] = rot[(row0 + r) * d + c];
  }
  __syncthreads();
  for (int r = threadIdx.x >> 3; r < ((rows + 3) & ~3); r += kRowThreads / 8) {
    const int rr = r < rows ? r : 0;
    const double s = pw_sumsq_lane8(sm + rr * ld, d);
    if ((threadIdx.x & 7) == 0 && r < rows) nrm[r] = __dsqrt_rn(s);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < rows * W; i += blockDim.x) {
    int r = i / W, w = i - r * W;
    uint32_t word = 0;
    if (norms[row0 + r] != 0) {  // binary16 +0 => dead row, codes stay 0
      const double* rp = sm + r * ld;
      double nr = nrm[r];
      for (int f = 0; f < fpw; ++f) {
        int j = w * fpw + f;
        if (j >= d) break;
        double u = __ddiv_rn(rp[j], nr);
        word |= quant_field(u, bnd, qc, levels) << (fb * f);
      }
    }
    words[(row0 + r) * W + w] = word;
  }
}

// ---- tensor-core encoder (index.py:247-262 with the rotation on tcgen05) -------
// (1) unit residual rows, split for the tensor cores: r = xn - c_l in f64 as the
// reference computes it, ||r|| in numpy's pairwise order -> binary16 (both
// bit-exact), then a = r / ||r|| scaled by 2^14 and split into fp16 hi + lo,
// two coordinates per word along k, zero-padded to DP (coarse_tc.cu's
// A-operand row format). No f64 intermediate goes back to HBM.
__device__ __forceinline__ void split16e(float x, uint16_t& hi, uint16_t& lo) {
  const __half h = __float2half_rn(x);
  hi = __half_as_ushort(h);
  lo = __half_as_ushort(__float2half_rn(x - __half2float(h)));
}

constexpr int kSplitThreads = 256;
__global__ void __launch_bounds__(kSplitThreads)
resid_split_kernel(const double* __restrict__ xn, const float* __restrict__ cent,
                   const int32_t* __restrict__ lids, int64_t n, int d, int DP, int flat,
                   uint16_t* __restrict__ norm_out, uint32_t* __restrict__ hi,
                   uint32_t* __restrict__ lo) {
  extern __shared__ double sm[];
  __shared__ double nrm[kRowTile];
  const int ld = d + 1;
  int64_t row0 = (int64_t)blockIdx.x * kRowTile;
  int rows = (int)(n - row0 < kRowTile ? n - row0 : kRowTile);
  for (int i = threadIdx.x; i < rows * d; i += blockDim.x) {
    int r = i / d, c = i - r * d;
    double v = xn[(row0 + r) * d + c];
    if (!flat) v = __dsub_rn(v, (double)cent[(int64_t)lids[row0 + r] * d + c]);
    sm[r * ld + c] = v;
  }
  __syncthreads();
  for (int r = threadIdx.x >> 3; r < ((rows + 3) & ~3); r += kSplitThreads / 8) {
    const int rr = r < rows ? r : 0;
    const double s = pw_sumsq_lane8(sm + rr * ld, d);
    if ((threadIdx.x & 7) == 0 && r < rows) {
      const double q = __dsqrt_rn(s);
      nrm[r] = q;
      norm_out[row0 + r] = d2h_bits(q);
    }
  }
  __syncthreads();
  const int hw = DP / 2;
  for (int i = threadIdx.x; i < rows * hw; i += blockDim.x) {
    const int r = i / hw, k = (i - r * hw) * 2;
    const double q = nrm[r];
    const double* rp = sm + r * ld;
    uint16_t h0, l0, h1, l1;
    split16e(k < d && q > 0.0 ? (float)(__ddiv_rn(rp[k], q) * 16384.0) : 0.f, h0, l0);
    split16e(k + 1 < d && q > 0.0 ? (float)(__ddiv_rn(rp[k + 1], q) * 16384.0) : 0.f, h1, l1);
    hi[(row0 + r) * hw + (k >> 1)] = h0 | ((uint32_t)h1 << 16);
    lo[(row0 + r) * hw + (k >> 1)] = l0 | ((uint32_t)l1 << 16);
  }
}

// The same step for 8 <= d <= 128 without shared-memory staging (eight lanes
// per row as in normalize_direct_kernel); a lane pair (j even, j + 1) packs
// its two coordinates into one operand word.
__global__ void __launch_bounds__(256)
resid_split_direct_kernel(const double* __restrict__ xn, const float* __restrict__ cent,
                          const int32_t* __restrict__ lids, int64_t n, int d, int DP, int flat,
                          uint16_t* __restrict__ norm_out, uint32_t* __restrict__ hi,
                          uint32_t* __restrict__ lo) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = gid >> 3;
  const int j = (int)(gid & 7);
  const bool live = row < n;
  const int64_t rr = live ? row : n - 1;
  const double* xr = xn + rr * (int64_t)d;
  const float* cr = flat ? nullptr : cent + (int64_t)lids[rr] * d;
  const int lim = d - (d % 8), cnt = lim >> 3;
  double v[kDirectMax / 8];
#pragma unroll
  for (int i = 0; i < kDirectMax / 8; ++i) {
    double t = 0.0;
    if (i < cnt) {
      t = xr[j + 8 * i];
      if (cr) t = __dsub_rn(t, (double)cr[j + 8 * i]);
    }
    v[i] = t;
  }
  double tail = 0.0;
  if (lim + j < d) {
    tail = xr[lim + j];
    if (cr) tail = __dsub_rn(tail, (double)cr[lim + j]);
  }
  double r = sq(v[0]);
#pragma unroll
  for (int i = 1; i < kDirectMax / 8; ++i)
    if (i < cnt) r = add(r, sq(v[i]));
  const unsigned gm = 0xffu << (threadIdx.x & 24);
  r = add(r, __shfl_xor_sync(gm, r, 1));
  r = add(r, __shfl_xor_sync(gm, r, 2));
  r = add(r, __shfl_xor_sync(gm, r, 4));
  for (int i = lim; i < d; ++i) r = add(r, sq(__shfl_sync(gm, tail, (threadIdx.x & 24) + i - lim)));
  const double q = __dsqrt_rn(r);
  if (live && j == 0) norm_out[row] = d2h_bits(q);
  // operand words: coordinates k = j + 8 i for k < DP (zeros past d)
  const int hw = DP / 2;
#pragma unroll
  for (int i = 0; i < (kDirectMax + 31) / 32 * 4; ++i) {
    const int k = j + 8 * i;
    if (k - j >= DP) break;  // uniform over the group
    // k < lim: this lane's i-th element; k = lim + j < d: its tail element
    const double val = k < lim ? v[i < kDirectMax / 8 ? i : 0] : (k < d ? tail : 0.0);
    uint16_t h, l;
    split16e(k < d && q > 0.0 ? (float)(__ddiv_rn(val, q) * 16384.0) : 0.f, h, l);
    const uint32_t ph = __shfl_xor_sync(gm, (uint32_t)h, 1), pl = __shfl_xor_sync(gm, (uint32_t)l, 1);
    if (live) {
      if ((j & 1) == 0) hi[row * hw + (k >> 1)] = h | (ph << 16);
      else lo[row * hw + (k >> 1)] = pl | ((uint32_t)l << 16);
    }
  }
}

// (3) Lloyd-Max bins + signs from the tensor-core unit coordinates u' (f32),
// packed. A row with any coordinate within `eps` of a decision threshold (a
// bin boundary or its bin's half-bin centroid) is listed for the exact pass:
// |u' - u| < eps, so every other row's fields equal the f64 path's.
__global__ void __launch_bounds__(256)
quantize_guard_kernel(const float* __restrict__ U, const uint16_t* __restrict__ norms, int64_t n,
                      int d, int bits, int use_sign, const double* __restrict__ boundaries,
                      const double* __restrict__ qcent, double eps, uint32_t* __restrict__ words,
                      int32_t* __restrict__ flag, int32_t* __restrict__ list,
                      int32_t* __restrict__ count) {
  __shared__ double bnd[257];
  __shared__ double qc[256];
  const int levels = 1 << bits;
  const int fb = field_bits(bits, use_sign), fpw = fields_per_word(fb);
  const int W = words_per_vec(d, fb);
  for (int i = threadIdx.x; i <= levels; i += blockDim.x) bnd[i] = boundaries[i];
  for (int i = threadIdx.x; i < levels; i += blockDim.x) qc[i] = qcent[i];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * W) return;
  const int64_t r = i / W;
  const int w = (int)(i - r * W);
  uint32_t word = 0;
  bool amb = false;
  if (norms[r] != 0) {  // binary16 +0 => dead row, codes stay 0
    const float* up = U + r * d;
    for (int f = 0; f < fpw; ++f) {
      const int j = w * fpw + f;
      if (j >= d) break;
      const double u = (double)up[j];
      const uint32_t c = quant_field(u, bnd, qc, levels);
      const int b = (int)(c >> 1);
      word |= c << (fb * f);
      amb |= fabs(u - qc[b]) <= eps;
      if (b > 0) amb |= u - bnd[b] <= eps;
      if (b + 1 < levels) amb |= bnd[b + 1] - u <= eps;
    }
  }
  words[i] = word;
  if (amb && atomicExch(&flag[r], 1) == 0) list[atomicAdd(count, 1)] = (int32_t)r;
}

// (4) exact f64 re-encode of the listed rows, kFixRows at a time per block:
// r = xn - c, rot = r.R^T as a sequential FMA chain per coordinate (each R^T
// element loaded once for the kFixRows rows), u = rot / ||rot|| (numpy
// pairwise norm), then the same quant_field as quantize_pack_kernel.
constexpr int kFixRows = 8;
__global__ void __launch_bounds__(128)
encode_fixup_kernel(const double* __restrict__ xn, const float* __restrict__ cent,
                    const int32_t* __restrict__ lids, int d, int flat,
                    const double* __restrict__ RT, int bits, int use_sign,
                    const double* __restrict__ boundaries, const double* __restrict__ qcent,
                    const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                    uint32_t* __restrict__ words) {
  extern __shared__ double sm[];  // r[kFixRows][d] | rot[kFixRows][d]
  __shared__ double bnd[257];
  __shared__ double qc[256];
  __shared__ double nrm[kFixRows];
  __shared__ int64_t rid[kFixRows];
  double* rs = sm;
  double* rot = sm + (size_t)kFixRows * d;
  const int levels = 1 << bits;
  const int fb = field_bits(bits, use_sign), fpw = fields_per_word(fb);
  const int W = words_per_vec(d, fb);
  for (int i = threadIdx.x; i <= levels; i += blockDim.x) bnd[i] = boundaries[i];
  for (int i = threadIdx.x; i < levels; i += blockDim.x) qc[i] = qcent[i];
  const int total = *count;
  for (int it = blockIdx.x * kFixRows; it < total; it += gridDim.x * kFixRows) {
    const int nr = total - it < kFixRows ? total - it : kFixRows;
    __syncthreads();
    if (threadIdx.x < kFixRows) rid[threadIdx.x] = threadIdx.x < nr ? list[it + threadIdx.x] : -1;
    __syncthreads();
    for (int i = threadIdx.x; i < kFixRows * d; i += blockDim.x) {
      const int x = i / d, k = i - x * d;
      double v = 0.0;
      if (x < nr) {
        const int64_t r = rid[x];
        v = xn[r * d + k];
        if (!flat) v = __dsub_rn(v, (double)cent[(int64_t)lids[r] * d + k]);
      }
      rs[i] = v;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      double acc[kFixRows];
#pragma unroll
      for (int x = 0; x < kFixRows; ++x) acc[x] = 0.0;
      for (int k = 0; k < d; ++k) {
        const double rv = RT[(int64_t)k * d + j];
#pragma unroll
        for (int x = 0; x < kFixRows; ++x) acc[x] = __fma_rn(rs[x * d + k], rv, acc[x]);
      }
#pragma unroll
      for (int x = 0; x < kFixRows; ++x) rot[x * d + j] = acc[x];
    }
    __syncthreads();
    if (threadIdx.x < 8 * kFixRows) {  // one lane group of 8 per row
      const int x = threadIdx.x >> 3;
      const double s = pw_sumsq_lane8(rot + x * d, d);
      if ((threadIdx.x & 7) == 0) nrm[x] = __dsqrt_rn(s);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nr * W; i += blockDim.x) {
      const int x = i / W, w = i - x * W;
      const double q = nrm[x];
      uint32_t word = 0;
      for (int f = 0; f < fpw; ++f) {
        const int j = w * fpw + f;
        if (j >= d) break;
        word |= quant_field(__ddiv_rn(rot[x * d + j], q), bnd, qc, levels) << (fb * f);
      }
      words[rid[x] * W + w] = word;
    }
  }
}

__global__ void transpose_kernel(const double* __restrict__ R, int d, double* __restrict__ RT) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d * d) RT[(i % d) * d + i / d] = R[i];
}

__global__ void pack_codes_kernel(const uint8_t* __restrict__ bins,
                                  const uint8_t* __restrict__ signs, int64_t n, int d,
                                  int bits, int use_sign, uint32_t* __restrict__ words) {
  const int fb = field_bits(bits, use_sign), fpw = fields_per_word(fb);
  const int W = words_per_vec(d, fb);
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * W) return;
  int64_t r = i / W;
  int w = (int)(i - r * W);
  uint32_t word = 0;
  for (int f = 0; f < fpw; ++f) {
    int j = w * fpw + f;
    if (j >= d) break;
    uint32_t c = ((uint32_t)bins[r * d + j] << 1) | (signs[r * d + j] & 1u);
    word |= c << (fb * f);
  }
  words[i] = word;
}

// Both kernels skip a row whose list id lies outside [0, n_lists): a corrupt
// id from a direct C-ABI caller never writes outside the store (the Python
// layer rejects such ids before any device work, storage.py:load_index).
__global__ void histogram_kernel(const int32_t* __restrict__ lids, int64_t n, int n_lists,
                                 int32_t* __restrict__ counts) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int l = lids[i];
    if (l >= 0 && l < n_lists) atomicAdd(&counts[l], 1);
  }
}

__global__ void append_kernel(ivftq_store s, const uint32_t* __restrict__ words,
                              const uint16_t* __restrict__ norms,
                              const int32_t* __restrict__ lids, int64_t n, int64_t first_id,
                              int32_t* __restrict__ cursor, int64_t* __restrict__ slot_of) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int W = s.words_per_vec;
  int l = lids[i];
  if (l < 0 || l >= s.n_lists) return;
  int r = atomicAdd(&cursor[l], 1);
  int64_t slot = s.list_offset[l] + s.list_size[l] + r;
  int64_t blk = slot >> 5;
  int lane = (int)(slot & 31);
  uint32_t* dst = s.codes + blk * W * 32 + lane;
  for (int w = 0; w < W; ++w) dst[w * 32] = words[i * W + w];
  s.norms[slot] = norms[i];
  s.ids[slot] = (int32_t)(first_id + i);
  slot_of[first_id + i] = slot;
}

__global__ void relayout_kernel(ivftq_store src, ivftq_store dst, int64_t* slot_of) {
  int l = blockIdx.x;
  int size = src.list_size[l];
  if (size == 0) return;
  const int W = src.words_per_vec;
  int64_t so = src.list_offset[l], doff = dst.list_offset[l];
  int nblk = (size + 31) >> 5;
  const uint32_t* cs = src.codes + (so >> 5) * W * 32;
  uint32_t* cd = dst.codes + (doff >> 5) * W * 32;
  int64_t nw = (int64_t)nblk * W * 32;
  for (int64_t i = threadIdx.x; i < nw; i += blockDim.x) cd[i] = cs[i];
  for (int i = threadIdx.x; i < nblk * 32; i += blockDim.x) {
    dst.norms[doff + i] = src.norms[so + i];
    int id = src.ids[so + i];
    dst.ids[doff + i] = id;
    if (i < size && id >= 0) slot_of[id] = doff + i;
  }
}

__global__ void export_codes_kernel(ivftq_store s, const int64_t* __restrict__ slot_of,
                                    int64_t first, int64_t n, uint8_t* __restrict__ bins,
                                    uint8_t* __restrict__ signs) {
  const int W = s.words_per_vec, fb = s.field_bits, fpw = s.fields_per_word, d = s.dim;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * W) return;
  int64_t r = i / W;
  int w = (int)(i - r * W);
  int64_t slot = slot_of[first + r];
  uint32_t word = s.codes[((slot >> 5) * W + w) * 32 + (slot & 31)];
  uint32_t mask = (1u << fb) - 1u;
  for (int f = 0; f < fpw; ++f) {
    int j = w * fpw + f;
    if (j >= d) break;
    uint32_t c = (word >> (fb * f)) & mask;
    bins[r * d + j] = (uint8_t)(c >> 1);
    if (signs) signs[r * d + j] = (uint8_t)(c & 1u);
  }
}

__global__ void xor_codes_kernel(ivftq_store s, const int64_t* __restrict__ slot_of,
                                 int64_t n, const uint8_t* __restrict__ mask, int which,
                                 int flip) {
  const int W = s.words_per_vec, fb = s.field_bits, fpw = s.fields_per_word, d = s.dim;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * W) return;
  int64_t r = i / W;
  int w = (int)(i - r * W);
  int64_t slot = slot_of[r];
  uint32_t* p = s.codes + ((slot >> 5) * W + w) * 32 + (slot & 31);
  uint32_t x = 0;
  for (int f = 0; f < fpw; ++f) {
    int j = w * fpw + f;
    if (j >= d) break;
    if (mask[r * d + j]) {
      uint32_t v = (which == 1) ? 1u : (uint32_t)flip << 1;
      x |= v << (fb * f);
    }
  }
  *p ^= x;
}

}  // namespace ivftq

using namespace ivftq;

static inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

static int row_smem(int d) { return kRowTile * (d + 1) * (int)sizeof(double); }

static int set_row_smem_bytes(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)bytes);
    if (e != cudaSuccess) {
      set_error("shared memory request %zu B rejected: %s", bytes, cudaGetErrorString(e));
      return IVFTQ_ERR_UNSUPPORTED;
    }
  }
  return 0;
}

static int set_row_smem(const void* fn, int d) {
  int bytes = row_smem(d);
  if (bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) {
      set_error("dim %d too large for row kernels: %s", d, cudaGetErrorString(e));
      return IVFTQ_ERR_UNSUPPORTED;
    }
  }
  return 0;
}

extern "C" int ivftq_normalize_rows(const void* x, int x_dtype, int64_t n, int dim,
                                    double* xn, int64_t* bad_row, void* stream) {
  if (n < 0 || dim < 1 || (x_dtype != IVFTQ_F32 && x_dtype != IVFTQ_F64)) {
    set_error("normalize_rows: bad arguments");
    return IVFTQ_ERR_ARG;
  }
  init_i64<<<1, 1, 0, S(stream)>>>(bad_row, n);
  if (int e = check_launch("init_bad_row")) return e;
  if (n == 0) return 0;
  if (dim >= 8 && dim <= kDirectMax && !getenv("IVFTQ_ROWS_STAGED")) {
    const unsigned g = (unsigned)((n * 8 + 255) / 256);
    if (x_dtype == IVFTQ_F32)
      normalize_direct_kernel<float><<<g, 256, 0, S(stream)>>>((const float*)x, n, dim, xn,
                                                                (unsigned long long*)bad_row);
    else
      normalize_direct_kernel<double><<<g, 256, 0, S(stream)>>>((const double*)x, n, dim, xn,
                                                                 (unsigned long long*)bad_row);
    return check_launch("normalize_rows");
  }
  int grid = (int)((n + kNormRows - 1) / kNormRows);
  const size_t nsm = (size_t)kNormRows * (dim + 1) * sizeof(double);
  if (x_dtype == IVFTQ_F32) {
    if (int e = set_row_smem_bytes((const void*)normalize_kernel<float>, nsm)) return e;
    normalize_kernel<float><<<grid, kRowThreads, nsm, S(stream)>>>(
        (const float*)x, n, dim, xn, (unsigned long long*)bad_row);
  } else {
    if (int e = set_row_smem_bytes((const void*)normalize_kernel<double>, nsm)) return e;
    normalize_kernel<double><<<grid, kRowThreads, nsm, S(stream)>>>(
        (const double*)x, n, dim, xn, (unsigned long long*)bad_row);
  }
  return check_launch("normalize_rows");
}

extern "C" int ivftq_residuals(const double* xn, const float* centroids,
                               const int32_t* list_ids, int64_t n, int dim, int flat,
                               double* resid_out, uint16_t* norm_out, void* stream) {
  if (n == 0) return 0;
  if (int e = set_row_smem((const void*)residual_kernel, dim)) return e;
  int grid = (int)((n + kRowTile - 1) / kRowTile);
  residual_kernel<<<grid, kRowThreads, row_smem(dim), S(stream)>>>(
      xn, centroids, list_ids, n, dim, flat, resid_out, norm_out);
  return check_launch("residuals");
}

extern "C" int ivftq_quantize_pack(const double* rot, const uint16_t* norms, int64_t n,
                                   int dim, int bits, int use_sign,
                                   const double* boundaries, const double* qcent,
                                   uint32_t* words_out, void* stream) {
  if (bits < 1 || bits > 8) {
    set_error("bits must be in [1, 8], got %d", bits);
    return IVFTQ_ERR_ARG;
  }
  if (n == 0) return 0;
  if (int e = set_row_smem((const void*)quantize_pack_kernel, dim)) return e;
  int grid = (int)((n + kRowTile - 1) / kRowTile);
  quantize_pack_kernel<<<grid, kRowThreads, row_smem(dim), S(stream)>>>(
      rot, norms, n, dim, bits, use_sign, boundaries, qcent, words_out);
  return check_launch("quantize_pack");
}

// Tensor-core rotation of pre-split rows (coarse_tc.cu): U = A . R^T in f32.
namespace ivftq {
int rotate_tc(const uint32_t* xh, const uint32_t* xl, int64_t n, int dim, const double* R,
              float* U, void* prep, cudaStream_t s);
}

extern "C" size_t ivftq_coarse_prep_bytes(int n_lists, int dim);
extern "C" int ivftq_coarse_tc_supported(int dim, int n_lists);

static size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

extern "C" size_t ivftq_encode_tc_scratch_bytes(int64_t n, int dim) {
  const int DP = (dim + 31) / 32 * 32;
  return a256(ivftq_coarse_prep_bytes(dim, dim)) + a256((size_t)n * DP * 4) +
         a256((size_t)n * dim * 4) + 2 * a256((size_t)n * 4) + 256 +
         a256((size_t)dim * dim * 8) + 256;
}

// Guard width of the tensor-core encoder: |u' - u| stays below 2^-20 on
// every measured shape (tests/test_gpu_parity.py::test_rotate_tc_error_inside_guard
// asserts a 4x margin); IVFTQ_ROT_EPS overrides it for experiments.
static double rot_eps() {
  const char* e = getenv("IVFTQ_ROT_EPS");
  return e ? atof(e) : 0x1p-18;
}

extern "C" int ivftq_encode_supported_tc(int dim) {
  return ivftq_coarse_tc_supported(dim, dim) && !getenv("IVFTQ_ENCODE_F64");
}

// residual -> unit -> tensor-core rotation: U (n, dim) f32 and the binary16
// residual norms. scratch >= ivftq_encode_tc_scratch_bytes(n, dim).
extern "C" int ivftq_rotate_unit_tc(const double* xn, const float* centroids,
                                    const int32_t* list_ids, int64_t n, int dim, int flat,
                                    const double* R, float* U_out, uint16_t* norm_out,
                                    void* scratch, size_t scratch_bytes, void* stream) {
  if (n == 0) return 0;
  if (!ivftq_coarse_tc_supported(dim, dim)) {
    set_error("rotate_unit_tc: dim %d not supported", dim);
    return IVFTQ_ERR_UNSUPPORTED;
  }
  if (scratch_bytes < ivftq_encode_tc_scratch_bytes(n, dim)) {
    set_error("rotate_unit_tc: scratch too small");
    return IVFTQ_ERR_SCRATCH;
  }
  const int DP = (dim + 31) / 32 * 32;
  unsigned char* p = (unsigned char*)scratch;
  void* prep = p;
  p += a256(ivftq_coarse_prep_bytes(dim, dim));
  uint32_t* xh = (uint32_t*)p;
  uint32_t* xl = xh + (size_t)n * (DP / 2);
  if (dim >= 8 && dim <= kDirectMax && !getenv("IVFTQ_ROWS_STAGED")) {
    resid_split_direct_kernel<<<(unsigned)((n * 8 + 255) / 256), 256, 0, S(stream)>>>(
        xn, centroids, list_ids, n, dim, DP, flat, norm_out, xh, xl);
  } else {
    if (int e = set_row_smem((const void*)resid_split_kernel, dim)) return e;
    const int grid = (int)((n + kRowTile - 1) / kRowTile);
    resid_split_kernel<<<grid, kSplitThreads, row_smem(dim), S(stream)>>>(
        xn, centroids, list_ids, n, dim, DP, flat, norm_out, xh, xl);
  }
  if (int e = check_launch("resid_split")) return e;
  return rotate_tc(xh, xl, n, dim, R, U_out, prep, S(stream));
}

// The whole post-assignment encoder on the tensor-core path:
// resid_split -> rotate_tc -> quantize_guard -> exact fix-up of the listed rows.
extern "C" int ivftq_encode_tail_tc(const double* xn, const float* centroids,
                                    const int32_t* list_ids, int64_t n, int dim, int bits,
                                    int use_sign, int flat, const double* R,
                                    const double* boundaries, const double* qcent,
                                    uint16_t* norm_out, uint32_t* words_out, void* scratch,
                                    size_t scratch_bytes, void* stream) {
  if (bits < 1 || bits > 8) {
    set_error("bits must be in [1, 8], got %d", bits);
    return IVFTQ_ERR_ARG;
  }
  if (n == 0) return 0;
  if (scratch_bytes < ivftq_encode_tc_scratch_bytes(n, dim)) {
    set_error("encode_tail_tc: scratch too small");
    return IVFTQ_ERR_SCRATCH;
  }
  const int DP = (dim + 31) / 32 * 32;
  unsigned char* p = (unsigned char*)scratch;
  p += a256(ivftq_coarse_prep_bytes(dim, dim)) + a256((size_t)n * DP * 4);
  float* U = (float*)p;
  p += a256((size_t)n * dim * 4);
  int32_t* flag = (int32_t*)p;
  p += a256((size_t)n * 4);
  int32_t* list = (int32_t*)p;
  p += a256((size_t)n * 4);
  int32_t* count = (int32_t*)p;
  p += 256;
  double* RT = (double*)p;
  cudaStream_t s = S(stream);
  if (int e = ivftq_rotate_unit_tc(xn, centroids, list_ids, n, dim, flat, R, U, norm_out, scratch,
                                   scratch_bytes, stream))
    return e;
  IVFTQ_CHECK_CUDA(cudaMemsetAsync(flag, 0, a256((size_t)n * 4) * 2 + 256, s));
  const int W = words_per_vec(dim, field_bits(bits, use_sign));
  const int64_t tot = n * W;
  quantize_guard_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(
      U, norm_out, n, dim, bits, use_sign, boundaries, qcent, rot_eps(), words_out, flag, list,
      count);
  if (int e = check_launch("quantize_guard")) return e;
  transpose_kernel<<<(dim * dim + 255) / 256, 256, 0, s>>>(R, dim, RT);
  if (int e = check_launch("transpose")) return e;
  const int fgrid = ivftq::device_sm_count() * 6;
  encode_fixup_kernel<<<fgrid, 128, sizeof(double) * 2 * kFixRows * dim, s>>>(
      xn, centroids, list_ids, dim, flat, RT, bits, use_sign, boundaries, qcent, list, count,
      words_out);
  return check_launch("encode_fixup");
}

extern "C" int ivftq_pack_codes(const uint8_t* bins, const uint8_t* signs, int64_t n,
                                int dim, int bits, int use_sign, uint32_t* words_out,
                                void* stream) {
  if (n == 0) return 0;
  int W = words_per_vec(dim, field_bits(bits, use_sign));
  int64_t tot = n * W;
  pack_codes_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, S(stream)>>>(
      bins, signs, n, dim, bits, use_sign, words_out);
  return check_launch("pack_codes");
}

extern "C" int ivftq_histogram(const int32_t* list_ids, int64_t n, int n_lists,
                               int32_t* counts, void* stream) {
  IVFTQ_CHECK_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * n_lists, S(stream)));
  if (n == 0) return 0;
  histogram_kernel<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(list_ids, n, n_lists,
                                                                     counts);
  return check_launch("histogram");
}

extern "C" int ivftq_append(const ivftq_store* store, const uint32_t* words,
                            const uint16_t* norms, const int32_t* list_ids, int64_t n,
                            int64_t first_id, int32_t* cursor, int64_t* slot_of,
                            void* stream) {
  IVFTQ_CHECK_CUDA(cudaMemsetAsync(cursor, 0, sizeof(int32_t) * store->n_lists, S(stream)));
  if (n == 0) return 0;
  append_kernel<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(
      *store, words, norms, list_ids, n, first_id, cursor, slot_of);
  return check_launch("append");
}

extern "C" int ivftq_relayout(const ivftq_store* src, const ivftq_store* dst,
                              int64_t* slot_of, void* stream) {
  if (src->n_lists != dst->n_lists || src->words_per_vec != dst->words_per_vec) {
    set_error("relayout: incompatible stores");
    return IVFTQ_ERR_ARG;
  }
  relayout_kernel<<<src->n_lists, 256, 0, S(stream)>>>(*src, *dst, slot_of);
  return check_launch("relayout");
}

extern "C" int ivftq_export_codes(const ivftq_store* store, const int64_t* slot_of,
                                  int64_t first, int64_t n, uint8_t* bins, uint8_t* signs,
                                  void* stream) {
  if (n == 0) return 0;
  int64_t tot = n * store->words_per_vec;
  export_codes_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, S(stream)>>>(
      *store, slot_of, first, n, bins, signs);
  return check_launch("export_codes");
}

extern "C" int ivftq_xor_codes(const ivftq_store* store, const int64_t* slot_of, int64_t n,
                               const uint8_t* mask, int which, int flip, void* stream) {
  if (n == 0) return 0;
  int64_t tot = n * store->words_per_vec;
  xor_codes_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, S(stream)>>>(
      *store, slot_of, n, mask, which, flip);
  return check_launch("xor_codes");
}
