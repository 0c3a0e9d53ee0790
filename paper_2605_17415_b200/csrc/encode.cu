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
