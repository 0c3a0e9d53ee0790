// Search-side kernels: probe selection, LUT list scan + top-k, split merge,
// raw-store rerank.
//
// Reference: IvfTqIndex.search_batch (index.py:409-478) and _positions
// (index.py:480-483). The reference scores candidates with
//     coarse[q,l] (f64) + f64( (f32(T[code]) * f32(||r||)) @ f32(R q) )
// through a per-list f32 sgemm; the LUT scan computes the same residual term
// as ||r|| * sum_j f32(qrot_j * T32[code_j]) accumulated in f32, so scores
// agree to ~1e-7 relative (SURVEY.md §7 emulation: 9.6e-8).
#include <cstdio>

#include "common.cuh"
#include "topk.cuh"

namespace ivftq {

constexpr int kScanThreads = 128;  // 4 warps; one warp scores 32 slots per step
constexpr int kMaxProbesPerBlock = 1024;
constexpr int kMaxDepth = 7936;  // topk_cap(depth, 128) <= 8192

// ---------------------------------------------------------------------------
// Per-row top-n of an f64 score matrix (stable argsort order, index.py:438).
__global__ void __launch_bounds__(128)
select_topn_kernel(const double* __restrict__ scores, int cols, int n,
                   int32_t* __restrict__ idx_out, double* __restrict__ val_out) {
  extern __shared__ __align__(16) char smem[];
  BlockTopK tk;
  tk.carve(smem, topk_cap(n, 128), n);
  tk.init();
  __syncthreads();
  const double* row = scores + (int64_t)blockIdx.x * cols;
  for (int base = 0; base < cols; base += 128) {
    int c = base + threadIdx.x;
    double v = c < cols ? row[c] : -INFINITY;
    bool pass = c < cols && tk.passes(v, c);
    tk.push_warp(pass, v, c);
    tk.round_end(128);
  }
  tk.merge();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    idx_out[(int64_t)blockIdx.x * n + i] = i < *tk.cnt ? tk.id[i] : -1;
    val_out[(int64_t)blockIdx.x * n + i] = i < *tk.cnt ? tk.s[i] : -INFINITY;
  }
}

// ---------------------------------------------------------------------------
// LUT list scan. Block = (query q, probe split). The block builds the query's
// LUT lut[j][c] = f32(qrot_j * T32[c]) in shared memory (field c is the
// lane-private code of coordinate j; with all lanes on the same j the bank is
// c, so lookups are conflict-free for field_bits <= 5), then walks its probed
// lists 32 slots per warp step, one slot per lane.
template <int FB, bool DIRECT>
__global__ void __launch_bounds__(kScanThreads)
scan_lut_kernel(ivftq_store st, const int32_t* __restrict__ probe,
                const double* __restrict__ coarse, const float* __restrict__ qrot,
                const double* __restrict__ levels, int n_p, int n_split, int K,
                double* __restrict__ part_s, int32_t* __restrict__ part_id) {
  constexpr int C = 1 << FB;
  constexpr int FPW = 32 / FB;
  constexpr uint32_t MASK = (1u << FB) - 1u;
  extern __shared__ __align__(16) char smem[];
  const int d = st.dim, W = st.words_per_vec;
  const int64_t q = blockIdx.x;
  const int split = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // LUT mode: lut[j*C + c]; DIRECT mode (LUT too large for shared memory):
  // qs[j] and Ts[c] with the identical f32 product formed per lookup.
  float* lut = (float*)smem;
  float* Ts = lut + d;
  int* pl = (int*)(lut + (DIRECT ? (size_t)d + C : (size_t)d * C));
  int* pref = pl + kMaxProbesPerBlock;  // kMaxProbesPerBlock + 1
  double* pc = (double*)(((uintptr_t)(pref + kMaxProbesPerBlock + 2) + 7) & ~(uintptr_t)7);
  char* tkbase = (char*)(pc + kMaxProbesPerBlock);
  BlockTopK tk;
  tk.carve(tkbase, topk_cap(K, kScanThreads), K);
  tk.init();

  const float* qr = qrot + q * d;
  if (DIRECT) {
    for (int i = threadIdx.x; i < d; i += blockDim.x) lut[i] = qr[i];
    for (int i = threadIdx.x; i < C; i += blockDim.x) Ts[i] = (float)levels[i];
  } else {
    for (int i = threadIdx.x; i < d * C; i += blockDim.x) {
      int j = i / C, c = i - j * C;
      lut[i] = __fmul_rn(qr[j], (float)levels[c]);
    }
  }
  int np_b = (n_p - split + n_split - 1) / n_split;
  if (threadIdx.x == 0) {
    int acc = 0;
    pref[0] = 0;
    for (int t = 0; t < np_b; ++t) {
      int p = split + t * n_split;
      int l = probe[q * n_p + p];
      pl[t] = l;
      pc[t] = coarse[q * n_p + p];
      int sz = l >= 0 ? st.list_size[l] : 0;
      acc += (sz + 31) >> 5;
      pref[t + 1] = acc;
    }
  }
  __syncthreads();
  const int total = pref[np_b];
  int t = 0;
  for (int base = 0; base < total; base += kScanThreads / 32) {
    int item = base + warp;
    bool pass = false;
    double score = 0.0;
    int vid = 0;
    if (item < total) {
      while (pref[t + 1] <= item) ++t;
      DCHECK(t < np_b, "t=%d np_b=%d item=%d total=%d", t, np_b, item, total);
      int l = pl[t];
      DCHECK(l >= 0 && l < st.n_lists, "l=%d t=%d q=%lld", l, t, (long long)q);
      int blk = item - pref[t];
      int size = st.list_size[l];
      int64_t off = st.list_offset[l];
      DCHECK(off >= 0 && off + (int64_t)blk * 32 + 32 <= st.capacity + 32,
             "off=%lld blk=%d size=%d cap=%lld", (long long)off, blk, size,
             (long long)st.capacity);
      int64_t gblk = (off >> 5) + blk;
      bool valid = blk * 32 + lane < size;
      if (valid) {
        const uint32_t* cw = st.codes + gblk * W * 32 + lane;
        float acc = 0.f;
        int j0 = 0;
        for (int w = 0; w < W; ++w, j0 += FPW) {
          uint32_t word = __ldg(cw + w * 32);
          if (DIRECT) {
            for (int f = 0; f < FPW && j0 + f < d; ++f)
              acc = __fadd_rn(acc, __fmul_rn(lut[j0 + f], Ts[(word >> (FB * f)) & MASK]));
          } else {
            const float* lrow = lut + j0 * C;
            if (j0 + FPW <= d) {
#pragma unroll
              for (int f = 0; f < FPW; ++f)
                acc = __fadd_rn(acc, lrow[f * C + ((word >> (FB * f)) & MASK)]);
            } else {
              for (int f = 0; j0 + f < d; ++f)
                acc = __fadd_rn(acc, lrow[f * C + ((word >> (FB * f)) & MASK)]);
            }
          }
        }
        int64_t slot = (off) + blk * 32 + lane;
        float nr = h2f_bits(st.norms[slot]);
        float res = __fmul_rn(acc, nr);
        score = pc[t] + (double)res;
        vid = st.ids[slot];
        pass = tk.passes(score, vid);
      }
    }
    tk.push_warp(pass, score, vid);
    tk.round_end(kScanThreads);
  }
  tk.merge();
  int64_t ob = (q * n_split + split) * (int64_t)K;
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    bool have = i < *tk.cnt;
    part_s[ob + i] = have ? tk.s[i] : -INFINITY;
    part_id[ob + i] = have ? tk.id[i] : INT_MAX;
  }
}

// Merge the n_split partial lists of each query into the final top-k
// (index.py:460-478), padding with id -1 / score -inf.
__global__ void __launch_bounds__(128)
merge_kernel(const double* __restrict__ part_s, const int32_t* __restrict__ part_id,
             int n_in, int K, int64_t* __restrict__ ids_out, double* __restrict__ s_out) {
  extern __shared__ __align__(16) char smem[];
  BlockTopK tk;
  tk.carve(smem, topk_cap(K, 128), K);
  tk.init();
  __syncthreads();
  const int64_t q = blockIdx.x;
  const double* ps = part_s + q * n_in;
  const int32_t* pi = part_id + q * n_in;
  for (int base = 0; base < n_in; base += 128) {
    int c = base + threadIdx.x;
    double v = -INFINITY;
    int id = INT_MAX;
    if (c < n_in) { v = ps[c]; id = pi[c]; }
    bool pass = c < n_in && id != INT_MAX && tk.passes(v, id);
    tk.push_warp(pass, v, id);
    tk.round_end(128);
  }
  tk.merge();
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    bool have = i < *tk.cnt;
    ids_out[q * K + i] = have ? (int64_t)tk.id[i] : -1;
    s_out[q * K + i] = have ? tk.s[i] : -INFINITY;
  }
}

// Exact f64 re-score of candidates against the raw store (index.py:470-473).
__global__ void __launch_bounds__(128)
rerank_kernel(const float* __restrict__ raw, const double* __restrict__ qn,
              const int64_t* __restrict__ cand, int depth, int d, int k,
              int64_t* __restrict__ ids_out, double* __restrict__ s_out) {
  extern __shared__ __align__(16) char smem[];
  BlockTopK tk;
  tk.carve(smem, topk_cap(k, 128), k);
  tk.init();
  __syncthreads();
  const int64_t q = blockIdx.x;
  const double* qv = qn + q * d;
  for (int base = 0; base < depth; base += 128) {
    int c = base + threadIdx.x;
    int64_t id = c < depth ? cand[q * depth + c] : -1;
    double v = 0.0;
    if (id >= 0) {
      const float* r = raw + id * d;
      for (int j = 0; j < d; ++j) v = __fma_rn((double)r[j], qv[j], v);
    }
    bool pass = id >= 0 && tk.passes(v, (int)id);
    tk.push_warp(pass, v, (int)id);
    tk.round_end(128);
  }
  tk.merge();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    bool have = i < *tk.cnt;
    ids_out[q * k + i] = have ? (int64_t)tk.id[i] : -1;
    s_out[q * k + i] = have ? tk.s[i] : -INFINITY;
  }
}

}  // namespace ivftq

using namespace ivftq;

static int smem_opt_in(const void* fn, size_t bytes) {
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

extern "C" int ivftq_select_topn(const double* scores, int64_t rows, int cols, int n,
                                 int32_t* idx_out, double* val_out, void* stream) {
  if (n < 1 || n > cols || n > kMaxDepth) {
    set_error("select_topn: n=%d must be in [1, min(cols=%d, %d)]", n, cols, kMaxDepth);
    return IVFTQ_ERR_ARG;
  }
  if (rows == 0) return 0;
  size_t sm = BlockTopK::bytes(topk_cap(n, 128));
  if (int e = smem_opt_in((const void*)select_topn_kernel, sm)) return e;
  select_topn_kernel<<<(unsigned)rows, 128, sm, (cudaStream_t)stream>>>(scores, cols, n,
                                                                        idx_out, val_out);
  return check_launch("select_topn");
}

extern "C" size_t ivftq_probe_scratch_bytes(int64_t nq, int n_lists) {
  return (size_t)nq * n_lists * sizeof(double) + 256;
}

extern "C" int ivftq_probe(const double* qn, const float* centroids, int64_t nq, int n_lists,
                           int dim, int n_p, int32_t* probe_out, double* coarse_out,
                           void* scratch, size_t scratch_bytes, void* stream) {
  if (scratch_bytes < ivftq_probe_scratch_bytes(nq, n_lists)) {
    set_error("probe: scratch too small");
    return IVFTQ_ERR_SCRATCH;
  }
  double* S = (double*)scratch;
  if (int e = ivftq_gemm_nt(qn, centroids, IVFTQ_F32, nq, n_lists, dim, S, IVFTQ_F64, stream))
    return e;
  return ivftq_select_topn(S, nq, n_lists, n_p, probe_out, coarse_out, stream);
}

static int scan_splits(int64_t nq, int n_p) {
  int sm_count = 148;
  int want = (int)((4 * sm_count + nq - 1) / (nq > 0 ? nq : 1));
  int splits = want < 1 ? 1 : want;
  if (splits > n_p) splits = n_p;
  int need = (n_p + kMaxProbesPerBlock - 1) / kMaxProbesPerBlock;
  if (splits < need) splits = need;
  return splits;
}

static size_t lut_scratch_bytes(int64_t nq, int n_p, int depth) {
  int sp = scan_splits(nq, n_p);
  return (size_t)nq * sp * depth * (sizeof(double) + sizeof(int32_t)) + 512;
}

namespace ivftq {
int merge_smem_opt_in(int K) {
  return smem_opt_in((const void*)merge_kernel, BlockTopK::bytes(topk_cap(K, 128)));
}
void launch_merge(const double* part_s, const int32_t* part_id, int64_t nq, int n_in, int K,
                  int64_t* ids_out, double* s_out, cudaStream_t s) {
  merge_kernel<<<(unsigned)nq, 128, BlockTopK::bytes(topk_cap(K, 128)), s>>>(
      part_s, part_id, n_in, K, ids_out, s_out);
}
}  // namespace ivftq

extern "C" size_t ivftq_scan_scratch_bytes(int64_t nq, int n_p, int depth, int n_lists) {
  size_t a = lut_scratch_bytes(nq, n_p, depth);
  size_t b = ivftq_scan_tc_scratch_bytes(nq, n_p, n_lists, depth);
  return a > b ? a : b;
}

extern "C" int ivftq_scan_topk_lut(const ivftq_store* st, const int32_t* probe,
                                   const double* coarse, const float* qrot,
                                   const double* levels, int64_t nq, int n_p, int depth,
                                   int64_t* ids_out, double* scores_out, void* scratch,
                                   size_t scratch_bytes, void* stream) {
  if (depth < 1 || depth > kMaxDepth) {
    set_error("scan_topk: depth %d outside [1, %d]", depth, kMaxDepth);
    return IVFTQ_ERR_UNSUPPORTED;
  }
  if (n_p < 1) {
    set_error("scan_topk: n_p must be >= 1");
    return IVFTQ_ERR_ARG;
  }
  if (nq == 0) return 0;
  if (scratch_bytes < lut_scratch_bytes(nq, n_p, depth)) {
    set_error("scan_topk: scratch too small");
    return IVFTQ_ERR_SCRATCH;
  }
  int sp = scan_splits(nq, n_p);
  double* part_s = (double*)scratch;
  int32_t* part_id = (int32_t*)(part_s + (size_t)nq * sp * depth);
  int C = 1 << st->field_bits;
  size_t rest = (size_t)(2 * kMaxProbesPerBlock + 2) * 4 + (size_t)kMaxProbesPerBlock * 8 + 32 +
                BlockTopK::bytes(topk_cap(depth, kScanThreads));
  size_t lut_bytes = (size_t)st->dim * C * 4;
  bool direct = lut_bytes + rest > 200 * 1024;
  size_t sm = (direct ? (size_t)(st->dim + C) * 4 : lut_bytes) + rest;
  sm = (sm + 15) & ~(size_t)15;
  dim3 grid((unsigned)nq, sp);
  cudaStream_t s = (cudaStream_t)stream;
  const void* fn = nullptr;
  switch (st->field_bits) {
#define LAUNCH(FB, DIR)                                                             \
  fn = (const void*)scan_lut_kernel<FB, DIR>;                                       \
  if (int e = smem_opt_in(fn, sm)) return e;                                        \
  scan_lut_kernel<FB, DIR><<<grid, kScanThreads, sm, s>>>(                          \
      *st, probe, coarse, qrot, levels, n_p, sp, depth, part_s, part_id);
#define CASE(FB)                   \
  case FB:                         \
    if (direct) {                  \
      LAUNCH(FB, true)             \
    } else {                       \
      LAUNCH(FB, false)            \
    }                              \
    break;
    CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9)
#undef CASE
#undef LAUNCH
    default:
      set_error("scan_topk: unsupported field width %d", st->field_bits);
      return IVFTQ_ERR_UNSUPPORTED;
  }
  if (int e = check_launch("scan_lut")) return e;
  if (int e = merge_smem_opt_in(depth)) return e;
  launch_merge(part_s, part_id, nq, sp * depth, depth, ids_out, scores_out, s);
  return check_launch("merge");
}

// Batched queries with small depth go to the tensor-core list-major scan; a
// handful of queries (few queries per probed list) or large depth use the
// query-major LUT scan.
extern "C" int ivftq_scan_topk(const ivftq_store* st, const int32_t* probe, const double* coarse,
                               const float* qrot, const double* levels, int64_t nq, int n_p,
                               int depth, int64_t* ids_out, double* scores_out, void* scratch,
                               size_t scratch_bytes, void* stream) {
  bool tc = nq >= 64 && ivftq_scan_tc_supported(st->dim, st->bits, depth);
  if (tc)
    return ivftq_scan_topk_tc(st, probe, coarse, qrot, levels, nq, n_p, depth, ids_out,
                              scores_out, scratch, scratch_bytes, stream);
  return ivftq_scan_topk_lut(st, probe, coarse, qrot, levels, nq, n_p, depth, ids_out,
                             scores_out, scratch, scratch_bytes, stream);
}

extern "C" int ivftq_rerank(const float* raw, const double* qn, const int64_t* cand_ids,
                            int64_t nq, int depth, int dim, int k, int64_t* ids_out,
                            double* scores_out, void* stream) {
  if (k < 1 || k > kMaxDepth || depth < 1) {
    set_error("rerank: bad k/depth");
    return IVFTQ_ERR_ARG;
  }
  if (nq == 0) return 0;
  size_t sm = BlockTopK::bytes(topk_cap(k, 128));
  if (int e = smem_opt_in((const void*)rerank_kernel, sm)) return e;
  rerank_kernel<<<(unsigned)nq, 128, sm, (cudaStream_t)stream>>>(raw, qn, cand_ids, depth, dim,
                                                                 k, ids_out, scores_out);
  return check_launch("rerank");
}
