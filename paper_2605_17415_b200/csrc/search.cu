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

// Small n (every realistic nprobe): one warp per row keeps the row's best n
// as a sorted queue in registers, 32*S positions (position s*32+lane in
// slot s of that lane). Columns stream through in ascending order 32 at a
// time; a column enters only if it beats the current n-th entry, so after the
// first few chunks almost every column is rejected by one compare + ballot.
// Since columns arrive in ascending id order, an entry equal in value to a
// queued one belongs after it: the insert position is the count of queued
// keys >= its key, which reproduces (value desc, column asc) exactly.
// Values are compared as order-preserving int64 keys (-0.0 folded onto +0.0,
// NaN below -inf, matching a stable argsort of -scores).
__device__ __forceinline__ long long order_key(double x) {
  if (x == 0.0) x = 0.0;
  long long b = __double_as_longlong(x);
  if (x != x) return LLONG_MIN;
  return b >= 0 ? b : (b ^ 0x7fffffffffffffffLL);
}
__device__ __forceinline__ double key_value(long long k) {
  return __longlong_as_double(k >= 0 ? k : (k ^ 0x7fffffffffffffffLL));
}

template <int S>
__device__ void warp_queue_select(const double* __restrict__ row, int cols, int n,
                                  int32_t* __restrict__ io, double* __restrict__ vo) {
  const int lane = threadIdx.x & 31;
  long long qk[S];
  int qi[S];
#pragma unroll
  for (int s = 0; s < S; ++s) { qk[s] = LLONG_MIN; qi[s] = -1; }
  int cnt = 0;                      // filled positions
  long long thr = LLONG_MIN;        // key at position n-1 once full
  const int tl = (n - 1) & 31, ts = (n - 1) >> 5;
  constexpr int kPre = 4;           // chunks loaded ahead
  for (int base = 0; base < cols; base += 32 * kPre) {
    double v[kPre];
#pragma unroll
    for (int u = 0; u < kPre; ++u) {
      const int c = base + u * 32 + lane;
      v[u] = c < cols ? __ldg(row + c) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPre; ++u) {
      const int c = base + u * 32 + lane;
      const long long key = order_key(v[u]);
      unsigned m = __ballot_sync(kFull, c < cols && (cnt < n || key > thr));
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const long long k = __shfl_sync(kFull, key, src);
        if (cnt == n && !(k > thr)) continue;   // threshold rose meanwhile
        int p = 0;
#pragma unroll
        for (int s = 0; s < S; ++s)
          p += __popc(__ballot_sync(kFull, (s * 32 + lane) < cnt && qk[s] >= k));
        // shift positions >= p one place later; the entry at n-1 falls off
        long long rk[S];
        int ri[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
          rk[s] = __shfl_sync(kFull, qk[s], (lane + 31) & 31);
          ri[s] = __shfl_sync(kFull, qi[s], (lane + 31) & 31);
        }
#pragma unroll
        for (int s = S - 1; s >= 0; --s) {
          const int pos = s * 32 + lane;
          long long pk = rk[s];
          int pi = ri[s];
          if (lane == 0) {
            pk = s > 0 ? rk[s > 0 ? s - 1 : 0] : LLONG_MIN;
            pi = s > 0 ? ri[s > 0 ? s - 1 : 0] : -1;
          }
          if (pos > p) { qk[s] = pk; qi[s] = pi; }
          else if (pos == p) { qk[s] = k; qi[s] = base + u * 32 + src; }
        }
        cnt = min(cnt + 1, n);
        if (cnt == n) {
          long long t = qk[0];
#pragma unroll
          for (int s = 1; s < S; ++s) if (s == ts) t = qk[s];
          thr = __shfl_sync(kFull, t, tl);
        }
      }
    }
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int pos = s * 32 + lane;
    if (pos < n) {
      const bool ok = pos < cnt;
      io[pos] = ok ? qi[s] : -1;
      vo[pos] = ok ? key_value(qk[s]) : -INFINITY;
    }
  }
}

// Fast path, one warp per row, three passes over the (L1/L2-resident) row:
//   1. min / max;
//   2. a 256-bin histogram of the linear map (v - min) * 256 / (max - min),
//      monotone in v, so the bin b holding the n-th best value bounds the
//      selection: every value in bins > b is in, every value in bins < b out;
//   3. compact the values in bins >= b (normally n plus a few) into shared
//      memory and give each its exact rank (count of better candidates under
//      value desc / column asc); ranks < n are the answer.
// Rows the map cannot split (NaN, infinities, all-equal, or a boundary bin so
// crowded that the candidates overflow) take the warp-queue path above, which
// is exact for any input.
constexpr int kSelBins = 256;
template <int S>
__global__ void __launch_bounds__(256)
select_warp_kernel(const double* __restrict__ scores, int64_t rows, int cols, int n,
                   int32_t* __restrict__ idx_out, double* __restrict__ val_out) {
  constexpr int CAP = 32 * S + 64;
  constexpr int kWarps = 8;
  __shared__ unsigned hist_all[kWarps][kSelBins];
  __shared__ long long ck_all[kWarps][CAP];
  __shared__ int ci_all[kWarps][CAP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * kWarps + warp;
  if (r >= rows) return;
  const double* row = scores + r * cols;
  int32_t* io = idx_out + r * n;
  double* vo = val_out + r * n;
  unsigned* hist = hist_all[warp];
  long long* ck = ck_all[warp];
  int* ci = ci_all[warp];

  double mn = INFINITY, mx = -INFINITY;
  bool nan = false;
  for (int c = lane; c < cols; c += 32) {
    const double v = __ldg(row + c);
    nan |= v != v;
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(kFull, mn, o));
    mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
  }
  const double span = mx - mn;
  if (__any_sync(kFull, nan) || !(span > 0.0) || !(span < INFINITY)) {
    warp_queue_select<S>(row, cols, n, io, vo);
    return;
  }
  const double scale = (double)kSelBins / span;
  auto bin_of = [&](double v) { return min(kSelBins - 1, (int)((v - mn) * scale)); };
#pragma unroll
  for (int i = 0; i < kSelBins / 32; ++i) hist[i * 32 + lane] = 0;
  __syncwarp();
  for (int c = lane; c < cols; c += 32) atomicAdd(&hist[bin_of(__ldg(row + c))], 1u);
  __syncwarp();
  // lane l owns bins [kSelBins-8(l+1), kSelBins-8l), i.e. lane 0 the top bins
  unsigned own[kSelBins / 32];
  unsigned tot = 0;
#pragma unroll
  for (int i = 0; i < kSelBins / 32; ++i) {
    own[i] = hist[kSelBins - 1 - (lane * (kSelBins / 32) + i)];
    tot += own[i];
  }
  unsigned incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned t = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += t;
  }
  const unsigned excl = incl - tot;
  const int owner = __ffs(__ballot_sync(kFull, incl >= (unsigned)n)) - 1;
  int bsel = 0;
  if (lane == owner) {
    unsigned acc = excl;
#pragma unroll
    for (int i = 0; i < kSelBins / 32; ++i) {
      acc += own[i];
      if (acc >= (unsigned)n) { bsel = kSelBins - 1 - (lane * (kSelBins / 32) + i); break; }
    }
  }
  const int b = __shfl_sync(kFull, bsel, owner);
  const unsigned total = __shfl_sync(kFull, incl, owner);  // upper bound on candidates
  (void)total;
  int c_n = 0;
  for (int base = 0; base < cols; base += 32) {
    const int c = base + lane;
    double v = 0.0;
    bool in = false;
    if (c < cols) {
      v = __ldg(row + c);
      in = bin_of(v) >= b;
    }
    const unsigned m = __ballot_sync(kFull, in);
    const int at = c_n + __popc(m & ((1u << lane) - 1u));
    if (in && at < CAP) { ck[at] = order_key(v); ci[at] = c; }
    c_n += __popc(m);
  }
  if (c_n > CAP) {
    warp_queue_select<S>(row, cols, n, io, vo);
    return;
  }
  __syncwarp();
  constexpr int PER = (CAP + 31) / 32;
  long long mk[PER];
  int mi[PER], rank[PER];
#pragma unroll
  for (int t = 0; t < PER; ++t) {
    const int i = t * 32 + lane;
    mk[t] = i < c_n ? ck[i] : LLONG_MIN;
    mi[t] = i < c_n ? ci[i] : INT_MAX;
    rank[t] = 0;
  }
  for (int j = 0; j < c_n; ++j) {
    const long long kj = ck[j];
    const int ij = ci[j];
#pragma unroll
    for (int t = 0; t < PER; ++t) rank[t] += (kj > mk[t]) || (kj == mk[t] && ij < mi[t]);
  }
#pragma unroll
  for (int t = 0; t < PER; ++t) {
    const int i = t * 32 + lane;
    if (i < c_n && rank[t] < n) {
      io[rank[t]] = mi[t];
      vo[rank[t]] = key_value(mk[t]);
    }
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

// Warp-per-query merge for K <= 32*QS: a register queue sorted by (score
// desc, id asc) with early rejection against its last entry; candidates
// arrive in any order, so the insert position counts strictly better entries.
template <int QS>
__global__ void __launch_bounds__(256)
merge_warp_kernel(const double* __restrict__ part_s, const int32_t* __restrict__ part_id,
                  int64_t nq, int n_in, int K, int64_t* __restrict__ ids_out,
                  double* __restrict__ s_out, const int32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  const double* ps = part_s + q * n_in;
  const int32_t* pi = part_id + q * n_in;
  if (counts) n_in = min(n_in, counts[q]);  // compact per-query buffer
  long long qk[QS];
  int qi[QS];
#pragma unroll
  for (int s = 0; s < QS; ++s) { qk[s] = LLONG_MIN; qi[s] = INT_MAX; }
  int cnt = 0;
  long long tk = LLONG_MIN;
  int ti = INT_MAX;
  const int tl = (K - 1) & 31, ts = (K - 1) >> 5;
  for (int base = 0; base < n_in; base += 32) {
    const int c = base + lane;
    const int id = c < n_in ? pi[c] : INT_MAX;
    const long long key = id != INT_MAX ? order_key(ps[c]) : LLONG_MIN;
    unsigned m = __ballot_sync(kFull, id != INT_MAX && (cnt < K || key > tk || (key == tk && id < ti)));
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const long long k = __shfl_sync(kFull, key, src);
      const int kid = __shfl_sync(kFull, id, src);
      if (cnt == K && !(k > tk || (k == tk && kid < ti))) continue;
      int p = 0;
#pragma unroll
      for (int s = 0; s < QS; ++s)
        p += __popc(__ballot_sync(kFull, (s * 32 + lane) < cnt &&
                                             (qk[s] > k || (qk[s] == k && qi[s] < kid))));
      long long rk[QS];
      int ri[QS];
#pragma unroll
      for (int s = 0; s < QS; ++s) {
        rk[s] = __shfl_sync(kFull, qk[s], (lane + 31) & 31);
        ri[s] = __shfl_sync(kFull, qi[s], (lane + 31) & 31);
      }
#pragma unroll
      for (int s = QS - 1; s >= 0; --s) {
        const int pos = s * 32 + lane;
        long long pk = rk[s];
        int pv = ri[s];
        if (lane == 0) {
          pk = s > 0 ? rk[s > 0 ? s - 1 : 0] : LLONG_MIN;
          pv = s > 0 ? ri[s > 0 ? s - 1 : 0] : INT_MAX;
        }
        if (pos > p) { qk[s] = pk; qi[s] = pv; }
        else if (pos == p) { qk[s] = k; qi[s] = kid; }
      }
      cnt = min(cnt + 1, K);
      if (cnt == K) {
        long long t = qk[0];
        int u = qi[0];
#pragma unroll
        for (int s = 1; s < QS; ++s) if (s == ts) { t = qk[s]; u = qi[s]; }
        tk = __shfl_sync(kFull, t, tl);
        ti = __shfl_sync(kFull, u, tl);
      }
    }
  }
#pragma unroll
  for (int s = 0; s < QS; ++s) {
    const int pos = s * 32 + lane;
    if (pos < K) {
      const bool have = pos < cnt;
      ids_out[q * K + pos] = have ? (int64_t)qi[s] : -1;
      s_out[q * K + pos] = have ? key_value(qk[s]) : -INFINITY;
    }
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
  if (n <= 128) {
    const unsigned blocks = (unsigned)((rows + 7) / 8);
    auto s = (cudaStream_t)stream;
    if (n <= 32)
      select_warp_kernel<1><<<blocks, 256, 0, s>>>(scores, rows, cols, n, idx_out, val_out);
    else if (n <= 64)
      select_warp_kernel<2><<<blocks, 256, 0, s>>>(scores, rows, cols, n, idx_out, val_out);
    else
      select_warp_kernel<4><<<blocks, 256, 0, s>>>(scores, rows, cols, n, idx_out, val_out);
    return check_launch("select_warp");
  }
  size_t sm = BlockTopK::bytes(topk_cap(n, 128));
  if (int e = smem_opt_in((const void*)select_topn_kernel, sm)) return e;
  select_topn_kernel<<<(unsigned)rows, 128, sm, (cudaStream_t)stream>>>(scores, cols, n,
                                                                        idx_out, val_out);
  return check_launch("select_topn");
}

#include <atomic>
extern std::atomic<bool> g_probe_tc_force;
int probe_tc(const double* qn, const float* centroids, int64_t nq, int n_lists, int dim,
             int n_p, int32_t* probe_out, double* coarse_out, void* scratch,
             size_t scratch_bytes, cudaStream_t s, const void* prepared);
extern "C" size_t ivftq_probe_tc_scratch_bytes(int64_t nq, int n_lists, int dim);
extern "C" int ivftq_coarse_tc_supported(int dim, int n_lists);
static bool probe_tc_auto() { return ivftq_coarse_tc_supported(128, 1) != 0; }  // mode != 1
static bool probe_tc_enabled() {
  static const bool env = [] {  // thread-safe one-time read of the environment
    const char* e = getenv("IVFTQ_PROBE_TC");
    return e && e[0] == '1';
  }();
  return env || g_probe_tc_force;
}

extern "C" size_t ivftq_probe_scratch_bytes(int64_t nq, int n_lists, int dim) {
  const size_t t = ivftq_probe_tc_scratch_bytes(nq, n_lists, dim);
  const size_t f = (size_t)nq * n_lists * sizeof(double) + 256;
  return t > f ? t : f;
}

static size_t probe_f64_scratch_bytes(int64_t nq, int n_lists) {
  return (size_t)nq * n_lists * sizeof(double) + 256;
}

static int probe_impl(const double* qn, const float* centroids, const void* prepared,
                      int64_t nq, int n_lists, int dim, int n_p, int32_t* probe_out,
                      double* coarse_out, void* scratch, size_t scratch_bytes, void* stream);

extern "C" int ivftq_probe(const double* qn, const float* centroids, int64_t nq, int n_lists,
                           int dim, int n_p, int32_t* probe_out, double* coarse_out,
                           void* scratch, size_t scratch_bytes, void* stream) {
  return probe_impl(qn, centroids, nullptr, nq, n_lists, dim, n_p, probe_out, coarse_out,
                    scratch, scratch_bytes, stream);
}

extern "C" int ivftq_probe_prepared(const double* qn, const float* centroids,
                                    const void* prepared, int64_t nq, int n_lists, int dim,
                                    int n_p, int32_t* probe_out, double* coarse_out,
                                    void* scratch, size_t scratch_bytes, void* stream) {
  return probe_impl(qn, centroids, prepared, nq, n_lists, dim, n_p, probe_out, coarse_out,
                    scratch, scratch_bytes, stream);
}

static int probe_impl(const double* qn, const float* centroids, const void* prepared,
                      int64_t nq, int n_lists, int dim, int n_p, int32_t* probe_out,
                      double* coarse_out, void* scratch, size_t scratch_bytes, void* stream) {
  if (scratch_bytes < probe_f64_scratch_bytes(nq, n_lists)) {
    set_error("probe: scratch too small");
    return IVFTQ_ERR_SCRATCH;
  }
  if (n_p < 1 || n_p > n_lists) {
    set_error("probe: n_p=%d must be in [1, n_lists=%d]", n_p, n_lists);
    return IVFTQ_ERR_ARG;
  }
  if (nq == 0) return 0;
  // Path choice (identical probes; coarse values exact f64 in both, summed in
  // a different order): the tensor-core path pays a dense tcgen05 GEMM, a
  // fused per-row selection and an exact f64 re-score of ~n_p gathered
  // centroid rows per query; the f64 path a dense DFMA GEMM plus a top-n_p
  // select. Measured on B200 (scripts/probe_mode_bench.py, nq = 10k): L=1024
  // n_p=64: f64 0.243 ms vs tc 0.180; L=4096 d=96 n_p=32: 0.724 vs 0.223;
  // n_p=128: 0.858 vs 0.356; d=200 n_p=64: 1.206 vs 0.343 -- so tensor cores
  // whenever supported (mode 0 / 2 / IVFTQ_PROBE_TC=1), never (mode 1). The
  // choice never depends on the batch size, so a query's probes and coarse
  // values do not depend on which batch (or chunk) it arrives in.
  if (probe_tc_enabled() || probe_tc_auto()) {
    const int e = probe_tc(qn, centroids, nq, n_lists, dim, n_p, probe_out, coarse_out, scratch,
                           scratch_bytes, (cudaStream_t)stream, prepared);
    if (e != IVFTQ_ERR_UNSUPPORTED) return e;
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
                  int64_t* ids_out, double* s_out, cudaStream_t s,
                  const int32_t* counts = nullptr) {
  const unsigned wb = (unsigned)((nq + 7) / 8);
  if (K <= 32)
    merge_warp_kernel<1><<<wb, 256, 0, s>>>(part_s, part_id, nq, n_in, K, ids_out, s_out, counts);
  else if (K <= 64)
    merge_warp_kernel<2><<<wb, 256, 0, s>>>(part_s, part_id, nq, n_in, K, ids_out, s_out, counts);
  else  // deep rerank lists (LUT path only; the tensor-core scan caps depth at 32)
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
