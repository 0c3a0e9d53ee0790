// GPU spherical k-means for the partition refresh.
//
// Reference: partition.py:64-178 (train_partition: k-means++ seeding with
// 2 + log2(k) candidates per step, then Lloyd iterations on unit rows) as
// called by refresh.py:171-175 on the reconstructed sample.
//
//   * ivftq_kmeanspp_seed runs the whole seeding loop on the device: per step
//     a cdf search of the host-drawn uniforms over the potential d2 (the
//     reference's rng.choice(n, size=nc, p=d2/tot): same uniforms, same
//     inverse-cdf rule), one pass over the rows that scores the nc candidates
//     (f64 DFMA, rows staged through shared memory, a 2 x NCH register tile per
//     thread), the potential of each candidate by a fixed-order reduction,
//     the first arg-min, and the update of d2 with that candidate's column.
//     Nothing returns to the host inside the loop; the per-step potential
//     totals come back at the end so the caller can detect the degenerate
//     case the reference handles on its slow branch.
//   * ivftq_kmeans_sums is the Lloyd update: a stable counting sort of the
//     rows by list (per-block histograms, a column scan, in-order ranks), then
//     one thread per (list, coordinate) adding the list's rows, taken in
//     ascending row order, in the order of np.add.reduceat over
//     data[argsort(a, stable)] (first row + numpy's pairwise sum of the
//     rest), so the f64 sums are bit-identical to the reference's.
//   The Lloyd assignment is ivftq_assign_tc64 (coarse_tc.cu): the tensor-core
//   pass with the exact f64 guard band, on the step's f64 centroids.
//
// Every reduction has a fixed order: two runs give identical bits.
#include <cstdio>

#include "common.cuh"

namespace ivftq {
namespace km {

constexpr int kScanChunk = 1024;  // rows per potential block sum
constexpr int kCandRows = 128;    // rows per block of the candidate pass
constexpr int kMaxCand = 18;      // 2 + log2(k), k <= 65536
constexpr int kSortRows = 256;    // rows per block of the counting sort

// ---- seeding -----------------------------------------------------------------
// d2 <- column `which` of cd2t (or the only column at init), S[b] = block sums
__global__ void __launch_bounds__(kScanChunk)
kpp_update_kernel(double* __restrict__ d2, const double* __restrict__ cd2t,
                  const int* __restrict__ bsel, int64_t n, int init, double* __restrict__ S) {
  __shared__ double red[kScanChunk];
  const int64_t i = (int64_t)blockIdx.x * kScanChunk + threadIdx.x;
  const int col = init ? 0 : *bsel;
  double v = 0.0;
  if (i < n) {
    const double c = cd2t[(int64_t)col * n + i];
    v = init ? c : fmin(d2[i], c);
    d2[i] = v;
  }
  red[threadIdx.x] = v;
  __syncthreads();
  for (int o = kScanChunk / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) S[blockIdx.x] = red[0];
}

// One block. Total potential, then for each uniform u the first row whose
// running potential exceeds u * total (searchsorted(cdf, u, side="right")).
__global__ void __launch_bounds__(1024)
kpp_search_kernel(const double* __restrict__ d2, const double* __restrict__ S, int nb, int64_t n,
                  const double* __restrict__ u, int nc, int64_t* __restrict__ cand,
                  double* __restrict__ tot_out) {
  extern __shared__ double pre[];  // nb + 1 exclusive prefixes of the block sums
  __shared__ double carry;
  const int t = threadIdx.x;
  // sequential prefix in block-sum order (nb <= a few thousand): warp 0,
  // 32 sums at a time with an inclusive warp scan and a carried total
  if (t < 32) {
    double run = 0.0;
    for (int b0 = 0; b0 < nb; b0 += 32) {
      const int b = b0 + t;
      double v = b < nb ? S[b] : 0.0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double w = __shfl_up_sync(kFull, v, o);
        if (t >= o) v = __dadd_rn(v, w);
      }
      if (b < nb) pre[b + 1] = __dadd_rn(run, v);
      run = __dadd_rn(run, __shfl_sync(kFull, v, 31));
    }
    if (t == 0) {
      pre[0] = 0.0;
      carry = run;
      *tot_out = run;
    }
  }
  __syncthreads();
  const double total = carry;
  const int w = t >> 5, lane = t & 31;
  for (int c = w; c < nc; c += 32) {
    const double target = __dmul_rn(u[c], total);
    // last block whose exclusive prefix is <= target
    int lo = 0, hi = nb - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= target) lo = mid; else hi = mid - 1;
    }
    const int64_t r0 = (int64_t)lo * kScanChunk;
    const int rows = (int)((n - r0) < kScanChunk ? (n - r0) : kScanChunk);
    double run = pre[lo];
    int64_t found = r0 + rows - 1;  // rounding at the block's end: its last row
    bool done = false;
    for (int j0 = 0; j0 < rows && !done; j0 += 32) {
      const int j = j0 + lane;
      double v = j < rows ? d2[r0 + j] : 0.0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double x = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v = __dadd_rn(v, x);
      }
      const double cum = __dadd_rn(run, v);
      const unsigned m = __ballot_sync(kFull, j < rows && cum > target);
      if (m) {
        found = r0 + j0 + (__ffs(m) - 1);
        done = true;
      }
      run = __dadd_rn(run, __shfl_sync(kFull, v, 31));
    }
    if (lane == 0) cand[c] = found < n ? found : n - 1;
  }
}

// Scores of kCandRows rows against the nc candidate rows: cd2t[c][i] =
// max(2 - 2 x_i.x_c, 0), and the block's part of each candidate's potential
// sum_i min(d2[i], cd2[i][c]). Thread = 2 rows x NCH candidates; the rows
// pass through shared memory kCandK coordinates at a time (several blocks per
// SM: one block's loads overlap the others' DFMAs), the candidate rows sit
// transposed ([k][candidate], 16-byte pairs) for the whole block.
constexpr int kCandK = 32;
template <int NCH>
__global__ void __launch_bounds__(128)
kpp_cand_kernel(const double* __restrict__ X, int64_t n, int d, const int64_t* __restrict__ cand,
                int nc, const double* __restrict__ d2, int use_d2, double* __restrict__ cd2t,
                double* __restrict__ potp) {
  extern __shared__ __align__(16) double sm[];
  constexpr int NCHP = (NCH + 1) & ~1, CW = 2 * NCHP;
  constexpr int XLD = kCandK + 1;
  constexpr int XS = kCandRows * (XLD > 2 * NCH ? XLD : 2 * NCH);
  double* cs = sm;                  // d x CW
  double* xs = sm + (((size_t)d * CW + 1) & ~(size_t)1);  // kCandRows x XLD
  double* part = xs;                // kCandRows x 2 NCH once the rows are consumed
  (void)XS;
  const int t = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * kCandRows;
  const int rows = (int)((n - row0) < kCandRows ? (n - row0) : kCandRows);
  for (int i = t; i < d * CW; i += 128) {
    const int k = i / CW, w = i - k * CW;
    const int cg = w / NCHP, c = w - cg * NCHP;
    const int cc = cg * NCH + c;
    cs[i] = (c < NCH && cc < nc) ? X[cand[cc] * d + k] : 0.0;
  }
  const int rp = t & 63, cg = t >> 6;
  double acc0[NCHP], acc1[NCHP];
#pragma unroll
  for (int c = 0; c < NCHP; ++c) acc0[c] = acc1[c] = 0.0;
  const double* x0 = xs + rp * XLD;
  const double* x1 = xs + (rp + 64) * XLD;
  for (int k0 = 0; k0 < d; k0 += kCandK) {
    __syncthreads();  // the previous chunk is consumed (and cs is written)
    // asynchronous 8-byte copies: all of a thread's loads of the chunk in flight
#pragma unroll 8
    for (int i = t; i < kCandRows * kCandK; i += 128) {
      const int r = i / kCandK, kk = i - r * kCandK;
      if (r < rows && k0 + kk < d) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&xs[r * XLD + kk]);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst),
                     "l"(&X[(row0 + r) * d + k0 + kk])
                     : "memory");
      } else {
        xs[r * XLD + kk] = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    const int kc = d - k0 < kCandK ? d - k0 : kCandK;
    const double2* cp = (const double2*)(cs + (size_t)k0 * CW + cg * NCHP);
    for (int kk = 0; kk < kc; ++kk) {
      const double a = x0[kk], b = x1[kk];
#pragma unroll
      for (int c2 = 0; c2 < NCHP / 2; ++c2) {
        const double2 cv = cp[(size_t)kk * (CW / 2) + c2];
        acc0[2 * c2] = __fma_rn(a, cv.x, acc0[2 * c2]);
        acc1[2 * c2] = __fma_rn(b, cv.x, acc1[2 * c2]);
        acc0[2 * c2 + 1] = __fma_rn(a, cv.y, acc0[2 * c2 + 1]);
        acc1[2 * c2 + 1] = __fma_rn(b, cv.y, acc1[2 * c2 + 1]);
      }
    }
  }
  __syncthreads();  // the row tile is dead: its space takes the per-row parts
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int cc = cg * NCH + c;
    if (cc < nc) {
      const double v0 = fmax(__dsub_rn(2.0, __dmul_rn(2.0, acc0[c])), 0.0);
      const double v1 = fmax(__dsub_rn(2.0, __dmul_rn(2.0, acc1[c])), 0.0);
      if (rp < rows) cd2t[(int64_t)cc * n + row0 + rp] = v0;
      if (rp + 64 < rows) cd2t[(int64_t)cc * n + row0 + rp + 64] = v1;
      part[rp * 2 * NCH + cc] = rp < rows ? (use_d2 ? fmin(d2[row0 + rp], v0) : v0) : 0.0;
      part[(rp + 64) * 2 * NCH + cc] =
          rp + 64 < rows ? (use_d2 ? fmin(d2[row0 + rp + 64], v1) : v1) : 0.0;
    }
  }
  __syncthreads();
  if (t < nc) {  // rows in order
    double s = 0.0;
    for (int r = 0; r < kCandRows; ++r) s = __dadd_rn(s, part[r * 2 * NCH + t]);
    potp[(int64_t)blockIdx.x * kMaxCand + t] = s;
  }
}

// One block: potential of each candidate (block parts in order, 32 partial
// chains folded by a fixed tree), first arg-min -> chosen[j], column -> bsel.
__global__ void kpp_pick_kernel(const double* __restrict__ potp, int nblk, int nc,
                                const int64_t* __restrict__ cand, int64_t* __restrict__ chosen,
                                int j, int* __restrict__ bsel) {
  __shared__ double pot[kMaxCand];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w < nc) {
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s = __dadd_rn(s, potp[(int64_t)b * kMaxCand + w]);
#pragma unroll
    for (int o = 16; o; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(kFull, s, o));
    if (lane == 0) pot[w] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int b = 0;
    for (int c = 1; c < nc; ++c)
      if (pot[c] < pot[b]) b = c;
    *bsel = b;
    chosen[j] = cand[b];
  }
}

__global__ void set_cand_kernel(int64_t* cand, int64_t* chosen, int64_t first) {
  cand[0] = first;
  chosen[0] = first;
}

// ---- Lloyd update --------------------------------------------------------------
// per-block histogram of list ids: cnt[b][l]
__global__ void __launch_bounds__(kSortRows)
sort_count_kernel(const int32_t* __restrict__ lids, int64_t n, int L, int32_t* __restrict__ cnt) {
  extern __shared__ int32_t h[];
  for (int l = threadIdx.x; l < L; l += kSortRows) h[l] = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * kSortRows + threadIdx.x;
  if (i < n) atomicAdd(&h[lids[i]], 1);
  __syncthreads();
  int32_t* out = cnt + (int64_t)blockIdx.x * L;
  for (int l = threadIdx.x; l < L; l += kSortRows) out[l] = h[l];
}

// thread per list: exclusive scan of its column over the blocks, list total
__global__ void sort_colscan_kernel(int32_t* __restrict__ cnt, int nblk, int L,
                                    int32_t* __restrict__ total) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  int32_t run = 0;
  for (int b = 0; b < nblk; ++b) {
    const int32_t c = cnt[(int64_t)b * L + l];
    cnt[(int64_t)b * L + l] = run;
    run += c;
  }
  total[l] = run;
}

// one block: exclusive scan of the list totals -> start[L + 1]
__global__ void __launch_bounds__(1024)
sort_starts_kernel(const int32_t* __restrict__ total, int L, int32_t* __restrict__ start) {
  __shared__ int32_t buf[1024];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int l0 = 0; l0 < L; l0 += 1024) {
    const int l = l0 + threadIdx.x;
    const int32_t v = l < L ? total[l] : 0;
    buf[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int32_t x = threadIdx.x >= o ? buf[threadIdx.x - o] : 0;
      __syncthreads();
      buf[threadIdx.x] += x;
      __syncthreads();
    }
    if (l < L) start[l] = carry + buf[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += buf[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) start[L] = carry;
}

// one warp per block of rows, 32 rows at a time in order: a row's position is
// its list's start + the block's base + its rank among the block's earlier rows
__global__ void __launch_bounds__(32)
sort_place_kernel(const int32_t* __restrict__ lids, int64_t n, int L,
                  const int32_t* __restrict__ cnt, const int32_t* __restrict__ start,
                  int32_t* __restrict__ order) {
  extern __shared__ int32_t cur[];
  const int lane = threadIdx.x;
  const int32_t* base = cnt + (int64_t)blockIdx.x * L;
  const int64_t row0 = (int64_t)blockIdx.x * kSortRows;
  const int rows = (int)((n - row0) < kSortRows ? (n - row0) : kSortRows);
  // only the lists this block touches need a cursor: initialise lazily
  for (int j0 = 0; j0 < rows; j0 += 32) {
    const int j = j0 + lane;
    if (j < rows) {
      const int l = lids[row0 + j];
      cur[l] = start[l] + base[l];
    }
  }
  __syncwarp();
  for (int j0 = 0; j0 < rows; j0 += 32) {
    const int j = j0 + lane;
    const bool live = j < rows;
    const int l = live ? lids[row0 + j] : -1 - lane;
    const unsigned peers = __match_any_sync(kFull, l);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    int pos = 0;
    if (live) pos = cur[l] + rank;
    __syncwarp();
    if (live && rank == __popc(peers) - 1) cur[l] = pos + 1;
    __syncwarp();
    if (live) order[pos] = (int32_t)(row0 + j);
  }
}

// thread per (list, coordinate): np.add.reduceat's order over the list's rows
// in ascending row order -- the first row plus numpy's pairwise sum of the
// rest (the ufunc's binary-reduce inner loop: out = x[first] + pairwise(x[1:]))
__global__ void __launch_bounds__(128)
seg_sum_kernel(const double* __restrict__ X, int d, const int32_t* __restrict__ order,
               const int32_t* __restrict__ start, double* __restrict__ sums) {
  const int l = blockIdx.x;
  const int s = start[l], e = start[l + 1];
  for (int k = threadIdx.x; k < d; k += 128) {
    double acc = 0.0;
    if (e > s) {
      const double x0 = X[(int64_t)order[s] * d + k];
      acc = e - s > 1 ? __dadd_rn(x0, pw_sum([&](int i) { return X[(int64_t)order[s + 1 + i] * d + k]; },
                                             e - s - 1))
                      : x0;
    }
    sums[(int64_t)l * d + k] = acc;
  }
}

// x_i . C[lids[i]] (the reference's ips[arange(n), a], for the empty-list rule)
__global__ void rowdot_kernel(const double* __restrict__ X, const double* __restrict__ C,
                              const int32_t* __restrict__ lids, int64_t n, int d,
                              double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const double* x = X + i * d;
  const double* c = C + (int64_t)lids[i] * d;
  double s = 0.0;
  for (int k = lane; k < d; k += 32) s = __fma_rn(x[k], c[k], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(kFull, s, o));
  if (lane == 0) out[i] = s;
}

__global__ void lids_equal_kernel(const int32_t* __restrict__ a, const int32_t* __restrict__ b,
                                  int64_t n, int32_t* __restrict__ differ) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && a[i] != b[i]) *differ = 1;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct SeedScratch {
  double *d2, *S, *cd2t, *potp, *u, *tot;
  int64_t* cand;
  int* bsel;
  size_t bytes;
};

static SeedScratch seed_layout(void* base, int64_t n, int k, int nc) {
  SeedScratch s{};
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t o = off;
    off = align256(off + b);
    return (unsigned char*)base + o;
  };
  const int64_t nb = (n + kScanChunk - 1) / kScanChunk;
  const int64_t nblk = (n + kCandRows - 1) / kCandRows;
  s.d2 = (double*)take(sizeof(double) * n);
  s.S = (double*)take(sizeof(double) * nb);
  s.cd2t = (double*)take(sizeof(double) * n * nc);
  s.potp = (double*)take(sizeof(double) * nblk * kMaxCand);
  s.u = (double*)take(sizeof(double) * (size_t)(k > 1 ? k - 1 : 1) * nc);
  s.tot = (double*)take(sizeof(double) * k);
  s.cand = (int64_t*)take(sizeof(int64_t) * kMaxCand);
  s.bsel = (int*)take(sizeof(int) * 4);
  s.bytes = off;
  return s;
}

template <int NCH>
static int launch_cand(const double* X, int64_t n, int d, const int64_t* cand, int nc,
                       const double* d2, int use_d2, double* cd2t, double* potp, cudaStream_t s) {
  constexpr int NCHP = (NCH + 1) & ~1;
  const size_t tile = (size_t)kCandRows * (kCandK + 1 > 2 * NCH ? kCandK + 1 : 2 * NCH);
  const size_t smem = sizeof(double) * (tile + (((size_t)d * 2 * NCHP + 1) & ~(size_t)1));
  auto fn = kpp_cand_kernel<NCH>;
  if (int e = smem_opt_in_dev((const void*)fn, smem)) return e;
  const unsigned grid = (unsigned)((n + kCandRows - 1) / kCandRows);
  fn<<<grid, 128, smem, s>>>(X, n, d, cand, nc, d2, use_d2, cd2t, potp);
  return check_launch("kpp_cand");
}

static int cand_dispatch(int nch, const double* X, int64_t n, int d, const int64_t* cand, int nc,
                         const double* d2, int use_d2, double* cd2t, double* potp,
                         cudaStream_t s) {
  switch (nch) {
    case 1: return launch_cand<1>(X, n, d, cand, nc, d2, use_d2, cd2t, potp, s);
    case 2: return launch_cand<2>(X, n, d, cand, nc, d2, use_d2, cd2t, potp, s);
    case 3: return launch_cand<3>(X, n, d, cand, nc, d2, use_d2, cd2t, potp, s);
    case 4: return launch_cand<4>(X, n, d, cand, nc, d2, use_d2, cd2t, potp, s);
    case 5: return launch_cand<5>(X, n, d, cand, nc, d2, use_d2, cd2t, potp, s);
    case 6: return launch_cand<6>(X, n, d, cand, nc, d2, use_d2, cd2t, potp, s);
    case 7: return launch_cand<7>(X, n, d, cand, nc, d2, use_d2, cd2t, potp, s);
    case 8: return launch_cand<8>(X, n, d, cand, nc, d2, use_d2, cd2t, potp, s);
    default: return launch_cand<9>(X, n, d, cand, nc, d2, use_d2, cd2t, potp, s);
  }
}

}  // namespace km
}  // namespace ivftq

using namespace ivftq;

extern "C" int ivftq_kmeanspp_candidates(int k) {
  int lg = 0;
  while ((2 << lg) <= k) ++lg;  // floor(log2(k))
  return k > 1 ? 2 + lg : 1;
}

extern "C" size_t ivftq_kmeanspp_scratch_bytes(int64_t n, int dim, int k) {
  (void)dim;
  return km::seed_layout(nullptr, n, k, ivftq_kmeanspp_candidates(k)).bytes + 256;
}

extern "C" int ivftq_kmeanspp_seed(const double* X, int64_t n, int dim, int k, int64_t first,
                                   const double* host_uniforms, int64_t* chosen_out,
                                   double* totals_out, void* scratch, size_t scratch_bytes,
                                   void* stream) {
  const int nc = ivftq_kmeanspp_candidates(k);
  if (n < 1 || k < 1 || first < 0 || first >= n || nc > km::kMaxCand) {
    set_error("kmeanspp_seed: bad arguments (n %lld, k %d, first %lld)", (long long)n, k,
              (long long)first);
    return IVFTQ_ERR_ARG;
  }
  if (scratch_bytes < ivftq_kmeanspp_scratch_bytes(n, dim, k)) {
    set_error("kmeanspp_seed: scratch too small");
    return IVFTQ_ERR_SCRATCH;
  }
  cudaStream_t s = (cudaStream_t)stream;
  km::SeedScratch w = km::seed_layout(scratch, n, k, nc);
  const int nb = (int)((n + km::kScanChunk - 1) / km::kScanChunk);
  const int nblk = (int)((n + km::kCandRows - 1) / km::kCandRows);
  if ((size_t)(nb + 1) * sizeof(double) > 200 * 1024) {
    set_error("kmeanspp_seed: n %lld too large for the single-block search", (long long)n);
    return IVFTQ_ERR_UNSUPPORTED;
  }
  if (int e = smem_opt_in_dev((const void*)km::kpp_search_kernel, (size_t)(nb + 1) * sizeof(double)))
    return e;
  if (k > 1)
    IVFTQ_CHECK_CUDA(cudaMemcpyAsync(w.u, host_uniforms, sizeof(double) * (size_t)(k - 1) * nc,
                                     cudaMemcpyHostToDevice, s));
  IVFTQ_CHECK_CUDA(cudaMemsetAsync(totals_out, 0, sizeof(double) * k, s));
  km::set_cand_kernel<<<1, 1, 0, s>>>(w.cand, chosen_out, first);
  if (int e = check_launch("kpp_set")) return e;
  // d2 = distance to the first centre
  if (int e = km::cand_dispatch(1, X, n, dim, w.cand, 1, w.d2, 0, w.cd2t, w.potp, s)) return e;
  km::kpp_update_kernel<<<nb, km::kScanChunk, 0, s>>>(w.d2, w.cd2t, w.bsel, n, 1, w.S);
  if (int e = check_launch("kpp_update")) return e;
  const int nch = (nc + 1) / 2;
  for (int j = 1; j < k; ++j) {
    km::kpp_search_kernel<<<1, 1024, (size_t)(nb + 1) * sizeof(double), s>>>(
        w.d2, w.S, nb, n, w.u + (size_t)(j - 1) * nc, nc, w.cand, totals_out + j);
    if (int e = check_launch("kpp_search")) return e;
    if (int e = km::cand_dispatch(nch, X, n, dim, w.cand, nc, w.d2, 1, w.cd2t, w.potp, s)) return e;
    km::kpp_pick_kernel<<<1, 32 * km::kMaxCand, 0, s>>>(w.potp, nblk, nc, w.cand, chosen_out, j,
                                                         w.bsel);
    if (int e = check_launch("kpp_pick")) return e;
    km::kpp_update_kernel<<<nb, km::kScanChunk, 0, s>>>(w.d2, w.cd2t, w.bsel, n, 0, w.S);
    if (int e = check_launch("kpp_update")) return e;
  }
  return 0;
}

extern "C" size_t ivftq_kmeans_sums_scratch_bytes(int64_t n, int n_lists) {
  const int64_t nblk = (n + km::kSortRows - 1) / km::kSortRows;
  return km::align256(sizeof(int32_t) * (size_t)nblk * n_lists) +
         km::align256(sizeof(int32_t) * (size_t)(n_lists + 1)) + km::align256(sizeof(int32_t) * n) +
         256;
}

extern "C" int ivftq_kmeans_sums(const double* X, const int32_t* list_ids, int64_t n, int dim,
                                 int n_lists, double* sums_out, int32_t* counts_out,
                                 void* scratch, size_t scratch_bytes, void* stream) {
  if (scratch_bytes < ivftq_kmeans_sums_scratch_bytes(n, n_lists)) {
    set_error("kmeans_sums: scratch too small");
    return IVFTQ_ERR_SCRATCH;
  }
  if ((size_t)n_lists * sizeof(int32_t) > 200 * 1024) {
    set_error("kmeans_sums: n_lists %d too large", n_lists);
    return IVFTQ_ERR_UNSUPPORTED;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int nblk = (int)((n + km::kSortRows - 1) / km::kSortRows);
  int32_t* cnt = (int32_t*)scratch;
  int32_t* start = (int32_t*)((unsigned char*)cnt + km::align256(sizeof(int32_t) * (size_t)nblk * n_lists));
  int32_t* order = (int32_t*)((unsigned char*)start + km::align256(sizeof(int32_t) * (size_t)(n_lists + 1)));
  const size_t hs = sizeof(int32_t) * (size_t)n_lists;
  if (int e = smem_opt_in_dev((const void*)km::sort_count_kernel, hs)) return e;
  if (int e = smem_opt_in_dev((const void*)km::sort_place_kernel, hs)) return e;
  km::sort_count_kernel<<<nblk, km::kSortRows, hs, s>>>(list_ids, n, n_lists, cnt);
  if (int e = check_launch("sort_count")) return e;
  km::sort_colscan_kernel<<<(n_lists + 127) / 128, 128, 0, s>>>(cnt, nblk, n_lists, counts_out);
  if (int e = check_launch("sort_colscan")) return e;
  km::sort_starts_kernel<<<1, 1024, 0, s>>>(counts_out, n_lists, start);
  if (int e = check_launch("sort_starts")) return e;
  km::sort_place_kernel<<<nblk, 32, hs, s>>>(list_ids, n, n_lists, cnt, start, order);
  if (int e = check_launch("sort_place")) return e;
  km::seg_sum_kernel<<<n_lists, 128, 0, s>>>(X, dim, order, start, sums_out);
  return check_launch("seg_sum");
}

extern "C" int ivftq_rowdot64(const double* X, const double* C, const int32_t* list_ids, int64_t n,
                            int dim, double* out, void* stream) {
  if (n == 0) return 0;
  km::rowdot_kernel<<<(unsigned)((n + 7) / 8), 256, 0, (cudaStream_t)stream>>>(X, C, list_ids, n,
                                                                                dim, out);
  return check_launch("rowdot");
}

extern "C" int ivftq_lists_differ(const int32_t* a, const int32_t* b, int64_t n, int32_t* differ,
                                  void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  IVFTQ_CHECK_CUDA(cudaMemsetAsync(differ, 0, sizeof(int32_t), s));
  if (n == 0) return 0;
  km::lids_equal_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a, b, n, differ);
  return check_launch("lists_differ");
}
