// Tensor-core list scan (tcgen05) for batched search.
//
// The reference scores every probed list with a per-list f32 GEMM,
// w[members] @ q_rot[queries_of_list].T (index.py:442-458), then sorts all
// candidates per query (index.py:460-483). This kernel keeps that list-major
// structure on the 5th-gen tensor cores:
//
//   * probes are regrouped by list on the device (count / scan / scatter);
//   * a work item is (list l, tile of <=128 queries probing l); persistent CTAs
//     pull items from an atomic counter;
//   * per NV-vector tile of l, one elected thread issues a 1-D TMA bulk copy of
//     the packed codes + norms + ids (the 32-slot interleaved list layout makes
//     a tile one contiguous span), prefetched one tile ahead;
//   * all threads decode codes into fp16 operands in shared memory (UMMA
//     K-major canonical layout) through a 2^(b+1)-entry level table, with the
//     word/field walk unrolled per lcm(fields-per-word, 8) group;
//   * one thread issues tcgen05.mma kind::f16 into a double-buffered TMEM
//     accumulator, D[query][vector] = sum_j qrot_j * T[code_j];
//   * epilogue: warp w reads TMEM lanes 32*(w%4).. (one query per thread) over
//     its half of the tile's columns, filters candidates against the query's
//     running k-th score, appends the few survivors to a per-thread shared
//     buffer and drains it into a register top-K (the drain loop runs to the
//     warp's max survivor count, so rare inserts stay cheap and convergent);
//   * (query, list) winners go to a buffer merged per query afterwards.
//
// Numerics: f32 values are split into fp16 hi + lo with power-of-two scaling
// (T by 2^eT, q by 2^14) and D = Qhi.Thi + Qlo.Thi + Qhi.Tlo accumulated in
// fp32 -- "error-compensated" half precision, ~2^-22 relative per product, the
// same order as the reference's own f32 sgemm. The residual term is then
// D * (2^-(eT+14) * f32(||r||)), the candidate score coarse + (double)res.
#include <climits>
#include <cstdio>

#include "common.cuh"
#include "sm100.cuh"
#include "topk.cuh"

namespace ivftq {

void launch_merge(const double* part_s, const int32_t* part_id, int64_t nq, int n_in, int K,
                  int64_t* ids_out, double* s_out, cudaStream_t s);
int merge_smem_opt_in(int K);

namespace tc {

constexpr int kThreads = 256;  // 8 warps: warp w and w+4 share TMEM lanes, split columns
constexpr int kM = 128;        // queries per tile = MMA M
constexpr int kDrain = 16;     // columns between candidate-buffer drains

struct Params {
  ivftq_store st;
  const double* coarse;    // [nq*n_p] coarse score of pair (q, p)
  const float* qrot;       // [nq*d]
  const double* levels;    // [2^(bits+1)]
  const int32_t* pair_idx; // pair flat index q*n_p+p, grouped by list
  const int32_t* pstart;   // [L+1] first grouped pair of each list
  const int2* items;       // (list, query tile)
  const int32_t* n_items;  // device scalar
  int32_t* counter;        // work counter (zeroed per launch)
  double* part_s;          // [nq*n_p*k]
  int32_t* part_id;
  int n_p, k, d, DP, nbuf;
  float t_scale;    // 2^eT
  float inv_scale;  // 2^-(eT+14)
};

struct Layout {
  uint32_t qhi, qlo, bhi[2], blo[2], codes[2], norms[2], ids[2], nsc[2], vid[2], cand, tab,
      bars, misc, total;
};

__host__ __device__ inline Layout make_layout(int NV, int nbuf, int DP, int W, int C) {
  Layout L{};
  uint32_t off = 0;
  auto take = [&](uint32_t bytes) {
    uint32_t o = off;
    off = (off + bytes + 127u) & ~127u;
    return o;
  };
  L.qhi = take(kM * DP * 2);
  L.qlo = take(kM * DP * 2);
  for (int b = 0; b < 2; ++b) {
    L.bhi[b] = b < nbuf ? take(NV * DP * 2) : L.bhi[0];
    L.blo[b] = b < nbuf ? take(NV * DP * 2) : L.blo[0];
  }
  for (int b = 0; b < 2; ++b) {
    L.codes[b] = take(NV * W * 4);
    L.norms[b] = take(NV * 2);
    L.ids[b] = take(NV * 4);
    L.nsc[b] = take(NV * 4);
    L.vid[b] = take(NV * 4);
  }
  L.cand = take(kDrain * kThreads * 8);
  L.tab = take(C * 4);
  L.bars = take(64);
  L.misc = take(kM * 4 + 64);
  L.total = off;
  return L;
}

__device__ __forceinline__ uint32_t split_pack(float x, uint32_t& lo) {
  __half h = __float2half_rn(x);
  __half l = __float2half_rn(x - __half2float(h));
  lo = (uint32_t)__half_as_ushort(l);
  return (uint32_t)__half_as_ushort(h);
}

// Register top-K with the library key (score desc, id asc).
template <int K>
struct RegTopK {
  float s[K];
  int i[K];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int p = 0; p < K; ++p) { s[p] = -INFINITY; i[p] = INT_MAX; }
  }
  __device__ __forceinline__ bool beats(float v, int id) const {
    return v > s[K - 1] || (v == s[K - 1] && id < i[K - 1]);
  }
  // precondition: beats(v, id)
  __device__ __forceinline__ void insert(float v, int id) {
    bool placed = false;
#pragma unroll
    for (int p = K - 1; p > 0; --p) {
      bool up = !placed && (v > s[p - 1] || (v == s[p - 1] && id < i[p - 1]));
      float ns = up ? s[p - 1] : (placed ? s[p] : v);
      int ni = up ? i[p - 1] : (placed ? i[p] : id);
      s[p] = ns;
      i[p] = ni;
      placed = placed || !up;
    }
    if (!placed) { s[0] = v; i[0] = id; }
  }
};

#define SEL(arr, b) ((b) ? (arr)[1] : (arr)[0])

constexpr int gcd_c(int a, int b) { return b ? gcd_c(b, a % b) : a; }

template <int FB, int KMAX>
__global__ void __launch_bounds__(kThreads, 1) scan_tc_kernel(Params P, int NV) {
  constexpr int C = 1 << FB;
  constexpr int FPW = 32 / FB;
  constexpr uint32_t MASK = (1u << FB) - 1u;
  constexpr int G = FPW * 8 / gcd_c(FPW, 8);  // fields per decode group
  constexpr int GW = G / FPW, GC = G / 8;     // words, 8-field chunks per group
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int W = P.st.words_per_vec, DP = P.DP, d = P.d, NCH = DP / 8;
  const int NG = (DP + G - 1) / G;
  const int nbuf = P.nbuf;
  const uint32_t tmem_cols = 2 * NV < 32 ? 32 : 2 * NV;
  const Layout Lo = make_layout(NV, nbuf, DP, W, C);
  uint32_t* tab = (uint32_t*)(smem + Lo.tab);
  uint64_t* load_bar = (uint64_t*)(smem + Lo.bars);
  uint64_t* mma_bar = load_bar + 2;
  uint32_t* tmem_slot = (uint32_t*)(smem + Lo.misc);
  int* bcast = (int*)(smem + Lo.misc + 16);
  int* qrow = (int*)(smem + Lo.misc + 64);  // pair flat index per query row
  float* cand_v = (float*)(smem + Lo.cand);
  int* cand_c = (int*)(smem + Lo.cand + kDrain * kThreads * 4);

  // ---- one-time setup ---------------------------------------------------------
  for (int c = tid; c < C; c += kThreads) {
    uint32_t lo;
    uint32_t hi = split_pack((float)P.levels[c] * P.t_scale, lo);
    tab[c] = hi | (lo << 16);
  }
  if (warp == 0) sm100::tmem_alloc(tmem_slot, tmem_cols);
  if (tid == 0) {
    sm100::mbar_init(&load_bar[0], 1);
    sm100::mbar_init(&load_bar[1], 1);
    sm100::mbar_init(&mma_bar[0], 1);
    sm100::mbar_init(&mma_bar[1], 1);
    sm100::mbar_fence_init();
  }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = sm100::idesc_f16_f32(kM, NV);
  const uint32_t a_lbo = kM * 16, b_lbo = NV * 16, sbo = 128;
  const uint32_t qhi_a = sm100::smem_u32(smem + Lo.qhi), qlo_a = sm100::smem_u32(smem + Lo.qlo);
  const int n_items = *P.n_items;
  const int row = (warp & 3) * 32 + lane;  // query row == TMEM lane
  const int half = warp >> 2;              // which half of each tile's columns
  uint32_t g = 0;  // tiles processed by this CTA

  for (;;) {
    if (tid == 0) bcast[0] = atomicAdd(P.counter, 1);
    __syncthreads();
    const int item = bcast[0];
    if (item >= n_items) break;
    const int2 it = P.items[item];
    const int l = it.x;
    const int pbase = P.pstart[l] + it.y * kM;
    const int nqt = min(kM, P.pstart[l + 1] - pbase);
    if (tid < kM) qrow[tid] = tid < nqt ? P.pair_idx[pbase + tid] : -1;
    const int size = P.st.list_size[l];
    const int64_t off = P.st.list_offset[l];
    const int ntiles = (size + NV - 1) / NV;

    auto issue_load = [&](int tile, uint32_t sb) {
      int64_t s0 = off + (int64_t)tile * NV;
      uint32_t cb = NV * W * 4, nb = NV * 2, ib = NV * 4;
      sm100::mbar_arrive_expect_tx(&load_bar[sb], cb + nb + ib);
      sm100::bulk_g2s(smem + SEL(Lo.codes, sb), P.st.codes + (s0 >> 5) * W * 32, cb, &load_bar[sb]);
      sm100::bulk_g2s(smem + SEL(Lo.norms, sb), P.st.norms + s0, nb, &load_bar[sb]);
      sm100::bulk_g2s(smem + SEL(Lo.ids, sb), P.st.ids + s0, ib, &load_bar[sb]);
    };
    if (tid == 0 && ntiles > 0) issue_load(0, g & 1);
    __syncthreads();

    // ---- A operand: this tile's rotated queries, split hi/lo, scaled 2^14 ------
    for (int task = tid; task < kM * NCH; task += kThreads) {
      int r = task % kM, c = task / kM;
      int pi = qrow[r];
      uint32_t h[8], lw[8];
      const float* qv = pi >= 0 ? P.qrot + (int64_t)(pi / P.n_p) * d : nullptr;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        int j = c * 8 + e;
        float x = (qv && j < d) ? __ldg(qv + j) * 16384.0f : 0.0f;
        h[e] = split_pack(x, lw[e]);
      }
      uint4 vh = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16),
                            h[6] | (h[7] << 16));
      uint4 vl = make_uint4(lw[0] | (lw[1] << 16), lw[2] | (lw[3] << 16),
                            lw[4] | (lw[5] << 16), lw[6] | (lw[7] << 16));
      uint32_t o = c * (kM * 16) + (r >> 3) * 128 + (r & 7) * 16;
      *(uint4*)(smem + Lo.qhi + o) = vh;
      *(uint4*)(smem + Lo.qlo + o) = vl;
    }

    RegTopK<KMAX> top;
    top.init();

    auto epilogue = [&](uint32_t gt) {
      const uint32_t ab = gt & 1;
      sm100::mbar_wait(&mma_bar[ab], (gt >> 1) & 1);
      sm100::tc_fence_after();
      const float* nsc = (const float*)(smem + SEL(Lo.nsc, ab));
      const int* vid = (const int*)(smem + SEL(Lo.vid, ab));
      const int c0 = half * (NV / 2);
#pragma unroll 1
      for (int cc = 0; cc < NV / 2; cc += 32) {
        uint32_t r[32];
        sm100::tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + ab * NV + c0 + cc, r);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int h2 = 0; h2 < 32; h2 += kDrain) {
          int cnt = 0;
          const float thr = top.s[KMAX - 1];
#pragma unroll
          for (int e = 0; e < kDrain; ++e) {
            const int col = c0 + cc + h2 + e;
            float res = __fmul_rn(__uint_as_float(r[h2 + e]), nsc[col]);
            if (res >= thr) {
              cand_v[cnt * kThreads + tid] = res;
              cand_c[cnt * kThreads + tid] = col;
              ++cnt;
            }
          }
          const int mx = __reduce_max_sync(kFull, cnt);
          for (int i = 0; i < mx; ++i) {
            if (i < cnt) {
              float v = cand_v[i * kThreads + tid];
              int id = vid[cand_c[i * kThreads + tid]];
              if (top.beats(v, id)) top.insert(v, id);
            }
          }
        }
      }
      sm100::tc_fence_before();
    };

    for (int i = 0; i < ntiles; ++i) {
      const uint32_t gt = g + i;
      const uint32_t sb = gt & 1;                       // stage + accumulator buffer
      const uint32_t bb = nbuf == 2 ? (gt & 1) : 0;     // operand buffer
      __syncthreads();  // readers of this iteration's buffers are done
      if (tid == 0 && i + 1 < ntiles) issue_load(i + 1, sb ^ 1);
      sm100::mbar_wait(&load_bar[sb], (gt >> 1) & 1);
      // ---- decode tile i: codes -> fp16 hi/lo operand rows ------------------
      const uint32_t* cw = (const uint32_t*)(smem + SEL(Lo.codes, sb));
      for (int task = tid; task < NV * NG; task += kThreads) {
        const int v = task % NV, gi = task / NV;
        const uint32_t* wv = cw + (v >> 5) * W * 32 + (v & 31);
        uint32_t words[GW];
#pragma unroll
        for (int u = 0; u < GW; ++u) {
          int w = gi * GW + u;
          words[u] = w < W ? wv[w * 32] : 0u;
        }
#pragma unroll
        for (int cc = 0; cc < GC; ++cc) {
          const int c = gi * GC + cc;
          if (c < NCH) {
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int f = cc * 8 + e;  // field within group (compile time)
              uint32_t t = tab[(words[f / FPW] >> ((f % FPW) * FB)) & MASK];
              hi[e] = t & 0xFFFFu;
              lo[e] = t >> 16;
            }
            uint4 vh = make_uint4(hi[0] | (hi[1] << 16), hi[2] | (hi[3] << 16),
                                  hi[4] | (hi[5] << 16), hi[6] | (hi[7] << 16));
            uint4 vl = make_uint4(lo[0] | (lo[1] << 16), lo[2] | (lo[3] << 16),
                                  lo[4] | (lo[5] << 16), lo[6] | (lo[7] << 16));
            uint32_t o = c * (NV * 16) + (v >> 3) * 128 + (v & 7) * 16;
            *(uint4*)(smem + SEL(Lo.bhi, bb) + o) = vh;
            *(uint4*)(smem + SEL(Lo.blo, bb) + o) = vl;
          }
        }
      }
      {
        const int valid = min(NV, size - i * NV);
        const uint16_t* nb = (const uint16_t*)(smem + SEL(Lo.norms, sb));
        const int* ib = (const int*)(smem + SEL(Lo.ids, sb));
        float* nsc = (float*)(smem + SEL(Lo.nsc, sb));
        int* vid = (int*)(smem + SEL(Lo.vid, sb));
        for (int v = tid; v < NV; v += kThreads) {
          nsc[v] = v < valid ? h2f_bits(nb[v]) * P.inv_scale : __int_as_float(0x7fc00000);
          vid[v] = v < valid ? ib[v] : INT_MAX;
        }
      }
      sm100::fence_proxy_async_smem();
      sm100::tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        sm100::tc_fence_after();
        const uint32_t bh = sm100::smem_u32(smem + SEL(Lo.bhi, bb));
        const uint32_t bl = sm100::smem_u32(smem + SEL(Lo.blo, bb));
        const uint32_t dt = tmem + sb * NV;
        const int ks = DP / 16;
        uint32_t acc = 0;
        for (int pass = 0; pass < 3; ++pass) {
          const uint32_t aa = pass == 1 ? qlo_a : qhi_a;
          const uint32_t ba = pass == 2 ? bl : bh;
          for (int s = 0; s < ks; ++s) {
            uint64_t ad = sm100::smem_desc(aa + s * 2 * a_lbo, a_lbo, sbo);
            uint64_t bd = sm100::smem_desc(ba + s * 2 * b_lbo, b_lbo, sbo);
            sm100::mma_f16(dt, ad, bd, idesc, acc);
            acc = 1;
          }
        }
        sm100::mma_commit(&mma_bar[sb]);
      }
      if (nbuf == 2) {
        if (i > 0) epilogue(gt - 1);
      } else {
        epilogue(gt);
      }
    }
    if (nbuf == 2 && ntiles > 0) epilogue(g + ntiles - 1);
    g += ntiles;

    // ---- combine the two column halves, write (query, list) winners -----------
    __syncthreads();
    if (half == 1) {
#pragma unroll
      for (int p = 0; p < KMAX; ++p) {
        cand_v[p * kM + row] = top.s[p];
        cand_c[p * kM + row] = top.i[p];
      }
    }
    __syncthreads();
    if (half == 0 && row < nqt) {
#pragma unroll 1
      for (int p = 0; p < KMAX; ++p) {
        float v = cand_v[p * kM + row];
        int id = cand_c[p * kM + row];
        if (id != INT_MAX && top.beats(v, id)) top.insert(v, id);
      }
      const int pi = qrow[row];
      const double cs = P.coarse[pi];
      const int64_t ob = (int64_t)pi * P.k;
#pragma unroll
      for (int p = 0; p < KMAX; ++p) {
        if (p < P.k) {
          bool have = top.i[p] != INT_MAX;
          P.part_s[ob + p] = have ? cs + (double)top.s[p] : -INFINITY;
          P.part_id[ob + p] = have ? top.i[p] : INT_MAX;
        }
      }
    }
  }
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem, tmem_cols);
}

// ---- probe regrouping: pairs (q, p) bucketed by list ---------------------------
__global__ void pair_count_kernel(const int32_t* __restrict__ probe, int64_t npairs,
                                  int32_t* __restrict__ cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < npairs) atomicAdd(&cnt[probe[i]], 1);
}

// one block: exclusive scans of counts and of query tiles per list
__global__ void __launch_bounds__(1024) pair_scan_kernel(const int32_t* __restrict__ cnt, int L,
                                                         int32_t* __restrict__ pstart,
                                                         int32_t* __restrict__ istart,
                                                         int32_t* __restrict__ n_items) {
  __shared__ int sa[1024], sb[1024];
  const int per = (L + 1023) / 1024;
  const int b0 = threadIdx.x * per;
  int a = 0, t = 0;
  for (int i = b0; i < min(L, b0 + per); ++i) {
    a += cnt[i];
    t += (cnt[i] + kM - 1) / kM;
  }
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = t;
  __syncthreads();
  for (int s = 1; s < 1024; s <<= 1) {
    int va = threadIdx.x >= s ? sa[threadIdx.x - s] : 0;
    int vb = threadIdx.x >= s ? sb[threadIdx.x - s] : 0;
    __syncthreads();
    sa[threadIdx.x] += va;
    sb[threadIdx.x] += vb;
    __syncthreads();
  }
  a = sa[threadIdx.x] - a;  // exclusive
  t = sb[threadIdx.x] - t;
  for (int i = b0; i < min(L, b0 + per); ++i) {
    pstart[i] = a;
    istart[i] = t;
    a += cnt[i];
    t += (cnt[i] + kM - 1) / kM;
  }
  if (threadIdx.x == 1023) {
    pstart[L] = sa[1023];
    istart[L] = sb[1023];
    *n_items = sb[1023];
  }
}

__global__ void pair_scatter_kernel(const int32_t* __restrict__ probe, int64_t npairs,
                                    const int32_t* __restrict__ pstart,
                                    int32_t* __restrict__ cursor, int32_t* __restrict__ pairs) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npairs) return;
  int l = probe[i];
  pairs[pstart[l] + atomicAdd(&cursor[l], 1)] = (int32_t)i;
}

__global__ void items_fill_kernel(const int32_t* __restrict__ cnt,
                                  const int32_t* __restrict__ istart, int L,
                                  int2* __restrict__ items) {
  int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  int t = (cnt[l] + kM - 1) / kM, b = istart[l];
  for (int i = 0; i < t; ++i) items[b + i] = make_int2(l, i);
}

}  // namespace tc
}  // namespace ivftq

using namespace ivftq;
using namespace ivftq::tc;

static int g_num_sms = 0;

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct TcScratch {
  int32_t *cnt, *cursor, *pstart, *istart, *n_items, *counter, *pairs;
  int2* items;
  double* part_s;
  int32_t* part_id;
  size_t bytes;
};

static TcScratch carve_tc(void* base, int64_t nq, int n_p, int L, int k) {
  TcScratch S{};
  size_t off = 0;
  char* b = (char*)base;
  int64_t np = nq * n_p;
  int64_t max_items = np / kM + (np < L ? np : L) + 1;
  auto take = [&](size_t bytes) {
    char* p = b ? b + off : nullptr;
    off += align256(bytes);
    return p;
  };
  S.cnt = (int32_t*)take(4 * (size_t)L);
  S.cursor = (int32_t*)take(4 * (size_t)L);
  S.counter = (int32_t*)take(16);
  S.pstart = (int32_t*)take(4 * (size_t)(L + 1));
  S.istart = (int32_t*)take(4 * (size_t)(L + 1));
  S.n_items = (int32_t*)take(16);
  S.pairs = (int32_t*)take(4 * (size_t)np);
  S.items = (int2*)take(8 * (size_t)max_items);
  S.part_s = (double*)take(8 * (size_t)np * k);
  S.part_id = (int32_t*)take(4 * (size_t)np * k);
  S.bytes = off;
  return S;
}

extern "C" size_t ivftq_scan_tc_scratch_bytes(int64_t nq, int n_p, int n_lists, int depth) {
  return carve_tc(nullptr, nq, n_p, n_lists, depth).bytes + 256;
}

static const size_t kSmemLimit = 227 * 1024;

// Largest vector tile (double-buffered operands first) that fits in shared memory.
static bool pick_tile(int DP, int W, int C, int* nv, int* nbuf) {
  const int cands[4][2] = {{128, 2}, {64, 2}, {64, 1}, {32, 1}};
  for (auto& c : cands) {
    if (make_layout(c[0], c[1], DP, W, C).total + 1024 <= kSmemLimit) {
      *nv = c[0];
      *nbuf = c[1];
      return true;
    }
  }
  return false;
}

extern "C" int ivftq_scan_tc_supported(int dim, int bits, int depth) {
  int fb = field_bits(bits, 1);
  if (fb < 3 || fb > 5 || depth < 1 || depth > 32) return 0;
  int DP = (dim + 15) / 16 * 16;
  int W = words_per_vec(dim, fb);
  int nv, nbuf;
  return pick_tile(DP, W, 1 << fb, &nv, &nbuf) && nv >= 64;
}

template <int FB, int KMAX>
static int launch_tc(const Params& P, int NV, size_t smem, int grid, cudaStream_t s) {
  auto fn = scan_tc_kernel<FB, KMAX>;
  cudaError_t e = cudaFuncSetAttribute((const void*)fn,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    set_error("scan_tc: smem %zu rejected: %s", smem, cudaGetErrorString(e));
    return IVFTQ_ERR_UNSUPPORTED;
  }
  fn<<<grid, kThreads, smem, s>>>(P, NV);
  return check_launch("scan_tc");
}

extern "C" int ivftq_scan_topk_tc(const ivftq_store* st, const int32_t* probe,
                                  const double* coarse, const float* qrot,
                                  const double* levels, int64_t nq, int n_p, int depth,
                                  int64_t* ids_out, double* scores_out, void* scratch,
                                  size_t scratch_bytes, void* stream) {
  if (!ivftq_scan_tc_supported(st->dim, st->bits, depth)) {
    set_error("scan_tc: unsupported (dim %d, bits %d, depth %d)", st->dim, st->bits, depth);
    return IVFTQ_ERR_UNSUPPORTED;
  }
  if (nq == 0) return 0;
  const int L = st->n_lists;
  if (scratch_bytes < ivftq_scan_tc_scratch_bytes(nq, n_p, L, depth)) {
    set_error("scan_tc: scratch too small");
    return IVFTQ_ERR_SCRATCH;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  TcScratch S = carve_tc(scratch, nq, n_p, L, depth);
  int64_t np = nq * n_p;
  IVFTQ_CHECK_CUDA(cudaMemsetAsync(S.cnt, 0, (char*)S.pstart - (char*)S.cnt, s));
  unsigned gp = (unsigned)((np + 255) / 256);
  pair_count_kernel<<<gp, 256, 0, s>>>(probe, np, S.cnt);
  if (int e = check_launch("pair_count")) return e;
  pair_scan_kernel<<<1, 1024, 0, s>>>(S.cnt, L, S.pstart, S.istart, S.n_items);
  if (int e = check_launch("pair_scan")) return e;
  pair_scatter_kernel<<<gp, 256, 0, s>>>(probe, np, S.pstart, S.cursor, S.pairs);
  if (int e = check_launch("pair_scatter")) return e;
  items_fill_kernel<<<(L + 255) / 256, 256, 0, s>>>(S.cnt, S.istart, L, S.items);
  if (int e = check_launch("items_fill")) return e;

  const int fb = st->field_bits, C = 1 << fb;
  const int DP = (st->dim + 15) / 16 * 16;
  int NV = 0, nbuf = 0;
  pick_tile(DP, st->words_per_vec, C, &NV, &nbuf);
  Params P{};
  P.st = *st;
  P.coarse = coarse;
  P.qrot = qrot;
  P.levels = levels;
  P.pair_idx = S.pairs;
  P.pstart = S.pstart;
  P.items = S.items;
  P.n_items = S.n_items;
  P.counter = S.counter;
  P.part_s = S.part_s;
  P.part_id = S.part_id;
  P.n_p = n_p;
  P.k = depth;
  P.d = st->dim;
  P.DP = DP;
  P.nbuf = nbuf;
  // Every Lloyd-Max level satisfies |T| < 5/sqrt(d) < 4, so 2^12 keeps the
  // scaled table below 2^14 and its hi/lo halves in the fp16 normal range.
  const int eT = 12;
  P.t_scale = ldexpf(1.0f, eT);
  P.inv_scale = ldexpf(1.0f, -(eT + 14));
  size_t smem = make_layout(NV, nbuf, DP, st->words_per_vec, C).total + 1024;
  int grid = g_num_sms;
  int rc;
#define TC_CASE(FBV)                                                              \
  if (fb == FBV) {                                                                \
    rc = depth <= 10 ? launch_tc<FBV, 10>(P, NV, smem, grid, s)                   \
                     : launch_tc<FBV, 32>(P, NV, smem, grid, s);                  \
  }
  TC_CASE(3) else TC_CASE(4) else TC_CASE(5) else {
    set_error("scan_tc: field width %d", fb);
    return IVFTQ_ERR_UNSUPPORTED;
  }
#undef TC_CASE
  if (rc) return rc;
  if (int e = merge_smem_opt_in(depth)) return e;
  launch_merge(S.part_s, S.part_id, nq, n_p * depth, depth, ids_out, scores_out, s);
  return check_launch("merge");
}
