// Tensor-core list scan (tcgen05) for batched search, warp-specialised.
//
// The reference scores every probed list with a per-list f32 GEMM,
// w[members] @ q_rot[queries_of_list].T (index.py:442-458), then sorts all
// candidates per query (index.py:460-483). This kernel keeps that list-major
// structure on the 5th-gen tensor cores:
//
//   * probes are regrouped by list on the device (count / scan / scatter);
//     a work item is (list l, tile of <=128 queries probing l);
//   * persistent CTAs, one per SM (23 warps), run a pipeline over the stream
//     of NV-vector tiles (NV = 128, or 64 for wide d) of their items, handing
//     off through mbarrier rings:
//       - scheduler warp: pulls items from an atomic counter and prepares an
//         item record (list span, query rows, coarse scores, initial bounds)
//         up to two items ahead, prefetching the rows' A operands into L2;
//       - producer warp: per tile, query rows + fresh pruning bounds into a
//         stage slot, then one lane issues 1-D TMA bulk copies of the tile's
//         packed codes, norms and ids (the 32-slot interleaved list layout
//         makes each a contiguous span);
//       - 4 A-builder warps (one per TMEM lane quadrant): the item's rotated
//         queries as fp16 hi/lo into TMEM (the MMA A operand), one item ahead;
//       - 8 decoder warps: codes -> B operand (UMMA K-major canonical layout,
//         fp16 hi/lo) through a 2^(b+1)-entry level table, double-buffered;
//       - MMA warp: elected lane issues tcgen05.mma kind::f16 (3 products per
//         K step, see below) into a TMEM accumulator ring D[query][vector];
//       - 8 epilogue warps: warp w reads TMEM lanes 32*(w%4).. (one query per
//         thread) over half of the tile's columns, filters 16-column windows
//         against the pair's running k-th / the other half's / the query's
//         global bound, and inserts survivors into a branch-free register
//         top-K of 64-bit (score, ~id) keys; at an item's last tile each half
//         appends its entries above the global bound to the query's buffer,
//         which a second kernel merges per query.
//
// Numerics: f32 values are split into fp16 hi + lo with power-of-two scaling
// (T by 2^eT, q by 2^14) and D = Qhi.Thi + Qlo.Thi + Qhi.Tlo accumulated in
// fp32 -- "error-compensated" half precision, ~2^-22 relative per product, the
// same order as the reference's own f32 sgemm. The residual term is then
// D * (2^-(eT+14) * f32(||r||)), the candidate score coarse + (double)res.
#include <climits>
#include <string>
#include <cstdlib>
#include <cstdio>

#include "common.cuh"
#include "sm100.cuh"
#include "topk.cuh"

namespace ivftq {

void launch_merge(const double* part_s, const int32_t* part_id, int64_t nq, int n_in, int K,
                  int64_t* ids_out, double* s_out, cudaStream_t s,
                  const int32_t* counts = nullptr);
int merge_smem_opt_in(int K);
// scan_vq.cu: the vectors x queries scan (d <= 128)
bool scan_vq_supported(int dim, int field_bits_, int depth);
int launch_scan_vq(const ivftq_store* st, const double* coarse, const double* levels,
                   const int32_t* pairs, const int32_t* pstart, const int2* items,
                   const int32_t* n_items, int32_t* counter, double* part_s, int32_t* part_id,
                   int32_t* qcnt, long long* thr_key, const uint32_t* q_hi, const uint32_t* q_lo,
                   int n_p, int depth, int qcap, cudaStream_t s);

namespace tc {

constexpr int kM = 128;          // queries per item = MMA M
constexpr int kProdWarp = 0;     // producer (TMA + control records)
constexpr int kMmaWarp = 1;      // tcgen05.mma issuer, owns TMEM
constexpr int kDecWarp0 = 2;     // decoder warps 2..9
#ifndef IVFTQ_DEC_WARPS
#define IVFTQ_DEC_WARPS 8
#endif
#ifndef IVFTQ_MID_PUBLISH
#define IVFTQ_MID_PUBLISH 1  // publish the pair K-th to the global bound per tile (C2 n_p=16 scan -1 %)
#endif
#ifndef IVFTQ_EPI_LD
#define IVFTQ_EPI_LD 16  // accumulator columns per epilogue TMEM load (16: C2 step 1.17 -> 1.16 ms)
#endif
constexpr int kDecWarps = IVFTQ_DEC_WARPS;
constexpr int kEpiWarp0 = kDecWarp0 + kDecWarps;  // epilogue warps (8)
constexpr int kEpiWarps = 8;
constexpr int kSchedWarp = kEpiWarp0 + kEpiWarps;  // 18: item scheduler
constexpr int kAbWarp0 = kSchedWarp + 1;             // 19..22: A-operand builders
constexpr int kThreads = 32 * (kAbWarp0 + 4);        // 736
#ifndef IVFTQ_ITEM_SLOTS
#define IVFTQ_ITEM_SLOTS 2
#endif
#ifndef IVFTQ_META
#define IVFTQ_META 4
#endif
constexpr int kItemSlots = IVFTQ_ITEM_SLOTS;  // item-record ring (scheduler -> producer)
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kDrain = 16;       // columns per TMEM load / candidate drain
constexpr int kNS = 4;           // stage ring depth (power of two)
constexpr int kMeta = IVFTQ_META;  // tile-record ring depth (power of two)
// mbarrier slots (8 bytes each): st_full[8] st_empty[8] op_full[2] op_empty[2]
// a_full[2] a_empty[2] meta_full[kMeta] meta_empty[kMeta] it_full[kItemSlots]
// it_empty[kItemSlots] acc_full[kAccMax] acc_empty[kAccMax]
constexpr int kBarMetaF = 24, kBarMetaE = kBarMetaF + kMeta, kBarItF = kBarMetaE + kMeta,
              kBarItE = kBarItF + kItemSlots, kBarAccF = kBarItE + kItemSlots,
              kBarAccE = kBarAccF + 4, kBarCount = kBarAccE + 4;
constexpr int kAccMax = 4;       // TMEM accumulator ring depth bound (power of two)
// Tile shapes (vectors per tile = MMA N, accumulator ring depth): 128 x 2 when
// shared memory and TMEM allow, else 64 x 4. TMEM budget: nAcc accumulators of
// NV columns + nA A-operand buffers of DP columns <= 512.
constexpr int kMaxDim = 256;


// control record of one tile in a stage slot
struct Ctrl {
  int list;    // -1 = stop
  int tile;    // tile index within the item
  int ntiles;
  int valid;   // vectors of this tile that exist
  int nqt;     // queries in the item
  int pad[3];
};

// one work item as the scheduler warp prepares it for the producer
struct ItemRec {
  int list;    // -1 = stop
  int nqt;
  int size;
  int ntiles;
  long long off;
  long long pad;
  int prow[kM];       // pair index of each query row (-1 = padding)
  float bnd[kM];      // residual-space pruning bound at fetch time
  double cs[kM];      // coarse score of each pair
};

struct Layout {
  uint32_t items, item_bytes;
  uint32_t bhi[2], blo[2], stage, stage_bytes, st_codes, st_norms, st_ids, st_ctrl,
      st_qrow, meta0, meta_bytes, m_nsc, m_ids, m_qrow, cand, tab, thr, bars, misc, total;
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) & ~(a - 1); }

// candidate-buffer entries per epilogue thread: a drain window, or a whole
// top-K list when the two column halves merge at the end of an item

__host__ __device__ inline Layout make_layout(int NV, int NS, int DP, int W, int C, int KMAX) {
  Layout L{};
  uint32_t off = 0;
  auto take = [&](uint32_t bytes) {
    uint32_t o = off;
    off = align_up(off + bytes, 128u);
    return o;
  };
  for (int b = 0; b < 2; ++b) {
    L.bhi[b] = take(NV * DP * 2);
    L.blo[b] = take(NV * DP * 2);
  }
  // stage slot: codes | norms | ids | ctrl | qrow  (each 128-aligned)
  L.st_codes = 0;
  L.st_norms = align_up(NV * (uint32_t)W * 4, 128);
  L.st_ids = L.st_norms + align_up(NV * 2, 128);
  L.st_ctrl = L.st_ids + align_up(NV * 4, 128);
  L.st_qrow = L.st_ctrl + 128;
  L.stage_bytes = L.st_qrow + kM * 8;  // query rows (int) + pruning bounds (float)
  L.stage = take(L.stage_bytes * NS);
  // per-accumulator-buffer epilogue record: ctrl | nsc | ids | qrow
  L.m_nsc = 128;
  L.m_ids = L.m_nsc + align_up(NV * 4, 128);
  L.m_qrow = L.m_ids + align_up(NV * 4, 128);
  L.meta_bytes = align_up(L.m_qrow + kM * 8, 128);
  L.meta0 = take(L.meta_bytes * kMeta);
  L.cand = 0;
  L.tab = take(C * 4);
  L.thr = take(2 * kM * 8);  // per half and row: (item tag << 32) | f32 k-th score
  L.item_bytes = align_up(sizeof(ItemRec), 128);
  L.items = take(L.item_bytes * kItemSlots);
  L.bars = take(8 * kBarCount);
  L.misc = take(64);
  L.total = off;
  return L;
}

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
  double* part_s;          // [nq][2*n_p*k] per-query candidate buffer
  int32_t* part_id;
  int32_t* qcnt;           // [nq] candidates appended per query
  long long* thr_key;      // [nq] order-preserving key of a lower bound on the k-th score
  long long* trace;        // debug timeline of CTA 0 (IVFTQ_TRACE), else null
  const uint32_t* q_hi;    // [nq][DP/2] rotated query rows, fp16 hi halves (x 2^14), packed pairs
  const uint32_t* q_lo;    // [nq][DP/2] matching lo halves
  int n_p, k, d, DP, NV, NS;
  int qcap;         // candidate buffer capacity per query (2*n_p*k)
  int nAcc;         // TMEM accumulator ring depth (<= kAccMax)
  int nA;           // A-operand buffers in TMEM (2 when they fit: next item's
                    // queries are written while the current item's MMAs run)
  float t_scale;    // 2^eT
  float inv_scale;  // 2^-(eT+14)
  Layout lo;        // shared-memory carve-up, computed once on the host
};

__device__ __forceinline__ uint32_t split_pack(float x, uint32_t& lo) {
  __half h = __float2half_rn(x);
  __half l = __float2half_rn(x - __half2float(h));
  lo = (uint32_t)__half_as_ushort(l);
  return (uint32_t)__half_as_ushort(h);
}

// Register top-K over 64-bit keys that encode the library order (score desc,
// id asc): high word = order-preserving bits of the f32 residual term (one
// pair has one coarse score, so the f64 candidate score is monotone in it;
// -0.0 is folded onto +0.0 so the tie goes to the id), low word = ~id. Key 0
// is "empty" and sorts below every real candidate (NaN never reaches insert).
__device__ __forceinline__ uint64_t cand_key(float v, int id) {
  uint32_t b = __float_as_uint(v + 0.0f);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((uint64_t)b << 32) | (uint32_t)~(uint32_t)id;
}
__device__ __forceinline__ float key_score(uint64_t k) {
  const uint32_t o = (uint32_t)(k >> 32);
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
__device__ __forceinline__ int key_id(uint64_t k) { return (int)~(uint32_t)k; }

// v[j] for a lane-varying j without local memory: a 4-level select tree
__device__ __forceinline__ float pick16(const float (&v)[16], int j) {
  float a[8], b[4], c[2];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (j & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = (j & 2) ? a[2 * i + 1] : a[2 * i];
#pragma unroll
  for (int i = 0; i < 2; ++i) c[i] = (j & 4) ? b[2 * i + 1] : b[2 * i];
  return (j & 8) ? c[1] : c[0];
}

template <int K>
struct RegTopK {
  uint64_t k[K];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int p = 0; p < K; ++p) k[p] = 0;
  }
  __device__ __forceinline__ float kth() const {
    return k[K - 1] ? key_score(k[K - 1]) : -INFINITY;
  }
  // Branch-free and chain-free: every position compares against the old list
  // at once (g is monotone in p because the list is sorted), so an insert is
  // K compares + 2K selects at depth ~3; a key that does not beat k[K-1]
  // (including 0) leaves the list unchanged, so callers need no branch.
  __device__ __forceinline__ void insert(uint64_t key) {
    bool g[K];
#pragma unroll
    for (int p = 0; p < K; ++p) g[p] = key > k[p];
#pragma unroll
    for (int p = K - 1; p > 0; --p) k[p] = g[p] ? (g[p - 1] ? k[p - 1] : key) : k[p];
    k[0] = g[0] ? key : k[0];
  }
};

constexpr int gcd_c(int a, int b) { return b ? gcd_c(b, a % b) : a; }

constexpr int kTraceTiles = 4096;
constexpr int kSeedP = 4;  // seed slots per query / 32 (IVFTQ_SEED_P overrides): 128 slots
                           // (C3 n_p=32: scan 1.46 -> 1.37 ms, 5.32 -> 5.45 M QPS; C2 neutral)
// Timeline instrumentation (CTA 0, lane 0 of the role's first warp), compiled
// in only for the trace build (make trace -> libivftq_b200_trace.so, used with
// IVFTQ_LIB=... and IVFTQ_TRACE=<file>): even untaken, the checks cost ~5 %.
#ifdef IVFTQ_TRACE_BUILD
#define TRACE(slot)                                                              \
  do {                                                                           \
    if (P.trace && blockIdx.x == 0 && lane == 0 && t < (uint32_t)kTraceTiles)    \
      P.trace[t * 8 + (slot)] = clock64();                                       \
  } while (0)
// epilogue-internal timeline (warp kEpiWarp0)
#define ETRACE(slot, val)                                                        \
  do {                                                                           \
    if (P.trace && blockIdx.x == 0 && lane == 0 && warp == kEpiWarp0 &&          \
        t < (uint32_t)kTraceTiles)                                               \
      P.trace[8 * kTraceTiles + t * 8 + (slot)] = (val);                         \
  } while (0)
// decoder-internal timeline (warp kDecWarp0)
#define DTRACE(slot)                                                             \
  do {                                                                           \
    if (P.trace && blockIdx.x == 0 && lane == 0 && warp == kDecWarp0 &&          \
        t < (uint32_t)kTraceTiles)                                               \
      P.trace[16 * kTraceTiles + t * 8 + (slot)] = clock64();                    \
  } while (0)
#else
#define TRACE(slot) do {} while (0)
#define ETRACE(slot, val) do {} while (0)
#define DTRACE(slot) do {} while (0)
#endif

// f64 <-> int64 key preserving order, so atomicMax works on scores
__device__ __forceinline__ long long dkey(double x) {
  long long b = __double_as_longlong(x);
  return b >= 0 ? b : (b ^ 0x7FFFFFFFFFFFFFFFLL);
}
__device__ __forceinline__ double dkey_inv(long long k) {
  return __longlong_as_double(k >= 0 ? k : (k ^ 0x7FFFFFFFFFFFFFFFLL));
}

// Residual-space pruning bound for pair `pi`: a candidate with residual term
// res < bound has coarse + res < (known lower bound on the query's k-th final
// score) strictly -- the 1e-12 margin dominates the f64 rounding of
// coarse + res and nextafterf undoes the f32 conversion's rounding -- so it
// can never enter the query's top-k, ties included.
__device__ __forceinline__ float prune_bound(long long key, double coarse) {
  const double thr = dkey_inv(key);
  if (!(thr > -INFINITY)) return -INFINITY;
  const float b = (float)(thr - coarse - 1e-12);
  return nextafterf(b, -INFINITY);
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sm100::smem_u32(bar)) : "memory");
}
// 32 lanes x 16 consecutive 32-bit TMEM columns
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

template <int FB, int KMAX>
__global__ void __launch_bounds__(kThreads, 1) scan_tc_kernel(Params P) {
  constexpr int C = 1 << FB;
  constexpr int FPW = 32 / FB;
  constexpr uint32_t MASK = (1u << FB) - 1u;
  constexpr int G = FPW * 8 / gcd_c(FPW, 8);  // fields per decode group
  constexpr int GW = G / FPW, GC = G / 8;     // words, 8-field chunks per group
  extern __shared__ __align__(1024) unsigned char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NV = P.NV;
  constexpr int NS = kNS;
  const int W = P.st.words_per_vec, DP = P.DP, d = P.d, NCH = DP / 8;
  // TMEM columns: kAcc accumulators of NV columns, then the A operand
  // (Qhi, Qlo: DP/2 columns each)
  const int nAcc = P.nAcc;
  const uint32_t a_col = nAcc * NV;
  const uint32_t need = a_col + P.nA * DP;
  const uint32_t tmem_cols = need <= 32 ? 32u : need <= 64 ? 64u : need <= 128 ? 128u : need <= 256 ? 256u : 512u;
  const Layout& Lo = P.lo;  // kernel-parameter space: no per-use recomputation
  // level table in static shared memory: lookups address it as reg + symbol
  __shared__ __align__(4 * C) uint32_t s_tab[C];  // aligned to its size: base | offset == base + offset
  uint32_t* tab = s_tab;
  uint64_t* bars = (uint64_t*)(smem + Lo.bars);
  uint64_t* st_full = bars;            // [NS] producer -> decoders/epilogue (TMA tx)
  uint64_t* st_empty = bars + 8;       // [NS] decoders + epilogue -> producer
  uint64_t* op_full = bars + 16;       // [2] decoders -> MMA
  uint64_t* op_empty = bars + 18;      // [2] MMA commit -> decoders
  uint64_t* acc_full = bars + kBarAccF;   // [nAcc] MMA commit -> epilogue
  uint64_t* acc_empty = bars + kBarAccE;  // [nAcc] epilogue -> MMA
  uint64_t* a_full = bars + 20;        // [nA] decoders -> MMA (A operand built)
  uint64_t* a_empty = bars + 22;       // [nA] MMA commit -> decoders (A operand free)
  uint64_t* meta_full = bars + kBarMetaF;   // [kMeta] decoders -> MMA/epilogue (tile record)
  uint64_t* meta_empty = bars + kBarMetaE;  // [kMeta] epilogue -> decoders
  uint64_t* it_full = bars + kBarItF;       // [kItemSlots] scheduler -> producer
  uint64_t* it_empty = bars + kBarItE;      // [kItemSlots] producer -> scheduler
  uint32_t* tmem_slot = (uint32_t*)(smem + Lo.misc);
  for (int i = tid; i < 2 * kM; i += kThreads) ((unsigned long long*)(smem + Lo.thr))[i] = 0ull;
  auto meta = [&](int m) { return smem + Lo.meta0 + (uint32_t)m * Lo.meta_bytes; };
  auto stage = [&](int s) { return smem + Lo.stage + (uint32_t)s * Lo.stage_bytes; };

  // ---- one-time setup ---------------------------------------------------------
  for (int c = tid; c < C; c += kThreads) {
    uint32_t lo;
    uint32_t hi = split_pack((float)P.levels[c] * P.t_scale, lo);
    tab[c] = hi | (lo << 16);
  }
  if (warp == kMmaWarp) sm100::tmem_alloc(tmem_slot, tmem_cols);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      sm100::mbar_init(&st_full[s], 1);
      sm100::mbar_init(&st_empty[s], kDecWarps);
    }
    for (int b = 0; b < 2; ++b) {
      sm100::mbar_init(&op_full[b], kDecWarps);
      sm100::mbar_init(&op_empty[b], 1);
    }
    for (int b = 0; b < kAccMax; ++b) {
      sm100::mbar_init(&acc_full[b], 1);
      sm100::mbar_init(&acc_empty[b], kEpiWarps);
    }
    for (int m = 0; m < kMeta; ++m) {
      sm100::mbar_init(&meta_full[m], kDecWarps);
      sm100::mbar_init(&meta_empty[m], kEpiWarps);
    }
    for (int b = 0; b < 2; ++b) {
      sm100::mbar_init(&a_full[b], 4);
      sm100::mbar_init(&a_empty[b], 1);
    }
    for (int b = 0; b < kItemSlots; ++b) {
      sm100::mbar_init(&it_full[b], 1);
      sm100::mbar_init(&it_empty[b], 5);  // producer + 4 A builders
    }
    sm100::mbar_fence_init();
  }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kProdWarp) {
    // ================= producer =================================================
    // Per tile: query rows + fresh pruning bounds into the stage slot, then one
    // lane issues the TMA bulk copies. Item metadata arrives ready-made from
    // the scheduler warp; the bounds' global loads for tile i+1 are issued
    // during tile i, so no global latency sits on this warp's per-tile path.
    uint32_t t = 0, j = 0;
    for (;;) {
      const int slot = j % kItemSlots;
      sm100::mbar_wait_sleep<512>(&it_full[slot], (j / kItemSlots) & 1);
      const ItemRec* rec = (const ItemRec*)(smem + Lo.items + slot * Lo.item_bytes);
      const int l = rec->list;
      if (l < 0) {
        const int s = t % NS;
        if (t >= (uint32_t)NS) sm100::mbar_wait_sleep<512>(&st_empty[s], ((t / NS) - 1) & 1);
        if (lane == 0) {
          Ctrl* c = (Ctrl*)(stage(s) + Lo.st_ctrl);
          c->list = -1;
          mbar_arrive(&st_full[s]);
        }
        break;
      }
      const int nqt = rec->nqt, size = rec->size, ntiles = rec->ntiles;
      const int64_t off = rec->off;
      int prow[kM / 32];
      double pcs[kM / 32];
      float pb[kM / 32];
#pragma unroll
      for (int q = 0; q < kM / 32; ++q) {
        prow[q] = rec->prow[q * 32 + lane];
        pcs[q] = rec->cs[q * 32 + lane];
        pb[q] = rec->bnd[q * 32 + lane];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&it_empty[slot]);
      ++j;
      long long kq[kM / 32];
      for (int i = 0; i < ntiles; ++i, ++t) {
        if (i > 0) {
#pragma unroll
          for (int q = 0; q < kM / 32; ++q)
            pb[q] = prow[q] >= 0 ? fmaxf(pb[q], prune_bound(kq[q], pcs[q])) : -INFINITY;
        }
        if (i + 1 < ntiles) {  // bounds for the next tile: in flight during this one
#pragma unroll
          for (int q = 0; q < kM / 32; ++q)
            kq[q] = prow[q] >= 0 ? *(volatile const long long*)&P.thr_key[prow[q] / P.n_p]
                                 : LLONG_MIN;
        }
        const int s = t % NS;
        if (t >= (uint32_t)NS) sm100::mbar_wait_sleep<512>(&st_empty[s], ((t / NS) - 1) & 1);
        unsigned char* sp = stage(s);
        int* qrow = (int*)(sp + Lo.st_qrow);
        float* qb = (float*)(qrow + kM);
#pragma unroll
        for (int q = 0; q < kM / 32; ++q) {
          qrow[q * 32 + lane] = prow[q];
          qb[q * 32 + lane] = pb[q];
        }
        if (lane == 0) {
          Ctrl* c = (Ctrl*)(sp + Lo.st_ctrl);
          c->list = l;
          c->tile = i;
          c->ntiles = ntiles;
          c->valid = min(NV, size - i * NV);
          c->nqt = nqt;
        }
        __syncwarp();
        if (lane == 0) {
          const int64_t s0 = off + (int64_t)i * NV;
          const uint32_t cb = NV * W * 4, nb = NV * 2, ib = NV * 4;
          sm100::mbar_arrive_expect_tx(&st_full[s], cb + nb + ib);
          sm100::bulk_g2s(sp + Lo.st_codes, P.st.codes + (s0 >> 5) * W * 32, cb, &st_full[s]);
          sm100::bulk_g2s(sp + Lo.st_norms, P.st.norms + s0, nb, &st_full[s]);
          sm100::bulk_g2s(sp + Lo.st_ids, P.st.ids + s0, ib, &st_full[s]);
          TRACE(0);
        }
      }
    }
  } else if (warp == kSchedWarp) {
    // ================= item scheduler ==========================================
    // Pulls work items from the global counter and resolves everything the
    // producer needs per item (list span, query rows, coarse scores, initial
    // bounds; L2 prefetch of the rows' A operands) up to kItemSlots items ahead.
    const int n_items = *P.n_items;
    uint32_t j = 0;
    for (;;) {
      int item = 0;
      if (lane == 0) item = atomicAdd(P.counter, 1);
      item = __shfl_sync(kFull, item, 0);
      const int slot = j % kItemSlots;
      ItemRec* rec = (ItemRec*)(smem + Lo.items + slot * Lo.item_bytes);
      if (item >= n_items) {
        if (j >= (uint32_t)kItemSlots) sm100::mbar_wait_sleep<512>(&it_empty[slot], ((j / kItemSlots) - 1) & 1);
        if (lane == 0) {
          rec->list = -1;
          mbar_arrive(&it_full[slot]);
        }
        break;
      }
      const int2 it = P.items[item];
      const int l = it.x;
      const int pbase = P.pstart[l] + it.y * kM;
      const int nqt = min(kM, P.pstart[l + 1] - pbase);
      const int size = P.st.list_size[l];
      const int64_t off = P.st.list_offset[l];
      const int ntiles = (size + NV - 1) / NV;
      if (ntiles == 0) continue;  // empty list: contributes no candidates
      int prow[kM / 32];
      double pcs[kM / 32];
      long long kq[kM / 32];
#pragma unroll
      for (int q = 0; q < kM / 32; ++q) {
        const int r = q * 32 + lane;
        prow[q] = r < nqt ? P.pair_idx[pbase + r] : -1;
      }
#pragma unroll
      for (int q = 0; q < kM / 32; ++q) {
        pcs[q] = prow[q] >= 0 ? P.coarse[prow[q]] : 0.0;
        kq[q] = prow[q] >= 0 ? *(volatile const long long*)&P.thr_key[prow[q] / P.n_p] : LLONG_MIN;
        if (prow[q] >= 0) {  // the decoders read these A rows at the item's first tile
          const int64_t qo = (int64_t)(prow[q] / P.n_p) * (DP / 2);
          for (int b = 0; b < DP * 2; b += 128) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(P.q_hi + qo) + b));
            asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(P.q_lo + qo) + b));
          }
        }
      }
      if (j >= (uint32_t)kItemSlots) sm100::mbar_wait_sleep<512>(&it_empty[slot], ((j / kItemSlots) - 1) & 1);
#pragma unroll
      for (int q = 0; q < kM / 32; ++q) {
        rec->prow[q * 32 + lane] = prow[q];
        rec->cs[q * 32 + lane] = pcs[q];
        rec->bnd[q * 32 + lane] = prow[q] >= 0 ? prune_bound(kq[q], pcs[q]) : -INFINITY;
      }
      if (lane == 0) {
        rec->list = l;
        rec->nqt = nqt;
        rec->size = size;
        rec->ntiles = ntiles;
        rec->off = off;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&it_full[slot]);
      ++j;
    }
  } else if (warp >= kAbWarp0) {
    // ================= A-operand builders ========================================
    // One item ahead of the MMA (A is double-buffered in TMEM when it fits):
    // warp w writes TMEM lane quadrant w%4 -- the item's query rows, fp16 hi in
    // the first DP/2 columns and lo in the next, straight from the pre-split
    // rows -- once the MMAs of the item that last used the buffer are done.
    const int quad = warp & 3;
    uint32_t j = 0;
    for (;;) {
      const int slot = j % kItemSlots;
      sm100::mbar_wait_sleep<512>(&it_full[slot], (j / kItemSlots) & 1);
      const ItemRec* rec = (const ItemRec*)(smem + Lo.items + slot * Lo.item_bytes);
      const int l = rec->list;
      const int pi = l >= 0 ? rec->prow[quad * 32 + lane] : -1;
      __syncwarp();
      if (lane == 0) mbar_arrive(&it_empty[slot]);
      if (l < 0) break;
      const uint32_t ab_ = j % P.nA;
      if (j >= (uint32_t)P.nA) sm100::mbar_wait_sleep<512>(&a_empty[ab_], ((j / P.nA) - 1) & 1);
      sm100::tc_fence_after();
      const int64_t qo = (int64_t)(pi >= 0 ? pi / P.n_p : 0) * (DP / 2);
#pragma unroll 1
      for (int part = 0; part < 2; ++part) {
        const uint4* src = (const uint4*)((part ? P.q_lo : P.q_hi) + qo);
        const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + a_col + ab_ * DP + part * (DP / 2);
#pragma unroll 1
        for (int c16 = 0; c16 < DP / 2; c16 += 64) {
          uint32_t v[4][16];
#pragma unroll
          for (int hh = 0; hh < 4; ++hh)
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              const bool ok = pi >= 0 && c16 + hh * 16 < DP / 2;
              const uint4 w4 = ok ? __ldg(src + (c16 + hh * 16) / 4 + x) : make_uint4(0, 0, 0, 0);
              v[hh][4 * x] = w4.x;
              v[hh][4 * x + 1] = w4.y;
              v[hh][4 * x + 2] = w4.z;
              v[hh][4 * x + 3] = w4.w;
            }
#pragma unroll
          for (int hh = 0; hh < 4; ++hh)
            if (c16 + hh * 16 < DP / 2) sm100::tmem_st16(ta + c16 + hh * 16, v[hh]);
        }
      }
      sm100::tmem_st_wait();
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_full[ab_]);
      ++j;
    }
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer ===============================================
    const uint32_t idesc = sm100::idesc_f16_f32(kM, NV);
    const uint32_t b_lbo = NV * 16, sbo = 128;
    uint32_t abuf = 0;  // A buffer of the current item
    uint32_t t = 0, u = 0;
    for (;;) {
      const int ob = t & 1;
      sm100::mbar_wait_sleep<32>(&op_full[ob], (t >> 1) & 1);
      const Ctrl c = *(const Ctrl*)(meta(t & (kMeta - 1)));
      const int ab = t % nAcc;
      if (t >= (uint32_t)nAcc) sm100::mbar_wait_sleep<32>(&acc_empty[ab], ((t / nAcc) - 1) & 1);
      if (c.list < 0) {
        if (lane == 0) mbar_arrive(&acc_full[ab]);
        break;
      }
      if (c.tile == 0) {
        abuf = u % P.nA;
        sm100::mbar_wait_sleep<32>(&a_full[abuf], (u / P.nA) & 1);
        ++u;
      }
      const uint32_t qhi_t = tmem + a_col + abuf * DP, qlo_t = qhi_t + DP / 2;  // A in TMEM
      sm100::tc_fence_after();
      TRACE(3);
      {
        // whole warp, one elected issuer per instruction; descriptors advance
        // by a constant (start address field) per K step
        const uint32_t bh = sm100::smem_u32(smem + (ob ? Lo.bhi[1] : Lo.bhi[0]));
        const uint32_t bl = sm100::smem_u32(smem + (ob ? Lo.blo[1] : Lo.blo[0]));
        const uint32_t dt = tmem + ab * NV;
        const int ks = DP / 16;
        const uint64_t dstep = (2 * b_lbo) >> 4;
        const uint64_t dh = sm100::smem_desc(bh, b_lbo, sbo), dl = sm100::smem_desc(bl, b_lbo, sbo);
#ifdef IVFTQ_EXP_NOMMA
        if (c.nqt < 0)  // experiment build: MMAs skipped (timing bound only)
#endif
#pragma unroll 1
        for (int pass = 0; pass < 3; ++pass) {
          const uint32_t at = pass == 1 ? qlo_t : qhi_t;
          const uint64_t db = pass == 2 ? dl : dh;
#pragma unroll 4
          for (int s = 0; s < ks; ++s)
            sm100::mma_f16_ts_warp(dt, at + s * 8, db + s * dstep, idesc, (pass | s) ? 1u : 0u);
        }
        sm100::mma_commit_warp(&op_empty[ob]);
        sm100::mma_commit_warp(&acc_full[ab]);
        if (c.tile == c.ntiles - 1) sm100::mma_commit_warp(&a_empty[abuf]);
        TRACE(4);
      }
      __syncwarp();
      ++t;
    }
  } else if (warp < kEpiWarp0) {
    // ================= decoders ==============================================
    const int dt_ = tid - 32 * kDecWarp0;  // 0..255
    constexpr int kDecThreads = 32 * kDecWarps;
    const int NG = (DP + G - 1) / G;
    // Tile record for the MMA issuer and the epilogue (ctrl, query rows +
    // bounds, scaled norms, ids), copied out of the stage slot so the slot
    // returns to the producer as soon as decoding is done.
    auto publish_meta = [&](uint32_t t, const Ctrl& c, const unsigned char* sp) {
      const int ms = t & (kMeta - 1);
      if (t >= (uint32_t)kMeta) sm100::mbar_wait_sleep(&meta_empty[ms], ((t / kMeta) - 1) & 1);
      DTRACE(5);
      unsigned char* mp = meta(ms);
      if (dt_ == 0) *(Ctrl*)mp = c;
      if (c.list >= 0) {
        const int* qsrc = (const int*)(sp + Lo.st_qrow);
        const uint16_t* nrm = (const uint16_t*)(sp + Lo.st_norms);
        const int* idsrc = (const int*)(sp + Lo.st_ids);
        int* qdst = (int*)(mp + Lo.m_qrow);
        float* nsc = (float*)(mp + Lo.m_nsc);
        int* idd = (int*)(mp + Lo.m_ids);
        for (int i = dt_; i < 2 * kM; i += kDecThreads) qdst[i] = qsrc[i];
        for (int v = dt_; v < NV; v += kDecThreads) {
          const bool ok = v < c.valid;
          nsc[v] = ok ? __half2float(__ushort_as_half(nrm[v])) * P.inv_scale
                      : __int_as_float(0x7fc00000);
          idd[v] = ok ? idsrc[v] : INT_MAX;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&meta_full[ms]);
    };
    uint32_t t = 0;
    for (;;) {
      const int s = t % NS;
      sm100::mbar_wait_sleep(&st_full[s], (t / NS) & 1);
      if (warp == kDecWarp0) TRACE(1);
      unsigned char* sp = stage(s);
      const Ctrl c = *(const Ctrl*)(sp + Lo.st_ctrl);
      const int ob = t & 1;
      DTRACE(0);
      if (t >= 2) sm100::mbar_wait_sleep(&op_empty[ob], ((t >> 1) - 1) & 1);
      DTRACE(1);
      if (c.list < 0) {  // stop record: forward it to the MMA issuer and the epilogue
        publish_meta(t, c, sp);
        __syncwarp();
        if (lane == 0) mbar_arrive(&op_full[ob]);
        break;
      }
      // ---- decode this tile's codes into the B operand ----------------------------
      const uint32_t* cw = (const uint32_t*)(sp + Lo.st_codes);
      unsigned char* bhi = smem + (ob ? Lo.bhi[1] : Lo.bhi[0]);
      unsigned char* blo = smem + (ob ? Lo.blo[1] : Lo.blo[0]);
      const int nvshift = __ffs(NV) - 1;
      const uint32_t tab_s = sm100::smem_u32(s_tab);
#ifdef IVFTQ_EXP_NODEC
      if (c.nqt < 0)  // experiment build: decode skipped (timing bound only)
#endif
      for (int task = dt_; task < NV * NG; task += kDecThreads) {
        const int v = task & (NV - 1), gi = task >> nvshift;
        const uint32_t* wv = cw + (v >> 5) * W * 32 + (v & 31);
        uint32_t words[GW];
#pragma unroll
        for (int q = 0; q < GW; ++q) {
          const int w = gi * GW + q;
          words[q] = w < W ? wv[w * 32] : 0u;
        }
#pragma unroll
        for (int cc = 0; cc < GC; ++cc) {
          const int ch = gi * GC + cc;
          if (ch < NCH) {
            uint32_t tv[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int f = cc * 8 + e;  // field within group (compile time)
              // shared address of the entry in a shift and one LOP3 (scan_vq.cu decode_half)
              const int sh = (f % FPW) * FB;
              const uint32_t wf = words[f / FPW];
              const uint32_t ad = (((sh >= 2) ? (wf >> (sh >= 2 ? sh - 2 : 0)) : (wf << (sh < 2 ? 2 - sh : 0))) &
                                   (MASK << 2)) | tab_s;
              asm("ld.shared.u32 %0, [%1];\n" : "=r"(tv[e]) : "r"(ad));
            }
            // entry = hi | lo << 16: one byte permute packs each fp16 pair
            const uint32_t o = ch * (NV * 16) + (v >> 3) * 128 + (v & 7) * 16;
            *(uint4*)(bhi + o) = make_uint4(__byte_perm(tv[0], tv[1], 0x5410),
                                            __byte_perm(tv[2], tv[3], 0x5410),
                                            __byte_perm(tv[4], tv[5], 0x5410),
                                            __byte_perm(tv[6], tv[7], 0x5410));
            *(uint4*)(blo + o) = make_uint4(__byte_perm(tv[0], tv[1], 0x7632),
                                            __byte_perm(tv[2], tv[3], 0x7632),
                                            __byte_perm(tv[4], tv[5], 0x7632),
                                            __byte_perm(tv[6], tv[7], 0x7632));
          }
        }
      }
      sm100::fence_proxy_async_smem();
      DTRACE(4);
      publish_meta(t, c, sp);
      __syncwarp();
      if (warp == kDecWarp0) TRACE(2);
      if (lane == 0) {
        mbar_arrive(&op_full[ob]);
        mbar_arrive(&st_empty[s]);
      }
      ++t;
    }
  } else {
    // ================= epilogue =================================================
    // Thread = query row (TMEM lane); the two warps of a lane quadrant split a
    // tile's columns. Each keeps its own register top-K for the (query, list)
    // pair and emits it at the item's end as one of the pair's two partial
    // lists, so the halves never synchronise. Survivors of a 16-column window
    // (score >= max(own k-th, other half's k-th, global bound)) are taken from
    // registers one per lane per step; the warp steps max-over-lanes times.
    const int quad = warp & 3;             // TMEM lane quadrant (warp_id % 4)
    const int half = (warp - kEpiWarp0) >> 2;
    const int row = quad * 32 + lane;      // query row == TMEM lane
    unsigned long long* thr_sh = (unsigned long long*)(smem + Lo.thr);
    RegTopK<KMAX> top;
    top.init();
    double cs = 0.0;
    uint64_t pub = 0ull;  // last mid-item published K-th key
    uint32_t t = 0, tag = 0;
    const int cols = NV / 2;
    for (;;) {
      const int ab = t % nAcc, ms = t & (kMeta - 1);
      sm100::mbar_wait_sleep(&acc_full[ab], (t / nAcc) & 1);
      sm100::mbar_wait_sleep(&meta_full[ms], (t / kMeta) & 1);
      const unsigned char* mp = meta(ms);
      const Ctrl c = *(const Ctrl*)mp;
      if (c.list < 0) break;
      if (warp == kEpiWarp0) TRACE(5);
#ifdef IVFTQ_TRACE_BUILD
      if (P.trace && blockIdx.x == 0 && lane == 0 && warp == kEpiWarp0 && t < (uint32_t)kTraceTiles)
        P.trace[t * 8 + 7] = c.tile | (c.ntiles << 12) | ((long long)c.nqt << 24);
#endif
      const int pi = ((const int*)(mp + Lo.m_qrow))[row];
      const float bnd = ((const float*)(mp + Lo.m_qrow))[kM + row];
      if (c.tile == 0) {
        top.init();
        tag = t + 1;  // identical in both halves: they consume the same tiles
        cs = pi >= 0 ? P.coarse[pi] : 0.0;  // consumed at the item's end
        pub = 0ull;
      }
      sm100::tc_fence_after();
      const float* nsc = (const float*)(mp + Lo.m_nsc);
      const int* ids = (const int*)(mp + Lo.m_ids);
      const int c0 = half * cols;
      // a warp whose 32 query rows all lie past the item's queries (zero A
      // rows) has nothing to take: it skips the tile and frees its issue slots
#ifdef IVFTQ_EXP_NOEPI
      const int cols_here = 0;  // experiment build: epilogue skipped (timing bound only)
#else
      const int cols_here = quad * 32 < c.nqt ? cols : 0;
#endif
#pragma unroll 1
      for (int cc = 0; cc < cols_here; cc += IVFTQ_EPI_LD) {
        uint32_t r[IVFTQ_EPI_LD];
#if IVFTQ_EPI_LD == 32
        sm100::tmem_ld32(tmem + ((uint32_t)(quad * 32) << 16) + ab * NV + c0 + cc, r);
#else
        tmem_ld16(tmem + ((uint32_t)(quad * 32) << 16) + ab * NV + c0 + cc, r);
#endif
        sm100::tmem_ld_wait();
        ETRACE(cc == 0 ? 0 : 2, clock64());
#pragma unroll
        for (int h = 0; h < IVFTQ_EPI_LD; h += kDrain) {
          // the other half's k-th bounds this pair too (either half's K
          // entries are pair candidates); ignore it unless it is this item's
          const unsigned long long o = *(volatile unsigned long long*)&thr_sh[(half ^ 1) * kM + row];
          const float oth = (uint32_t)(o >> 32) == tag ? __uint_as_float((uint32_t)o) : -INFINITY;
          // rows past the item's queries (zero A rows) take nothing
          const float thr = row < c.nqt ? fmaxf(fmaxf(top.kth(), oth), bnd) : INFINITY;
          float res[kDrain];
          float mx = -INFINITY;  // fmaxf drops the NaN padding columns
#pragma unroll
          for (int e = 0; e < kDrain; e += 4) {
            const float4 f4 = *(const float4*)(nsc + c0 + cc + h + e);
            const float ns[4] = {f4.x, f4.y, f4.z, f4.w};
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              res[e + x] = __fmul_rn(__uint_as_float(r[h + e + x]), ns[x]);
              mx = fmaxf(mx, res[e + x]);
            }
          }

          // one compare per window; the per-column mask only when some lane
          // of the warp has a survivor in it
          uint32_t m = 0;
          if (__any_sync(kFull, mx >= thr)) {
#pragma unroll
            for (int e = 0; e < kDrain; ++e) m |= (res[e] >= thr ? 1u : 0u) << e;  // NaN never passes
          }
          if (__any_sync(kFull, m != 0)) {

            do {
              const int j = (__ffs(m) - 1) & (kDrain - 1);
              const float v = pick16(res, j);
              const int id = ids[c0 + cc + h + j];
              top.insert(m ? cand_key(v, id) : 0ull);
              m &= m - 1;
            } while (__any_sync(kFull, m != 0));
            *(volatile unsigned long long*)&thr_sh[half * kM + row] =
                ((unsigned long long)tag << 32) | __float_as_uint(top.kth());
          }
          if (h + kDrain >= IVFTQ_EPI_LD) ETRACE(cc == 0 ? 1 : 3, clock64());
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
      ETRACE(4, clock64());
#if IVFTQ_MID_PUBLISH
      // Mid-item bound: once this half holds KMAX >= k candidates of the pair,
      // their K-th score lower-bounds the query's final k-th, so the global
      // bound (read per tile by every item of the query) can rise now rather
      // than at the item's end. Published only when it improved.
      if (c.tile + 1 < c.ntiles && row < c.nqt && top.k[KMAX - 1] > pub) {
        pub = top.k[KMAX - 1];
        atomicMax(&P.thr_key[pi / P.n_p], dkey(cs + (double)key_score(pub)));
      }
#endif
      if (c.tile == c.ntiles - 1 && row < c.nqt) {
        // Append this half's candidates of the (query, list) pair to the
        // query's buffer -- only those at or above the query's current global
        // bound: thr_key only rises and lower-bounds the final k-th score, so
        // anything below it can never be returned (ties at the bound are kept).
        const int q = pi / P.n_p;
        const double bound = dkey_inv(*(volatile const long long*)&P.thr_key[q]);
        const int kk = P.k;
        double sv[KMAX];
        int m = 0;
#pragma unroll
        for (int p = 0; p < KMAX; ++p) {
          sv[p] = top.k[p] ? cs + (double)key_score(top.k[p]) : -INFINITY;
          if (p < kk && top.k[p] && sv[p] >= bound) m = p + 1;  // sorted: a prefix
        }
        if (m) {
          const int64_t o = (int64_t)q * P.qcap + atomicAdd(&P.qcnt[q], m);
#pragma unroll
          for (int p = 0; p < KMAX; ++p)
            if (p < m) {
              P.part_s[o + p] = sv[p];
              P.part_id[o + p] = key_id(top.k[p]);
            }
        }
        // KMAX >= k candidates of this query score >= this K-th: a global lower
        // bound on its final k-th that prunes its other lists
        if (top.k[KMAX - 1] != 0)
          atomicMax(&P.thr_key[q], dkey(sv[KMAX - 1]));
      }
      __syncwarp();
      ETRACE(7, clock64());
      if (warp == kEpiWarp0) TRACE(6);
      if (lane == 0) mbar_arrive(&meta_empty[ms]);
      ++t;
    }
  }
  __syncthreads();
  if (warp == kMmaWarp) sm100::tmem_dealloc(tmem, tmem_cols);
}

// ---- probe regrouping: pairs (q, p) bucketed by list ---------------------------
// Pairs are ordered inside each list by probe-rank class (rank 0..6, then 7+)
// and work items are emitted tile-major (every list's first query tile before
// any second tile). A query's best-ranked lists are therefore scanned first,
// which tightens its global pruning bound (thr_key) before its far lists run.
#ifndef IVFTQ_RC
#define IVFTQ_RC 8
#endif
constexpr int kRC = IVFTQ_RC;

__global__ void pair_count_kernel(const int32_t* __restrict__ probe, int64_t npairs, int n_p,
                                  int32_t* __restrict__ cnt2) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npairs) return;
  const int rc = min((int)(i % n_p), kRC - 1);
  atomicAdd(&cnt2[probe[i] * kRC + rc], 1);
}

// one block: exclusive scan over (list, rank class); per-list starts, tiles,
// and the per-tile-index list counts G[t]
__global__ void __launch_bounds__(1024) pair_scan_kernel(const int32_t* __restrict__ cnt2, int L,
                                                         int32_t* __restrict__ pstart2,
                                                         int32_t* __restrict__ pstart,
                                                         int32_t* __restrict__ ntile,
                                                         int32_t* __restrict__ G,
                                                         int32_t* __restrict__ n_items) {
  // One list per thread, 1024 lists per pass (the class counters of a list
  // are contiguous: coalesced loads, kept in registers for the second half),
  // a two-level shuffle scan of (pairs, tiles) per pass with carried totals.
  // G (per-tile-index list counts) is only needed by the tile-major item
  // order and is skipped when null.
  __shared__ int wa[32], wb[32];
  __shared__ int carry_a, carry_b;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { carry_a = 0; carry_b = 0; }
  __syncthreads();
  for (int l0 = 0; l0 < L; l0 += 1024) {
    const int l = l0 + threadIdx.x;
    int cls[kRC];
    int c = 0;
#pragma unroll
    for (int r = 0; r < kRC; ++r) {
      cls[r] = l < L ? cnt2[l * kRC + r] : 0;
      c += cls[r];
    }
    const int nt = (c + kM - 1) / kM;
    int a = c, t = nt;  // inclusive scans
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int va = __shfl_up_sync(kFull, a, o), vb = __shfl_up_sync(kFull, t, o);
      if (lane >= o) { a += va; t += vb; }
    }
    if (lane == 31) { wa[warp] = a; wb[warp] = t; }
    __syncthreads();
    if (warp == 0) {
      int xa = wa[lane], xb = wb[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int va = __shfl_up_sync(kFull, xa, o), vb = __shfl_up_sync(kFull, xb, o);
        if (lane >= o) { xa += va; xb += vb; }
      }
      wa[lane] = xa;
      wb[lane] = xb;
    }
    __syncthreads();
    const int base_a = carry_a + (warp ? wa[warp - 1] : 0);
    int excl = base_a + a - c;  // exclusive pair prefix of this list
    if (l < L) {
      pstart[l] = excl;
      int run = 0;
#pragma unroll
      for (int r = 0; r < kRC; ++r) {
        pstart2[l * kRC + r] = excl + run;
        run += cls[r];
      }
      ntile[l] = nt;
      if (G)
        for (int i = 0; i < nt; ++i) atomicAdd(&G[i], 1);
    }
    __syncthreads();
    if (threadIdx.x == 1023) {
      carry_a += wa[31];
      carry_b += wb[31];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pstart[L] = carry_a;
    pstart2[L * kRC] = carry_a;
    *n_items = carry_b;
  }
}

// one block: exclusive scan of G -> S (first item slot of each tile index)
__global__ void __launch_bounds__(1024) tile_scan_kernel(const int32_t* __restrict__ G, int T,
                                                         int32_t* __restrict__ S) {
  __shared__ int sa[1024];
  const int per = (T + 1023) / 1024;
  const int t0 = threadIdx.x * per, t1 = min(T, t0 + per);
  int a = 0;
  for (int t = t0; t < t1; ++t) a += G[t];
  sa[threadIdx.x] = a;
  __syncthreads();
  for (int s = 1; s < 1024; s <<= 1) {
    int v = threadIdx.x >= s ? sa[threadIdx.x - s] : 0;
    __syncthreads();
    sa[threadIdx.x] += v;
    __syncthreads();
  }
  a = sa[threadIdx.x] - a;
  for (int t = t0; t < t1; ++t) {
    S[t] = a;
    a += G[t];
  }
}

__global__ void pair_scatter_kernel(const int32_t* __restrict__ probe, int64_t npairs, int n_p,
                                    const int32_t* __restrict__ pstart2,
                                    int32_t* __restrict__ cursor2, int32_t* __restrict__ pairs) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npairs) return;
  const int b = probe[i] * kRC + min((int)(i % n_p), kRC - 1);
  pairs[pstart2[b] + atomicAdd(&cursor2[b], 1)] = (int32_t)i;
}

__global__ void items_fill_kernel(const int32_t* __restrict__ ntile, const int32_t* __restrict__ S,
                                  int32_t* __restrict__ fill, int L, int2* __restrict__ items) {
  int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const int nt = ntile[l];
  for (int t = 0; t < nt; ++t) items[S[t] + atomicAdd(&fill[t], 1)] = make_int2(l, t);
}

// Item order. Tile 0 of every list first (tile 0 holds a list's nearest-rank
// pairs: scanning those first tightens every query's global bound before its
// far lists run), then the remaining query tiles list-major: a list's tiles
// 1.. are consecutive items, so neighbouring CTAs stream the list at about
// the same time and its re-reads hit L2. `first_major` = 0 makes every tile
// list-major (measurement only). One block.
__global__ void __launch_bounds__(1024) items_fill_listmajor_kernel(
    const int32_t* __restrict__ ntile, int L, int first_major, int2* __restrict__ items) {
  __shared__ int sa[1024], sb[1024];
  const int per = (L + 1023) / 1024;
  const int l0 = threadIdx.x * per, l1 = min(L, l0 + per);
  int a = 0, f = 0;
  for (int l = l0; l < l1; ++l) {
    const int nt = ntile[l];
    const int head = first_major && nt > 0 ? 1 : 0;
    f += head;
    a += nt - head;
  }
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = f;
  __syncthreads();
  for (int s = 1; s < 1024; s <<= 1) {
    const int va = threadIdx.x >= s ? sa[threadIdx.x - s] : 0;
    const int vb = threadIdx.x >= s ? sb[threadIdx.x - s] : 0;
    __syncthreads();
    sa[threadIdx.x] += va;
    sb[threadIdx.x] += vb;
    __syncthreads();
  }
  const int nfirst = sb[1023];
  a = nfirst + sa[threadIdx.x] - a;
  f = sb[threadIdx.x] - f;
  for (int l = l0; l < l1; ++l) {
    const int nt = ntile[l];
    const int head = first_major && nt > 0 ? 1 : 0;
    if (head) items[f++] = make_int2(l, 0);
    for (int t = head; t < nt; ++t) items[a++] = make_int2(l, t);
  }
}

// Split each rotated query row once per search into fp16 hi/lo (scaled 2^14),
// packed 2 per word along K, zero-padded to DP: the A-operand rows of TMEM.
__global__ void q16_kernel(const float* __restrict__ qrot, int64_t nq, int d, int DP,
                           uint32_t* __restrict__ hi, uint32_t* __restrict__ lo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int hw = DP / 2;
  if (i >= nq * hw) return;
  const int64_t q = i / hw;
  const int j = (int)(i - q * hw) * 2;
  uint32_t h0, l0, h1, l1;
  h0 = split_pack(j < d ? qrot[q * d + j] * 16384.0f : 0.0f, l0);
  h1 = split_pack(j + 1 < d ? qrot[q * d + j + 1] * 16384.0f : 0.0f, l1);
  hi[i] = h0 | (h1 << 16);
  lo[i] = l0 | (l1 << 16);
}

// Seed each query's global pruning bound before the scan: score the first
// (up to) 32*P slots of the query's nearest probed list in f32 (q_rot * f32 T,
// four partial chains, times the f32 norm, plus the f64 coarse score) and
// take the k-th best. Those are k real candidates, so the query's final k-th
// score is at least their k-th -- once each seeded score is lowered by a
// rigorous bound on how far it can sit above the tensor-core scan's score of
// the same candidate. With S = sum_j |q_j| |T[f_j]| <= max|T| * ||q||_1, both
// computations lie within (6d + d/4 + 19) u S of the exact dot (u = 2^-24:
// the scan's fp32 accumulation of 3d exact fp16 products at <= 2u per add,
// allowing for truncating tensor-core adds; its hi/lo split and dropped
// lo*lo terms (3 * 2^-22); this kernel's four chains of d/4 terms), then one
// rounding for the norm product. The margin uses (8d + 64) u S nrm, plus
// 1e-12 (1 + |score|) for the f64 sum. One warp per query.
template <int P, int FB>
__global__ void __launch_bounds__(256)
seed_bound_kernel(ivftq_store st, const int32_t* __restrict__ probe,
                  const double* __restrict__ coarse, const float* __restrict__ qrot,
                  const double* __restrict__ levels, int64_t nq, int n_p, int k,
                  long long* __restrict__ key) {
  constexpr int FPW = 32 / FB;
  constexpr uint32_t mask = (1u << FB) - 1u;
  __shared__ float t32[1 << FB];           // f32 level table
  __shared__ float tmax;                   // max |T|
  __shared__ float qs_all[8][kMaxDim + 8];  // each warp's rotated query row (zero-padded)
  __shared__ double sc_all[8][32 * P];     // each warp's candidate scores
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int W = st.words_per_vec, d = st.dim;
  for (int c = threadIdx.x; c < (1 << FB); c += blockDim.x) t32[c] = (float)levels[c];
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  float* qr = qs_all[warp];
  float qabs = 0.f;
  if (q < nq)
    for (int j = lane; j < W * FPW; j += 32) {
      const float v = j < d ? qrot[q * d + j] : 0.f;
      qr[j] = v;
      qabs += fabsf(v);
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.f;
    for (int c = 0; c < (1 << FB); ++c) m = fmaxf(m, fabsf(t32[c]));
    tmax = m;
  }
  __syncthreads();
  if (q >= nq) return;
#pragma unroll
  for (int o = 16; o; o >>= 1) qabs += __shfl_xor_sync(kFull, qabs, o);
  // S bound, rounded up generously (1.001) for the f32 sums above
  const double slack = (double)(8 * d + 64) * 0x1p-24 * (double)tmax * (double)qabs * 1.001;
  const int l0 = probe[q * n_p];
  const int m = min(st.list_size[l0], 32 * P);
  const double cs = coarse[q * n_p];
  double* scw = sc_all[warp];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    double v = -INFINITY;
    const int i = p * 32 + lane;
    if (i < m) {
      const int64_t slot = st.list_offset[l0] + i;
      const uint32_t* cw = st.codes + (slot >> 5) * W * 32 + (slot & 31);
      // four partial sums (fields f % 4): independent chains; the f32 result
      // differs from a sequential fold by a few ulps, inside the bound's margin
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int w0 = 0; w0 < W; w0 += 8) {  // 8 words in flight per batch
        uint32_t wd[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) wd[x] = w0 + x < W ? cw[(w0 + x) * 32] : 0u;
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          if (w0 + x < W) {
            const float* qw = qr + (w0 + x) * FPW;  // padded past d with zeros
#pragma unroll
            for (int f = 0; f < FPW; ++f)
              acc[f & 3] = __fmaf_rn(qw[f], t32[(wd[x] >> (f * FB)) & mask], acc[f & 3]);
          }
        }
      }
      const float dot = (acc[0] + acc[1]) + (acc[2] + acc[3]);
      const float nrm = __half2float(__ushort_as_half(st.norms[slot]));
      v = cs + (double)__fmul_rn(nrm, dot);
      v -= (double)nrm * slack + 1e-12 * (1.0 + fabs(v));  // never above the scan's score
    }
    scw[p * 32 + lane] = v;
  }
  __syncwarp();
  // k-th best (with multiplicity; slots past the list hold -inf): k rounds of
  // "take the warp's maximum out", each lane holding P of the 32 P scores
  double mine[P];
#pragma unroll
  for (int p = 0; p < P; ++p) mine[p] = scw[p * 32 + lane];
  double kth = -INFINITY;
  for (int it = 0; it < k; ++it) {
    double lm = mine[0];
    int lp = 0;
#pragma unroll
    for (int p = 1; p < P; ++p)
      if (mine[p] > lm) { lm = mine[p]; lp = p; }
    double gm = lm;
#pragma unroll
    for (int o = 16; o; o >>= 1) gm = fmax(gm, __shfl_xor_sync(kFull, gm, o));
    kth = gm;
    if (!(gm > -INFINITY)) break;  // fewer than k scores: no bound
    const unsigned own = __ballot_sync(kFull, lm == gm);
    if (lane == __ffs(own) - 1) {
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (p == lp) mine[p] = -INFINITY;
    }
  }
  if (lane == 0) {
    double b = -INFINITY;
    if (m >= k && kth > -INFINITY) b = kth;
    key[q] = dkey(b);
  }
}

__global__ void thr_init_kernel(long long* __restrict__ key, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) key[i] = dkey(-INFINITY);
}

}  // namespace tc
}  // namespace ivftq

using namespace ivftq;
using namespace ivftq::tc;

// Optional device timing of the scan kernel alone (bench roofline evidence):
// a switch and an event pair per (host thread, device), so concurrent callers
// never record into each other's events.
#include <map>
#include <utility>
static thread_local bool t_time_kernel = false;
static thread_local const char* t_scan_kernel = "";

extern "C" const char* ivftq_last_scan_kernel(void) { return t_scan_kernel; }
static thread_local std::map<int, std::pair<cudaEvent_t, cudaEvent_t>> t_ev;

static std::pair<cudaEvent_t, cudaEvent_t>* timing_events() {
  int dev = 0;
  cudaGetDevice(&dev);
  auto it = t_ev.find(dev);
  if (it == t_ev.end()) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return nullptr;
    it = t_ev.emplace(dev, std::make_pair(a, b)).first;
  }
  return &it->second;
}

extern "C" int ivftq_set_kernel_timing(int on) {
  t_time_kernel = on != 0;
  if (t_time_kernel && !timing_events()) {
    set_error("set_kernel_timing: event creation failed");
    return IVFTQ_ERR_CUDA;
  }
  return 0;
}

extern "C" int ivftq_get_kernel_timing(void) { return t_time_kernel ? 1 : 0; }

extern "C" double ivftq_last_scan_kernel_ms(void) {
  int dev = 0;
  cudaGetDevice(&dev);
  auto it = t_ev.find(dev);
  if (it == t_ev.end()) return -1.0;
  float ms = -1.f;
  // events never recorded (no timed launch yet) fail here: report -1 and
  // clear the error so it does not surface at the next launch check
  if (cudaEventSynchronize(it->second.second) != cudaSuccess ||
      cudaEventElapsedTime(&ms, it->second.first, it->second.second) != cudaSuccess) {
    cudaGetLastError();
    return -1.0;
  }
  return ms;
}

// Records the start/stop events around one launch when timing is on; inside
// a stream capture they become external event nodes, marking every replay.
struct KernelTimer {
  cudaStream_t s;
  std::pair<cudaEvent_t, cudaEvent_t>* ev = nullptr;
  unsigned flags = cudaEventRecordDefault;
  explicit KernelTimer(cudaStream_t st) : s(st) {
    if (!t_time_kernel) return;
    ev = timing_events();
    if (!ev) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs == cudaStreamCaptureStatusActive) flags = cudaEventRecordExternal;
    cudaEventRecordWithFlags(ev->first, s, flags);
  }
  void stop() {
    if (ev) cudaEventRecordWithFlags(ev->second, s, flags);
  }
};

// Joins the side stream back into the caller's stream on every exit path, so
// an error return inside a capture never leaves the capture forked.
struct SideJoin {
  SideStream* ss;
  cudaStream_t s;
  bool done = false;
  ~SideJoin() {
    if (!done) join();
  }
  cudaError_t join() {
    done = true;
    cudaError_t e = cudaEventRecord(ss->join, ss->stream);
    cudaError_t e2 = cudaStreamWaitEvent(s, ss->join, 0);
    return e != cudaSuccess ? e : e2;
  }
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct TcScratch {
  int32_t *cnt2, *cursor2, *G, *fill, *counter, *pstart2, *pstart, *ntile, *S, *n_items, *pairs;
  long long* thr_key;
  uint32_t *q_hi, *q_lo;
  int2* items;
  double* part_s;
  int32_t* part_id;
  int32_t* qcnt;
  char* zero_end;
  int T;
  size_t bytes;
};

static int pad_dp(int dim) { return (dim + 31) / 32 * 32; }

static TcScratch carve_tc(void* base, int64_t nq, int n_p, int L, int k, int dim) {
  TcScratch S{};
  size_t off = 0;
  char* b = (char*)base;
  int64_t np = nq * n_p;
  int64_t max_items = np / kM + (np < L ? np : L) + 1;
  S.T = (int)(nq / kM + 2);
  auto take = [&](size_t bytes) {
    char* p = b ? b + off : nullptr;
    off += align256(bytes);
    return p;
  };
  // zero-initialised block first
  S.cnt2 = (int32_t*)take(4 * (size_t)L * kRC);
  S.cursor2 = (int32_t*)take(4 * (size_t)L * kRC);
  S.G = (int32_t*)take(4 * (size_t)S.T);
  S.fill = (int32_t*)take(4 * (size_t)S.T);
  S.counter = (int32_t*)take(16);
  S.qcnt = (int32_t*)take(4 * (size_t)nq);
  S.zero_end = b ? b + off : nullptr;
  S.pstart2 = (int32_t*)take(4 * ((size_t)L * kRC + 1));
  S.pstart = (int32_t*)take(4 * (size_t)(L + 1));
  S.ntile = (int32_t*)take(4 * (size_t)L);
  S.S = (int32_t*)take(4 * (size_t)(S.T + 1));
  S.n_items = (int32_t*)take(16);
  S.thr_key = (long long*)take(8 * (size_t)nq);
  S.pairs = (int32_t*)take(4 * (size_t)np);
  S.q_hi = (uint32_t*)take(4 * (size_t)nq * (pad_dp(dim) / 2));
  S.q_lo = (uint32_t*)take(4 * (size_t)nq * (pad_dp(dim) / 2));
  S.items = (int2*)take(8 * (size_t)max_items);
  S.part_s = (double*)take(8 * (size_t)np * 2 * k);  // two partial lists per pair
  S.part_id = (int32_t*)take(4 * (size_t)np * 2 * k);
  S.bytes = off;
  return S;
}

extern "C" size_t ivftq_scan_tc_scratch_bytes(int64_t nq, int n_p, int n_lists, int depth) {
  // dim is not known here: size the query rows for the widest supported dim
  return carve_tc(nullptr, nq, n_p, n_lists, depth, kMaxDim).bytes + 256;
}

static const size_t kSmemLimit = 227 * 1024;

// Widest vector tile, then deepest stage ring, that fits in shared memory.
static int kmax_for(int depth) { return depth <= 10 ? 10 : 32; }

static bool pick_tile(int DP, int W, int C, int kmax, int* nv, int* ns, int* nacc = nullptr) {
  if (DP > kMaxDim) return false;
  static const int shapes[3][2] = {{128, 2}, {128, 3}, {64, 4}};  // (NV, nAcc), widest first
  const char* force = getenv("IVFTQ_SCAN_NV");
  const char* facc = getenv("IVFTQ_SCAN_ACC");
  for (const auto& sh : shapes) {
    if (force && atoi(force) != sh[0]) continue;
    if (facc && atoi(facc) != sh[1]) continue;
    if (sh[0] * sh[1] + DP > 512) continue;  // one A buffer at least
    if (make_layout(sh[0], kNS, DP, W, C, kmax).total + 1024 > kSmemLimit) continue;
    *nv = sh[0];
    *ns = kNS;
    if (nacc) *nacc = sh[1];
    return true;
  }
  return false;
}

extern "C" int ivftq_scan_tc_supported(int dim, int bits, int depth) {
  int fb = field_bits(bits, 1);
  if (fb < 3 || fb > 5 || depth < 1 || depth > 32) return 0;
  int DP = pad_dp(dim);
  int W = words_per_vec(dim, fb);
  int nv, ns;
  return pick_tile(DP, W, 1 << fb, kmax_for(depth), &nv, &ns);
}

template <int FB, int KMAX>
static int launch_tc(const Params& P, size_t smem, int grid, cudaStream_t s) {
  auto fn = scan_tc_kernel<FB, KMAX>;
  if (int e = smem_opt_in_dev((const void*)fn, smem)) return e;
  KernelTimer timer(s);
  fn<<<grid, kThreads, smem, s>>>(P);
  timer.stop();
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
  TcScratch S = carve_tc(scratch, nq, n_p, L, depth, st->dim);
  int64_t np = nq * n_p;
  IVFTQ_CHECK_CUDA(cudaMemsetAsync(S.cnt2, 0, S.zero_end - (char*)S.cnt2, s));
  unsigned gp = (unsigned)((np + 255) / 256);
  // The seeded bounds and the probe regrouping both only read the probes:
  // the seeding runs on this thread's side stream, overlapping the
  // (latency-bound, partly single-block) regroup kernels, and the scan waits
  // for both.
  SideStream* ss = nullptr;
  if (int e = side_stream(&ss)) return e;
  cudaStream_t side = ss->stream;
  IVFTQ_CHECK_CUDA(cudaEventRecord(ss->fork, s));
  IVFTQ_CHECK_CUDA(cudaStreamWaitEvent(side, ss->fork, 0));
  SideJoin join{ss, s};
  // global pruning bounds: seeded from each query's nearest list (exactness
  // preserved by a margin), unless disabled for measurement
  if (getenv("IVFTQ_NO_SEED")) {
    thr_init_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, side>>>(S.thr_key, nq);
  } else {
    const char* sp_env = getenv("IVFTQ_SEED_P");
    const int sp = sp_env ? atoi(sp_env) : kSeedP;
    const unsigned sb = (unsigned)((nq + 7) / 8);
#define SEED_CASE(PV, FBV)                                                              \
  seed_bound_kernel<PV, FBV><<<sb, 256, 0, side>>>(*st, probe, coarse, qrot, levels, nq, \
                                                   n_p, depth, S.thr_key)
#define SEED_FB(PV)                                                 \
  if (st->field_bits == 3) SEED_CASE(PV, 3);                        \
  else if (st->field_bits == 4) SEED_CASE(PV, 4);                   \
  else SEED_CASE(PV, 5)
    if (sp >= 4) {
      SEED_FB(4);
    } else if (sp == 2) {
      SEED_FB(2);
    } else {
      SEED_FB(1);
    }
#undef SEED_FB
#undef SEED_CASE
  }
  if (int e = check_launch("thr_init")) return e;
  {  // the scan's A-operand rows (fp16 hi/lo of the rotated queries), also off the main stream
    const int DPq = pad_dp(st->dim);
    const int64_t nw = nq * (DPq / 2);
    q16_kernel<<<(unsigned)((nw + 255) / 256), 256, 0, side>>>(qrot, nq, st->dim, DPq, S.q_hi,
                                                                S.q_lo);
    if (int e = check_launch("q16")) return e;
  }
  pair_count_kernel<<<gp, 256, 0, s>>>(probe, np, n_p, S.cnt2);
  if (int e = check_launch("pair_count")) return e;
  const char* order = getenv("IVFTQ_ITEMS_ORDER");
  const bool tile_major = order && order[0] == 't';
  pair_scan_kernel<<<1, 1024, 0, s>>>(S.cnt2, L, S.pstart2, S.pstart, S.ntile,
                                      tile_major ? S.G : nullptr, S.n_items);
  if (int e = check_launch("pair_scan")) return e;
  if (tile_major) {
    tile_scan_kernel<<<1, 1024, 0, s>>>(S.G, S.T, S.S);
    if (int e = check_launch("tile_scan")) return e;
  }
  pair_scatter_kernel<<<gp, 256, 0, s>>>(probe, np, n_p, S.pstart2, S.cursor2, S.pairs);
  if (int e = check_launch("pair_scatter")) return e;
  // default: tile 0 of every list first, then each list's further tiles back to
  // back (C2 n_p=64: 211 MB of DRAM reads per scan instead of 405 MB, same
  // time); IVFTQ_ITEMS_ORDER=tile (round 1's tile-major order) or =list
  // (everything list-major: 114 MB, 3-12 % slower) for measurement
  if (tile_major)
    items_fill_kernel<<<(L + 255) / 256, 256, 0, s>>>(S.ntile, S.S, S.fill, L, S.items);
  else
    items_fill_listmajor_kernel<<<1, 1024, 0, s>>>(S.ntile, L, order && order[0] == 'l' ? 0 : 1,
                                                   S.items);
  if (int e = check_launch("items_fill")) return e;

  const int fb = st->field_bits, C = 1 << fb;
  const int DP = pad_dp(st->dim);
  IVFTQ_CHECK_CUDA(join.join());  // seeded bounds, A rows in place
  // The vectors x queries scan sizes the MMA N to the queries a list really
  // has; with 128+ queries per list on average (C2: ~625) every item of the
  // queries-on-M scan is full and its fused per-query top-k wins, so the
  // choice follows the batch shape (both return the exact same top-k).
  const char* force_vq = getenv("IVFTQ_SCAN_VQ");
  const bool vq_shape = force_vq ? atoi(force_vq) != 0 : (double)nq * n_p < 128.0 * L;
  if (vq_shape && scan_vq_supported(st->dim, fb, depth)) {
    t_scan_kernel = "scan_vq_kernel";
    const int qcap = n_p * depth;  // one partial list per (query, list) pair
    int rc;
    {
      KernelTimer timer(s);
      rc = launch_scan_vq(st, coarse, levels, S.pairs, S.pstart, S.items, S.n_items, S.counter,
                          S.part_s, S.part_id, S.qcnt, S.thr_key, S.q_hi, S.q_lo, n_p, depth,
                          qcap, s);
      timer.stop();
    }
    if (rc) return rc;
    if (int e = merge_smem_opt_in(depth)) return e;
    // fixed k-slot per pair, empty entries id INT_MAX: no per-query counts
    launch_merge(S.part_s, S.part_id, nq, qcap, depth, ids_out, scores_out, s, nullptr);
    return check_launch("merge");
  }
  t_scan_kernel = "scan_tc_kernel";
  Params P{};
  const int kmax = kmax_for(depth);
  pick_tile(DP, st->words_per_vec, C, kmax, &P.NV, &P.NS, &P.nAcc);
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
  P.qcnt = S.qcnt;
  P.qcap = n_p * 2 * depth;
  P.thr_key = S.thr_key;
  P.q_hi = S.q_hi;
  P.q_lo = S.q_lo;
  const char* trace_path = getenv("IVFTQ_TRACE");
  long long* trace = nullptr;
  if (trace_path) {
    cudaMalloc(&trace, sizeof(long long) * 24 * kTraceTiles);
    cudaMemsetAsync(trace, 0, sizeof(long long) * 24 * kTraceTiles, s);
  }
  P.trace = trace;
  P.n_p = n_p;
  P.k = depth;
  P.d = st->dim;
  P.DP = DP;
  P.nA = (P.nAcc * P.NV + 2 * DP <= 512) ? 2 : 1;
  // Every Lloyd-Max level satisfies |T| < 5/sqrt(d) < 4, so 2^12 keeps the
  // scaled table below 2^14 and its hi/lo halves in the fp16 normal range.
  const int eT = 12;
  P.t_scale = ldexpf(1.0f, eT);
  P.inv_scale = ldexpf(1.0f, -(eT + 14));
  P.lo = make_layout(P.NV, P.NS, DP, st->words_per_vec, C, kmax);
  size_t smem = P.lo.total + 1024;
  int grid = device_sm_count();
  int rc;
#define TC_CASE(FBV)                                                              \
  if (fb == FBV) {                                                                \
    rc = kmax == 10 ? launch_tc<FBV, 10>(P, smem, grid, s)                        \
                    : launch_tc<FBV, 32>(P, smem, grid, s);                       \
  }
  TC_CASE(3) else TC_CASE(4) else TC_CASE(5) else {
    set_error("scan_tc: field width %d", fb);
    return IVFTQ_ERR_UNSUPPORTED;
  }
#undef TC_CASE
  if (rc) return rc;
  if (trace) {
    static long long h[24 * kTraceTiles];
    cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    FILE* f = fopen(trace_path, "w");
    if (f) {
      fprintf(f, "# NV=%d nbuf=2 tiles: t prod dec_start dec_end mma_start mma_end epi_start epi_end\n", P.NV);
      for (int t = 0; t < kTraceTiles; ++t) {
        if (!h[t * 8 + 1]) break;
        fprintf(f, "%d", t);
        for (int k = 0; k < 7; ++k) fprintf(f, " %lld", h[t * 8 + k] ? h[t * 8 + k] - h[1] : -1);
        fprintf(f, " %lld %lld %lld", h[t * 8 + 7] & 4095, (h[t * 8 + 7] >> 12) & 4095, h[t * 8 + 7] >> 24);
        fprintf(f, "\n");
      }
      fclose(f);
    }
    std::string dp = std::string(trace_path) + ".dec";
    f = fopen(dp.c_str(), "w");
    if (f) {
      fprintf(f, "# t after_stfull after_opempty after_aempty after_abuild after_decode after_metaempty (rel. dec_start)\n");
      for (int t = 0; t < kTraceTiles; ++t) {
        const long long* e = h + 16 * kTraceTiles + t * 8;
        if (!h[t * 8 + 1]) break;
        const long long b = h[t * 8 + 1];
        fprintf(f, "%d", t);
        for (int k = 0; k < 6; ++k) fprintf(f, " %lld", e[k] ? e[k] - b : -1);
        fprintf(f, "\n");
      }
      fclose(f);
    }
    std::string ep = std::string(trace_path) + ".epi";
    f = fopen(ep.c_str(), "w");
    if (f) {
      fprintf(f, "# t ld0 win0 ld1 win1 acc_released x x end (rel. epi_start)\n");
      for (int t = 0; t < kTraceTiles; ++t) {
        const long long* e = h + 8 * kTraceTiles + t * 8;
        if (!h[t * 8 + 1]) break;
        const long long b = h[t * 8 + 5];
        fprintf(f, "%d %lld %lld %lld %lld %lld %lld %lld %lld\n", t, e[0] - b, e[1] - b,
                e[2] - b, e[3], e[4] - b, e[5] - b, e[6], e[7] - b);
      }
      fclose(f);
    }
    cudaFree(trace);
  }
  if (int e = merge_smem_opt_in(depth)) return e;
  launch_merge(S.part_s, S.part_id, nq, n_p * 2 * depth, depth, ids_out, scores_out, s, S.qcnt);
  return check_launch("merge");
}
