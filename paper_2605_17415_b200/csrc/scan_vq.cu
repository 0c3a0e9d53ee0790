// Tensor-core list scan, vectors x queries (tcgen05), for d <= 128.
//
// Same reference semantics as scan_tc.cu (index.py:442-458 list-major scan,
// index.py:460-483 per-query top-k), with the roles of the two MMA operands
// swapped so that every stage's work is proportional to real (query, vector)
// pairs:
//
//   * MMA M = 128 list vectors (TMEM lanes), N = the item's queries rounded
//     up to 16 (an item holds <= 128 queries of one list): D[v][q];
//   * A (the decoded vectors, fp16 hi/lo) is written straight into TMEM by
//     the decoder warps with tcgen05.st -- no shared-memory image of the
//     decoded tile, no K-major swizzle bookkeeping on the decode side;
//   * B (the item's rotated queries, fp16 hi/lo, K-major canonical layout) is
//     gathered into shared memory once per item and reused by all its tiles;
//   * the epilogue is a filter, thread = vector: per 16-query window one
//     TMEM load, one FFMA per pair against the query's current threshold
//     (res - thr, with thr lowered by a rigorous rounding margin), one max;
//     each warp keeps its lane quadrant's top-k of every query it filters in
//     shared memory and inserts the rare survivors warp-cooperatively; a full
//     list raises the query's threshold and its global bound thr_key (read by
//     the other CTAs); at the item's end each pair's four quadrant lists are
//     merged into its fixed k-slot of the candidate buffer, which
//     merge_warp_kernel reduces;
//   * an emitter warp opens each item's threshold slot (from the queries'
//     global bounds) and keeps it fresh while the item runs.
//
// Warp roles (20 warps = 5 per SM sub-partition, 96 registers each; one CTA
// per SM, persistent over an atomic item counter):
//   0  producer   item records (list span, query rows, coarse scores) one
//                 item ahead; per tile a control record + 1-D TMA bulk copies
//                 of the tile's packed codes, norms and ids into a stage ring
//   1  MMA        tcgen05.mma kind::f16, A from TMEM, B from shared memory,
//                 3 products (Thi.Qhi + Thi.Qlo + Tlo.Qhi) per K step
//   2  loader     the item's query rows -> B (double-buffered)
//   3  emitter    each item's filter thresholds from the queries' global
//                 bounds, kept fresh while the item runs
//   4-11 decoders thread = (vector, K half): codes -> level table -> TMEM A
//   12-19 epilogue thread = vector, warp = (lane quadrant, window parity):
//                 filter, per-quadrant top-k, the pair's candidates at the
//                 item's end
//
// Numerics are scan_tc.cu's: q * 2^14 and T * 2^12 split into fp16 hi + lo,
// fp32 accumulation in TMEM, res = D * (f32(||r||) * 2^-26).
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "sm100.cuh"

namespace ivftq {

void launch_merge(const double* part_s, const int32_t* part_id, int64_t nq, int n_in, int K,
                  int64_t* ids_out, double* s_out, cudaStream_t s,
                  const int32_t* counts = nullptr);
int merge_smem_opt_in(int K);

namespace vq {

constexpr int kNV = 128;       // vectors per tile = MMA M = TMEM lanes
constexpr int kQM = 128;       // queries per item (max MMA N used)
constexpr int kProd = 0, kMma = 1, kLoad = 2, kEmit = 3;
constexpr int kDec0 = 4, kDecWarps = 8;
constexpr int kEpi0 = 12, kEpiWarps = 8;
constexpr int kWarps = 20, kThreads = 32 * kWarps;
constexpr int kItems = 4;      // item-record ring
constexpr int kMaxNS = 6;
constexpr int kMeta = 4;        // tile-record ring (decoders -> MMA, epilogue)

// barrier indices (8 bytes each)
constexpr int kBStF = 0, kBStE = kBStF + kMaxNS, kBAF = kBStE + kMaxNS, kBAE = kBAF + 2,
              kBAccF = kBAE + 2, kBAccE = kBAccF + 2, kBBF = kBAccE + 2, kBBE = kBBF + 2,
              kBItF = kBBE + 2, kBItE = kBItF + kItems, kBDone = kBItE + kItems,
              kBReady = kBDone + 2, kBMF = kBReady + 2, kBME = kBMF + kMeta,
              kBCount = kBME + kMeta;

struct Ctrl {
  int list;    // -1 = stop
  int tile;
  int ntiles;
  int valid;   // vectors of this tile that exist
  int item;    // per-CTA item sequence number (parities, slots)
  int nq;
  int N;       // MMA N (nq rounded up to 16)
  int pad;
};

struct ItemRec {
  int list;    // -1 = stop
  int nq;
  int N;
  int ntiles;
  int size;
  int pad0;
  long long off;
  int q[kQM];       // query index of each row
  int rank[kQM];    // its probe rank (the pair's slot in the candidate buffer)
  double cs[kQM];   // coarse score of each row's (query, list) pair
};

struct Layout {
  uint32_t bq[2], bq_bytes, stage, stage_bytes, st_norms, st_ids, st_ctrl, items, item_bytes,
      lists, thr, thr_raw, meta, meta_bytes, misc, bars, total;
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) & ~(a - 1); }

__host__ __device__ inline Layout make_layout(int DP, int W, int NS, int k) {
  Layout L{};
  uint32_t off = 0;
  auto take = [&](uint32_t bytes) {
    uint32_t o = off;
    off = align_up(off + bytes, 128u);
    return o;
  };
  L.bq_bytes = (uint32_t)DP * kQM * 2 * 2;  // hi + lo, fp16
  L.bq[0] = take(L.bq_bytes);
  L.bq[1] = take(L.bq_bytes);
  L.st_norms = align_up(kNV * (uint32_t)W * 4, 128);
  L.st_ids = L.st_norms + align_up(kNV * 2, 128);
  L.st_ctrl = L.st_ids + align_up(kNV * 4, 128);
  L.stage_bytes = L.st_ctrl + 128;
  L.stage = take(L.stage_bytes * NS);
  L.item_bytes = align_up(sizeof(ItemRec), 128);
  L.items = take(L.item_bytes * kItems);
  L.lists = take(4u * kQM * (uint32_t)k * 8);  // [lane quadrant][query row][k]
  L.thr = take(2u * kQM * 4);
  L.thr_raw = take(2u * kQM * 4);
  L.meta_bytes = align_up(sizeof(Ctrl) + kNV * 8, 128);  // ctrl | ns[kNV] f32 | id[kNV]
  L.meta = take(L.meta_bytes * kMeta);
  L.misc = take(64);
  L.bars = take(8 * kBCount);
  L.total = off;
  return L;
}

struct Params {
  ivftq_store st;
  const double* coarse;    // [nq*n_p]
  const int32_t* pair_idx; // pair flat index q*n_p+p, grouped by list
  const int32_t* pstart;   // [L+1]
  const int2* items;       // (list, query tile)
  const int32_t* n_items;
  int32_t* counter;
  double* part_s;          // [nq][qcap]
  int32_t* part_id;
  int32_t* qcnt;
  long long* thr_key;      // [nq]
  const uint32_t* q_hi;    // [nq][DP/2]
  const uint32_t* q_lo;
  const double* levels;
  long long* trace;        // trace build: CTA 0 per-tile timeline + [kTraceTiles*8] counters
  int n_p, k, d, NS, qcap;  // qcap = n_p * k: one k-slot per (query, list) pair
  float t_scale, inv_scale;
  Layout lo;
};

constexpr int kTraceTiles = 4096;
// Per-tile timeline of CTA 0 (trace build only: make trace, IVFTQ_TRACE=<file>):
// [t*8 + slot] = clock64 at: 0 producer issued the TMA, 1 decoders (warp 4)
// done, 2 MMA issue start, 3 MMA issue end, 4 epilogue (warp 12) start, 5
// epilogue end, 6 decoder start (stage ready), 7 tile | ntiles << 12 | nq << 24.
// Slot kTraceTiles*8 + 0: survivors (CTA 0), + 1: inserts (CTA 0); from
// kTraceTiles*8 + 8, per item j of CTA 0 (4 slots): -, -, emitted, slot_ready.
constexpr int kTraceItems = 1024;
#ifdef IVFTQ_TRACE_BUILD
#define VTRACE(slot, val)                                                          \
  do {                                                                             \
    if (P.trace && blockIdx.x == 0 && lane == 0 && t < (uint32_t)kTraceTiles)      \
      P.trace[t * 8 + (slot)] = (val);                                             \
  } while (0)
#define ITRACE(j, slot)                                                            \
  do {                                                                             \
    if (P.trace && blockIdx.x == 0 && lane == 0 && (j) < (uint32_t)kTraceItems)    \
      P.trace[kTraceTiles * 8 + 8 + (j) * 4 + (slot)] = clock64();                 \
  } while (0)
#define VCOUNT(slot, n)                                                            \
  do {                                                                             \
    if (P.trace && blockIdx.x == 0) atomicAdd((unsigned long long*)&P.trace[kTraceTiles * 8 + (slot)], \
                           (unsigned long long)(n));                               \
  } while (0)
#else
#define VTRACE(slot, val) do {} while (0)
#define VCOUNT(slot, n) do {} while (0)
#define ITRACE(j, slot) do {} while (0)
#endif

// ---- helpers -------------------------------------------------------------------
__device__ __forceinline__ uint32_t split_pack(float x, uint32_t& lo) {
  __half h = __float2half_rn(x);
  __half l = __float2half_rn(x - __half2float(h));
  lo = (uint32_t)__half_as_ushort(l);
  return (uint32_t)__half_as_ushort(h);
}
// (score desc, id asc) as one u64: order-preserving f32 bits, then ~id
__device__ __forceinline__ unsigned long long cand_key(float v, int id) {
  uint32_t b = __float_as_uint(v + 0.0f);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
  return ((unsigned long long)b << 32) | (uint32_t)~(uint32_t)id;
}
__device__ __forceinline__ float key_score(unsigned long long k) {
  const uint32_t o = (uint32_t)(k >> 32);
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
__device__ __forceinline__ int key_id(unsigned long long k) { return (int)~(uint32_t)k; }
__device__ __forceinline__ long long dkey(double x) {
  long long b = __double_as_longlong(x);
  return b >= 0 ? b : (b ^ 0x7FFFFFFFFFFFFFFFLL);
}
__device__ __forceinline__ double dkey_inv(long long k) {
  return __longlong_as_double(k >= 0 ? k : (k ^ 0x7FFFFFFFFFFFFFFFLL));
}
// residual-space bound from a query's global bound (scan_tc.cu prune_bound):
// res < bound  =>  coarse + res < the query's final k-th score
__device__ __forceinline__ float prune_bound(long long key, double coarse) {
  const double thr = dkey_inv(key);
  if (!(thr > -INFINITY)) return -INFINITY;
  const float b = (float)(thr - coarse - 1e-12);
  return nextafterf(b, -INFINITY);
}
// The epilogue passes a pair when fma(D, ns, -lower(T)) >= 0. With x = D*ns
// exact, fl(x) >= T implies x >= T - |T| 2^-24 - 2^-150 >= lower(T), and
// rounding is monotone, so every candidate whose stored res = fl(x) reaches
// T survives the filter (ties included); lower() sits >= 2^-23 |T| below T.
__device__ __forceinline__ float lower_thr(float T) {
  if (!(T > -INFINITY) || T == INFINITY) return T;
  return T - fabsf(T) * 0x1p-22f - 0x1p-126f;
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}
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
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(sm100::smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint32_t ld_vol(const uint32_t* p) {
  return *(volatile const uint32_t*)p;
}

// Roles that usually run ahead (producer, loader, decoders, emitter) poll
// with a short sleep, so their waits do not take issue slots from the
// epilogue warps sharing their SM sub-partition.
#ifndef IVFTQ_VQ_SLEEP
#define IVFTQ_VQ_SLEEP 64
#endif
__device__ __forceinline__ void vwait_sleep(uint64_t* bar, uint32_t parity) {
  while (!mbar_test(bar, parity)) __nanosleep(IVFTQ_VQ_SLEEP);
}
// mbarrier wait; the debug build (make debug) reports a wait that never ends
#ifdef IVFTQ_DEBUG
__shared__ int dbg_state[32];  // per warp: tag * 1000000 + tile counter
__device__ __forceinline__ void vwait(uint64_t* bar, uint32_t parity, int tag) {
  long long n = 0;
  if ((threadIdx.x & 31) == 0) dbg_state[threadIdx.x >> 5] = tag;
  while (!mbar_test(bar, parity)) {
    if (++n == (1ll << 22) && (threadIdx.x & 31) == 0) {
      printf("scan_vq hang: block %d warp %d wait tag %d parity %u | states %d %d %d %d | %d %d %d %d %d %d %d %d | %d %d %d %d %d %d %d %d\n", blockIdx.x,
             threadIdx.x >> 5, tag, parity, dbg_state[0], dbg_state[1], dbg_state[2], dbg_state[3],
             dbg_state[4], dbg_state[5], dbg_state[6], dbg_state[7], dbg_state[8], dbg_state[9], dbg_state[10], dbg_state[11],
             dbg_state[12], dbg_state[13], dbg_state[14], dbg_state[15], dbg_state[16], dbg_state[17], dbg_state[18], dbg_state[19]);
    }
    if (n == (1ll << 25)) __trap();
  }
  if ((threadIdx.x & 31) == 0) dbg_state[threadIdx.x >> 5] = -tag;
}
#define VWAIT(bar, parity, tag) vwait(bar, parity, tag)
#define VWAITS(bar, parity, tag) vwait(bar, parity, tag)
#define DSTATE(v) do { if ((threadIdx.x & 31) == 0) dbg_state[threadIdx.x >> 5] = (v); } while (0)
#else
#define DSTATE(v) do {} while (0)
#define VWAIT(bar, parity, tag) sm100::mbar_wait(bar, parity)
#define VWAITS(bar, parity, tag) vwait_sleep(bar, parity)
#endif

// Decode one K half (dims [KH*DP/2, (KH+1)*DP/2)) of one vector into TMEM:
// hi halves at columns dim/2 of the A buffer, lo halves DP/2 columns later.
template <int FB, int DP, int KH>
__device__ __forceinline__ void decode_half(const uint32_t* __restrict__ cw, int W,
                                            uint32_t tab, uint32_t ta) {
  constexpr int FPW = 32 / FB;
  constexpr uint32_t MASK = (1u << FB) - 1u;
  constexpr int H = DP / 2, J0 = KH * H;
  constexpr int W0 = J0 / FPW, W1 = (J0 + H - 1) / FPW, NW = W1 - W0 + 1;
  uint32_t wd[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) wd[i] = (W0 + i < W) ? cw[(W0 + i) * 32] : 0u;
#pragma unroll
  for (int g = 0; g < H / 16; ++g) {
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int j = J0 + g * 16 + 2 * e;
      // field -> shared address of its table entry in a shift and one LOP3:
      // ((w >> (s - 2)) & (MASK << 2)) | table base (the table is aligned to
      // its size, so the OR is the add)
      constexpr uint32_t BM = MASK << 2;
      const int s0 = (j % FPW) * FB, s1 = ((j + 1) % FPW) * FB;
      const uint32_t w0 = wd[j / FPW - W0], w1 = wd[(j + 1) / FPW - W0];
      const uint32_t a0 = (((s0 >= 2) ? (w0 >> (s0 >= 2 ? s0 - 2 : 0)) : (w0 << (s0 < 2 ? 2 - s0 : 0))) & BM) | tab;
      const uint32_t a1 = (((s1 >= 2) ? (w1 >> (s1 >= 2 ? s1 - 2 : 0)) : (w1 << (s1 < 2 ? 2 - s1 : 0))) & BM) | tab;
      uint32_t t0, t1;
      asm("ld.shared.u32 %0, [%1];\n" : "=r"(t0) : "r"(a0));
      asm("ld.shared.u32 %0, [%1];\n" : "=r"(t1) : "r"(a1));
      hi[e] = __byte_perm(t0, t1, 0x5410);
      lo[e] = __byte_perm(t0, t1, 0x7632);
    }
    tmem_st8(ta + J0 / 2 + g * 8, hi);
    tmem_st8(ta + DP / 2 + J0 / 2 + g * 8, lo);
  }
}

// v[j] for a warp-uniform j without local memory: a 4-level select tree
__device__ __forceinline__ uint32_t pick16(const uint32_t (&v)[16], int j) {
  uint32_t a[8], b[4], c[2];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (j & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = (j & 2) ? a[2 * i + 1] : a[2 * i];
#pragma unroll
  for (int i = 0; i < 2; ++i) c[i] = (j & 4) ? b[2 * i + 1] : b[2 * i];
  return (j & 8) ? c[1] : c[0];
}

template <int FB, int DP, int KL>
__global__ void __launch_bounds__(kThreads, 1) scan_vq_kernel(Params P) {
  constexpr int C = 1 << FB;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(4 * C) uint32_t s_tab[C];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Layout& Lo = P.lo;
  const int NS = P.NS, W = P.st.words_per_vec;
  uint64_t* bars = (uint64_t*)(smem + Lo.bars);
  uint64_t* st_full = bars + kBStF;
  uint64_t* st_empty = bars + kBStE;
  uint64_t* a_full = bars + kBAF;
  uint64_t* a_empty = bars + kBAE;
  uint64_t* acc_full = bars + kBAccF;
  uint64_t* acc_empty = bars + kBAccE;
  uint64_t* b_full = bars + kBBF;
  uint64_t* b_empty = bars + kBBE;
  uint64_t* it_full = bars + kBItF;
  uint64_t* it_empty = bars + kBItE;
  uint64_t* item_done = bars + kBDone;
  uint64_t* slot_ready = bars + kBReady;
  uint64_t* meta_full = bars + kBMF;
  uint64_t* meta_empty = bars + kBME;
  uint32_t* misc = (uint32_t*)(smem + Lo.misc);  // [0] tmem base
  float* thr = (float*)(smem + Lo.thr);          // [2][kQM] lowered filter thresholds
  float* thr_raw = (float*)(smem + Lo.thr_raw);  // [2][kQM] unlowered
  unsigned long long* lists = (unsigned long long*)(smem + Lo.lists);  // [4][kQM][k]
  auto stage = [&](int s) { return smem + Lo.stage + (uint32_t)s * Lo.stage_bytes; };
  auto meta_at = [&](uint32_t t) { return smem + Lo.meta + (t % kMeta) * Lo.meta_bytes; };
  auto rec_at = [&](int j) { return (ItemRec*)(smem + Lo.items + (uint32_t)(j % kItems) * Lo.item_bytes); };

  for (int c = tid; c < C; c += kThreads) {
    uint32_t lo;
    const uint32_t hi = split_pack((float)P.levels[c] * P.t_scale, lo);
    s_tab[c] = hi | (lo << 16);
  }
  for (int i = tid; i < 4 * kQM * P.k; i += kThreads) lists[i] = 0ull;
  if (warp == kMma) sm100::tmem_alloc(misc, 512);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      sm100::mbar_init(&st_full[s], 1);
      sm100::mbar_init(&st_empty[s], kDecWarps);
    }
    for (int b = 0; b < 2; ++b) {
      sm100::mbar_init(&a_full[b], kDecWarps);
      sm100::mbar_init(&a_empty[b], 1);
      sm100::mbar_init(&acc_full[b], 1);
      sm100::mbar_init(&acc_empty[b], kEpiWarps);
      sm100::mbar_init(&b_full[b], 1);
      sm100::mbar_init(&b_empty[b], 1);
      sm100::mbar_init(&item_done[b], kEpiWarps);
      sm100::mbar_init(&slot_ready[b], 1);
    }
    for (int m = 0; m < kMeta; ++m) {
      sm100::mbar_init(&meta_full[m], 4);  // the K-half-0 decoder warps
      sm100::mbar_init(&meta_empty[m], kEpiWarps);
    }
    for (int i = 0; i < kItems; ++i) {
      sm100::mbar_init(&it_full[i], 1);
      sm100::mbar_init(&it_empty[i], 2);  // loader, emitter
    }
    sm100::mbar_fence_init();
  }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = misc[0];
  const uint32_t a_col = 256;  // accumulators at [0, 256), A buffers after

  if (warp == kProd) {
    // ================= producer (+ item scheduler) =============================
    // Item records are fetched one item ahead of the tiles being issued (the
    // loader builds the next item's B operand while this item streams), and
    // the fetch latency sits behind the stage ring. Per tile: the control
    // record, then one lane issues the TMA bulk copies of codes, norms, ids.
    const int n_items = *P.n_items;
    uint32_t t = 0, jf = 0;
    bool fetched_all = false;
    auto publish_next = [&]() {
      for (;;) {
        int item = 0;
        if (lane == 0) item = atomicAdd(P.counter, 1);
        item = __shfl_sync(kFull, item, 0);
        if (jf >= (uint32_t)kItems) VWAITS(&it_empty[jf % kItems], ((jf / kItems) - 1) & 1, 1);
        ItemRec* rec = rec_at(jf);
        if (item >= n_items) {
          if (lane == 0) {
            rec->list = -1;
            sm100::mbar_arrive(&it_full[jf % kItems]);
          }
          ++jf;
          fetched_all = true;
          return;
        }
        const int2 it = P.items[item];
        const int l = it.x;
        const int pbase = P.pstart[l] + it.y * kQM;
        const int nq = min(kQM, P.pstart[l + 1] - pbase);
        const int size = P.st.list_size[l];
        const int ntiles = (size + kNV - 1) / kNV;
        if (nq <= 0) continue;
        if (ntiles == 0) {  // empty list: its pairs' candidate slots stay empty
          for (int x = lane; x < nq * P.k; x += 32) {
            const int p = P.pair_idx[pbase + x / P.k];
            const long long o = (long long)(p / P.n_p) * P.qcap + (long long)(p % P.n_p) * P.k + x % P.k;
            P.part_s[o] = -INFINITY;
            P.part_id[o] = INT_MAX;
          }
          continue;
        }
        const long long off = P.st.list_offset[l];
        int qv[kQM / 32], rv[kQM / 32];
        double cv[kQM / 32];
#pragma unroll
        for (int r = 0; r < kQM / 32; ++r) {
          const int row = r * 32 + lane;
          const int p = row < nq ? P.pair_idx[pbase + row] : -1;
          qv[r] = p >= 0 ? p / P.n_p : -1;
          rv[r] = p >= 0 ? p - qv[r] * P.n_p : 0;
          cv[r] = p >= 0 ? P.coarse[p] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < kQM / 32; ++r) {
          rec->q[r * 32 + lane] = qv[r];
          rec->rank[r * 32 + lane] = rv[r];
          rec->cs[r * 32 + lane] = cv[r];
        }
        if (lane == 0) {
          rec->list = l;
          rec->nq = nq;
          rec->N = (nq + 15) & ~15;
          rec->ntiles = ntiles;
          rec->size = size;
          rec->off = off;
        }
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&it_full[jf % kItems]);
        ++jf;
        return;
      }
    };
    publish_next();
    for (uint32_t j = 0;; ++j) {
      if (!fetched_all) publish_next();  // record j+1, one item ahead
      const ItemRec* rec = rec_at(j);
      const int l = rec->list, nq = rec->nq, N = rec->N, ntiles = rec->ntiles, size = rec->size;
      const long long off = rec->off;
      __syncwarp();
      if (l < 0) {
        const int s = t % NS;
        if (t >= (uint32_t)NS) VWAITS(&st_empty[s], ((t / NS) - 1) & 1, 2);
        if (lane == 0) {
          ((Ctrl*)(stage(s) + Lo.st_ctrl))->list = -1;
          sm100::mbar_arrive(&st_full[s]);
        }
        break;
      }
      for (int i = 0; i < ntiles; ++i, ++t) {
        const int s = t % NS;
        if (t >= (uint32_t)NS) VWAITS(&st_empty[s], ((t / NS) - 1) & 1, 3);
        if (lane == 0) {
          unsigned char* sp = stage(s);
          Ctrl* c = (Ctrl*)(sp + Lo.st_ctrl);
          c->list = l;
          c->tile = i;
          c->ntiles = ntiles;
          c->valid = min(kNV, size - i * kNV);
          c->item = (int)j;
          c->nq = nq;
          c->N = N;
          const long long s0 = off + (long long)i * kNV;
          const uint32_t cb = kNV * W * 4, nb = kNV * 2, ib = kNV * 4;
          sm100::mbar_arrive_expect_tx(&st_full[s], cb + nb + ib);
          sm100::bulk_g2s(sp, P.st.codes + (s0 >> 5) * W * 32, cb, &st_full[s]);
          sm100::bulk_g2s(sp + Lo.st_norms, P.st.norms + s0, nb, &st_full[s]);
          sm100::bulk_g2s(sp + Lo.st_ids, P.st.ids + s0, ib, &st_full[s]);
          VTRACE(0, clock64());
          VTRACE(7, i | (ntiles << 12) | ((long long)nq << 24));
        }
        __syncwarp();
      }
    }
  } else if (warp == kLoad) {
    // ================= query loader (B operand) ===============================
    // Row r of the item -> K-major canonical layout, no swizzle: 16-byte
    // chunk ch (8 dims) of row r at ch*(kQM*16) + (r/8)*128 + (r%8)*16, hi
    // image first, lo image DP*kQM*2 bytes later. Rows past nq are zero.
    constexpr int NCH = DP / 8;
    for (uint32_t j = 0;; ++j) {
      VWAITS(&it_full[j % kItems], (j / kItems) & 1, 4);
      const ItemRec* rec = rec_at(j);
      const int l = rec->list, nq = rec->nq, N = rec->N;
      if (l < 0) break;
      const int b = j & 1;
      if (j >= 2) VWAITS(&b_empty[b], ((j >> 1) - 1) & 1, 5);
      unsigned char* bq = smem + (b ? Lo.bq[1] : Lo.bq[0]);
      const int total = N * NCH * 2;
#pragma unroll 1
      for (int base = 0; base < total; base += 32 * 8) {
        uint4 v[8];
        uint32_t dst[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = base + u * 32 + lane;
          const int part = idx >= N * NCH;
          const int rem = idx - part * N * NCH;
          const int r = rem / NCH, ch = rem - r * NCH;
          const bool ok = idx < total && r < nq;
          const int q = ok ? rec->q[r] : 0;
          const uint4* src = (const uint4*)((part ? P.q_lo : P.q_hi) + (size_t)q * (DP / 2)) + ch;
          v[u] = ok ? __ldg(src) : make_uint4(0, 0, 0, 0);
          dst[u] = idx < total ? (uint32_t)part * (DP * kQM * 2) + ch * (kQM * 16) + (r >> 3) * 128 +
                                     (r & 7) * 16
                               : 0xffffffffu;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (dst[u] != 0xffffffffu) *(uint4*)(bq + dst[u]) = v[u];
      }
      sm100::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        sm100::mbar_arrive(&b_full[b]);
        sm100::mbar_arrive(&it_empty[j % kItems]);
      }
    }
  } else if (warp == kMma) {
    // ================= MMA issuer ==============================================
    uint32_t t = 0;
    for (;;) {
      const int ab = t & 1;
      VWAIT(&a_full[ab], (t >> 1) & 1, 6);
      const Ctrl c = *(const Ctrl*)meta_at(t);  // written before a_full
      // the buffer's previous tile must be consumed even before the stop
      // record: a phase completed early would alias the epilogue's parity
      if (t >= 2) VWAIT(&acc_empty[ab], ((t >> 1) - 1) & 1, 7);
      if (c.list < 0) {
        if (lane == 0) sm100::mbar_arrive(&acc_full[ab]);
        break;
      }
      const int bs = c.item & 1;
      if (c.tile == 0) VWAIT(&b_full[bs], (c.item >> 1) & 1, 8);
      sm100::tc_fence_after();
      if (lane == 0) VTRACE(2, clock64());
      const uint32_t idesc = sm100::idesc_f16_f32(kNV, c.N);
      const uint32_t dt = tmem + ab * kQM;
      const uint32_t at = tmem + a_col + ab * DP;
      const uint32_t bh = sm100::smem_u32(smem + (bs ? Lo.bq[1] : Lo.bq[0]));
      const uint32_t bl = bh + DP * kQM * 2;
      const uint32_t lbo = kQM * 16, sbo = 128;
      const uint64_t dh = sm100::smem_desc(bh, lbo, sbo), dl = sm100::smem_desc(bl, lbo, sbo);
      const uint64_t dstep = (2 * lbo) >> 4;
#pragma unroll
      for (int pass = 0; pass < 3; ++pass) {
        const uint32_t a = pass == 2 ? at + DP / 2 : at;
        const uint64_t db = pass == 1 ? dl : dh;
#pragma unroll
        for (int ks = 0; ks < DP / 16; ++ks)
          sm100::mma_f16_ts_warp(dt, a + ks * 8, db + ks * dstep, idesc, (pass | ks) ? 1u : 0u);
      }
      sm100::mma_commit_warp(&a_empty[ab]);
      sm100::mma_commit_warp(&acc_full[ab]);
      if (c.tile == c.ntiles - 1) sm100::mma_commit_warp(&b_empty[bs]);
      __syncwarp();
      VTRACE(3, clock64());
      ++t;
    }
  } else if (warp >= kDec0 && warp < kDec0 + kDecWarps) {
    // ================= decoders ================================================
    const int quad = warp & 3, kh = (warp - kDec0) >> 2;
    const int v = quad * 32 + lane;
    uint32_t t = 0;
    for (;;) {
      const int s = t % NS, ab = t & 1;
      VWAITS(&st_full[s], (t / NS) & 1, 9);
      if (warp == kDec0) VTRACE(6, clock64());
      unsigned char* sp = stage(s);
      const Ctrl c = *(const Ctrl*)(sp + Lo.st_ctrl);
      if (kh == 0) {
        // tile record for the MMA issuer and the epilogue: the stage slot
        // goes back to the producer as soon as this tile is decoded
        if (t >= (uint32_t)kMeta) VWAITS(&meta_empty[t % kMeta], ((t / kMeta) - 1) & 1, 10);
        unsigned char* mp = meta_at(t);
        if (warp == kDec0 && lane == 0) *(Ctrl*)mp = c;
        if (c.list >= 0) {
          const bool ok = v < c.valid;
          ((float*)(mp + sizeof(Ctrl)))[v] =
              ok ? __half2float(__ushort_as_half(((const uint16_t*)(sp + Lo.st_norms))[v])) * P.inv_scale
                 : __int_as_float(0x7fc00000);
          ((int*)(mp + sizeof(Ctrl) + kNV * 4))[v] = ((const int*)(sp + Lo.st_ids))[v];
        }
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&meta_full[t % kMeta]);
      }
      if (t >= 2) VWAITS(&a_empty[ab], ((t >> 1) - 1) & 1, 11);  // (also before a stop: parity)
      if (c.list < 0) {
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&a_full[ab]);
        break;
      }
      sm100::tc_fence_after();
      const uint32_t* cw = (const uint32_t*)sp + (v >> 5) * W * 32 + (v & 31);
      const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + a_col + ab * DP;
#ifdef IVFTQ_EXP_NODEC
      if (c.nq < 0)  // experiment build: decode skipped (timing bound only)
#endif
      {
        if (kh == 0)
          decode_half<FB, DP, 0>(cw, W, sm100::smem_u32(s_tab), ta);
        else
          decode_half<FB, DP, 1>(cw, W, sm100::smem_u32(s_tab), ta);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        sm100::mbar_arrive(&a_full[ab]);
        sm100::mbar_arrive(&st_empty[s]);
      }
      if (warp == kDec0) VTRACE(1, clock64());
      ++t;
    }
  } else if (warp >= kEpi0 && warp < kEpi0 + kEpiWarps) {
    // ================= epilogue (filter + per-quadrant top-k) =================
    // Thread = vector (TMEM lane). Per 16-query window: one TMEM load, one
    // FFMA per pair against the query's threshold, one max. Each warp owns its
    // lane quadrant's top-k of every query it filters (no cross-warp sharing)
    // and inserts survivors warp-cooperatively: the list is spread over lanes
    // 0..k-1, each survivor's key broadcast and placed by a ballot of the
    // entries above it plus a one-lane shift. A full list raises the query's
    // threshold and its global bound. At the item's end the four quadrant
    // lists of each query are merged and written to the pair's fixed slot of
    // the candidate buffer.
    const int quad = warp & 3, wpar = (warp - kEpi0) >> 2;
    const int v = quad * 32 + lane;
    const int kk = P.k;
    unsigned long long* qlists = lists + (size_t)quad * kQM * kk;  // this quadrant's lists
    uint32_t t = 0;
    for (;;) {
      const int ab = t & 1;
      VWAIT(&acc_full[ab], (t >> 1) & 1, 12);
      VWAIT(&meta_full[t % kMeta], (t / kMeta) & 1, 13);
      const unsigned char* mp = meta_at(t);
      const Ctrl c = *(const Ctrl*)mp;
      if (c.list < 0) break;
      const int ls = c.item & 1;
      const ItemRec* irec = rec_at((uint32_t)c.item);
      if (c.tile == 0) VWAIT(&slot_ready[ls], (c.item >> 1) & 1, 14);
      sm100::tc_fence_after();
      if (warp == kEpi0) VTRACE(4, clock64());
      const float ns = ((const float*)(mp + sizeof(Ctrl)))[v];  // NaN past the list's end
      const int id = ((const int*)(mp + sizeof(Ctrl) + kNV * 4))[v];
      float* th = thr + ls * kQM;
      float* thraw = thr_raw + ls * kQM;
      const uint32_t tl = tmem + ((uint32_t)(quad * 32) << 16) + ab * kQM;
#ifdef IVFTQ_EXP_NOEPI
      const int nwin = 0;  // experiment build: epilogue skipped (timing bound only)
#else
      const int nwin = c.N >> 4;
#endif
#pragma unroll 1
      for (int win = wpar; win < nwin; win += 2) {
        uint32_t r[16];
        tmem_ld16(tl + win * 16, r);
        float tv[16];
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          const float4 f4 = *(const float4*)(th + win * 16 + e);
          tv[e] = f4.x;
          tv[e + 1] = f4.y;
          tv[e + 2] = f4.z;
          tv[e + 3] = f4.w;
        }
        sm100::tmem_ld_wait();
        float diff[16];
        float mx = -INFINITY;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          diff[e] = __fmaf_rn(__uint_as_float(r[e]), ns, -tv[e]);
          mx = fmaxf(mx, diff[e]);
        }
#ifdef IVFTQ_EXP_NOPUSH
        if (__any_sync(kFull, mx >= 0.f) && c.nq < 0) {  // experiment: survivors dropped
#else
        if (__any_sync(kFull, mx >= 0.f)) {
#endif
          uint32_t pend = 0;
#pragma unroll
          for (int e = 0; e < 16; ++e) pend |= (diff[e] >= 0.f ? 1u : 0u) << e;
          VCOUNT(0, __popc(pend));
          uint32_t qm = __reduce_or_sync(kFull, pend);
          while (qm) {
            const int e = __ffs(qm) - 1;
            qm &= qm - 1;
            uint32_t me = __ballot_sync(kFull, (pend >> e) & 1u);
            const int row = win * 16 + e;
            unsigned long long* Lp = qlists + (size_t)row * kk;
            // one round of shared loads: this quadrant's list (lane = entry),
            // the four quadrants' witness entries i* (lanes 0-3, see below)
            // and the query's current raw threshold
            unsigned long long lv = lane < kk ? Lp[lane] : 0ull;
            unsigned long long w = lane < 4 ? lists[((size_t)lane * kQM + row) * kk + ((kk + 3) >> 2) - 1]
                                            : ~0ull;
            const float traw = thraw[row];
            const unsigned long long mykey = cand_key(__fmul_rn(__uint_as_float(pick16(r, e)), ns), id);
            bool changed = false;
            while (me) {
              const int src = __ffs(me) - 1;
              me &= me - 1;
              const unsigned long long key = __shfl_sync(kFull, mykey, src);
              const int pos = __popc(__ballot_sync(kFull, lane < kk && lv > key));
              if (pos < kk) {  // warp-uniform
                const unsigned long long up = __shfl_up_sync(kFull, lv, 1);
                lv = lane == pos ? key : (lane > pos && lane < kk ? up : lv);
                changed = true;
              }
            }
            if (changed) {
              if (lane < kk) Lp[lane] = lv;
              // Pair bound: each quadrant list holds real candidates, so if
              // every quadrant has an entry i* (i* = ceil(k/4) - 1), their
              // minimum has >= 4(i*+1) >= k candidates at or above it; and this
              // quadrant's k-th has k. Entries only ever improve, so the
              // witnesses read above (this quadrant's from before the inserts)
              // stay valid.
              w = min(w, __shfl_xor_sync(kFull, w, 1));
              w = min(w, __shfl_xor_sync(kFull, w, 2));
              const unsigned long long kth = max(__shfl_sync(kFull, lv, kk - 1), w);
              if (kth && lane == 0) {
                VCOUNT(1, 1);
                const float kr = key_score(kth);
                if (kr > traw) {  // racing quadrants: any written value is a valid bound
                  thraw[row] = kr;
                  th[row] = lower_thr(kr);
                  // mid-item publication to the other CTAs' items of this query
                  atomicMax(&P.thr_key[irec->q[row]], dkey(irec->cs[row] + (double)kr));
                }
              }
            }
          }
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        sm100::mbar_arrive(&acc_empty[ab]);
        sm100::mbar_arrive(&meta_empty[t % kMeta]);
      }
      if (c.tile == c.ntiles - 1) {
        // item end: the four quadrant warps of this window parity merge
        // their lists per query (thread i of the 128 <-> query i of the parity)
        __syncwarp();  // bar.sync is .aligned: the whole warp, converged
        named_bar(1 + wpar, 128);
        const int i = quad * 32 + lane;
        const int row = ((i >> 4) * 2 + wpar) * 16 + (i & 15);
        if (row < c.nq) {
          unsigned long long top[KL];
#pragma unroll
          for (int x = 0; x < KL; ++x) top[x] = x < KL - kk ? ~0ull : 0ull;  // k-th best at top[KL-1]
          for (int qd = 0; qd < 4; ++qd) {
            unsigned long long* Lp = lists + ((size_t)qd * kQM + row) * kk;
            for (int p = 0; p < kk; ++p) {
              const unsigned long long key = Lp[p];
              Lp[p] = 0ull;
              if (!key) break;  // sorted: the rest is empty
              bool g[KL];
#pragma unroll
              for (int x = 0; x < KL; ++x) g[x] = key > top[x];
#pragma unroll
              for (int x = KL - 1; x > 0; --x) top[x] = g[x] ? (g[x - 1] ? top[x - 1] : key) : top[x];
              top[0] = g[0] ? key : top[0];
            }
          }
          const int q = irec->q[row];
          const double cs = irec->cs[row];
          const long long o = (long long)q * P.qcap + (long long)irec->rank[row] * kk;
#pragma unroll
          for (int x = 0; x < KL; ++x)
            if (x >= KL - kk) {
              const unsigned long long key = top[x];
              P.part_s[o + x - (KL - kk)] = key ? cs + (double)key_score(key) : -INFINITY;
              P.part_id[o + x - (KL - kk)] = key ? key_id(key) : INT_MAX;
            }
          if (top[KL - 1]) atomicMax(&P.thr_key[q], dkey(cs + (double)key_score(top[KL - 1])));
        }
        __syncwarp();
        named_bar(1 + wpar, 128);  // lists clear before the next item's inserts
        if (lane == 0) sm100::mbar_arrive(&item_done[ls]);
      }
      if (warp == kEpi0) VTRACE(5, clock64());
      ++t;
    }
  } else if (warp == kEmit) {
    // ================= emitter: per-item thresholds ============================
    // Item j's threshold slot (j & 1) opens once item j-2 is done: each
    // query's threshold from its global bound. While items run, thresholds
    // follow the global bounds the other CTAs raise.
    auto refresh = [&](uint32_t j) {
      const ItemRec* rec = rec_at(j);
      const int ls = j & 1, nq = rec->nq;
      long long kq[kQM / 32];
#pragma unroll
      for (int x = 0; x < kQM / 32; ++x) {
        const int r = x * 32 + lane;
        kq[x] = r < nq ? *(volatile const long long*)&P.thr_key[rec->q[r]] : LLONG_MIN;
      }
#pragma unroll
      for (int x = 0; x < kQM / 32; ++x) {
        const int r = x * 32 + lane;
        if (r < nq) {
          const float gb = prune_bound(kq[x], rec->cs[r]);
          if (gb > thr_raw[ls * kQM + r]) {  // a racing insert may win: both are valid bounds
            thr_raw[ls * kQM + r] = gb;
            thr[ls * kQM + r] = lower_thr(gb);
          }
        }
      }
    };
    for (uint32_t j = 0;; ++j) {
      VWAITS(&it_full[j % kItems], (j / kItems) & 1, 15);
      const bool stop = rec_at(j)->list < 0;
      if (j >= 2) {  // slot j & 1 is free once item j-2 is done
        const uint32_t e = j - 2;
        while (!mbar_test(&item_done[e & 1], (e >> 1) & 1)) {
          refresh(j - 1);
          refresh(e);
          __nanosleep(1000);
        }
        ITRACE(e, 2);
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&it_empty[e % kItems]);
      }
      if (stop) break;
      const ItemRec* rec = rec_at(j);
      const int ls = j & 1, nq = rec->nq;
      for (int r = lane; r < kQM; r += 32) {
        thr_raw[ls * kQM + r] = r < nq ? -INFINITY : INFINITY;
        thr[ls * kQM + r] = r < nq ? -INFINITY : INFINITY;
      }
      __syncwarp();
      refresh(j);
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&slot_ready[ls]);
      ITRACE(j, 3);
    }
  }
  __syncthreads();
  if (warp == kMma) sm100::tmem_dealloc(tmem, 512);
}

}  // namespace vq

// ---- host side ----------------------------------------------------------------
// Deepest stage ring (3..kMaxNS) that fits in shared memory; 0 = unsupported.
static int vq_stages(int DP, int W, int k) {
  // 227 KB opt-in, less the static shared memory (~1 KB) and the 1 KB the
  // launch adds for aligning the dynamic base
  const size_t limit = 227 * 1024 - 1024 - 1024 - 256;
  for (int ns = vq::kMaxNS; ns >= 3; --ns)
    if (vq::make_layout(DP, W, ns, k).total <= limit) return ns;
  return 0;
}

bool scan_vq_supported(int dim, int field_bits_, int depth) {
  if (getenv("IVFTQ_SCAN_OLD")) return false;
  const int DP = (dim + 31) / 32 * 32;
  if (DP > 128 || field_bits_ < 3 || field_bits_ > 5 || depth < 1 || depth > 16) return false;
  return vq_stages(DP, words_per_vec(dim, field_bits_), depth) > 0;
}

template <int FB, int DP>
static int launch_vq_t(const vq::Params& P, size_t smem, int grid, cudaStream_t s) {
  auto fn = vq::scan_vq_kernel<FB, DP, 16>;
  if (int e = smem_opt_in_dev((const void*)fn, smem)) return e;
  fn<<<grid, vq::kThreads, smem, s>>>(P);
  return check_launch("scan_vq");
}

// Called by ivftq_scan_topk_tc after the regroup, seeding and query split.
int launch_scan_vq(const ivftq_store* st, const double* coarse, const double* levels,
                   const int32_t* pairs, const int32_t* pstart, const int2* items,
                   const int32_t* n_items, int32_t* counter, double* part_s, int32_t* part_id,
                   int32_t* qcnt, long long* thr_key, const uint32_t* q_hi, const uint32_t* q_lo,
                   int n_p, int depth, int qcap, cudaStream_t s) {
  vq::Params P{};
  const char* trace_path = getenv("IVFTQ_TRACE");
  if (trace_path) {
    cudaMalloc(&P.trace, sizeof(long long) * (vq::kTraceTiles * 8 + 8 + vq::kTraceItems * 4));
    cudaMemsetAsync(P.trace, 0, sizeof(long long) * (vq::kTraceTiles * 8 + 8 + vq::kTraceItems * 4), s);
  }
  const int DP = (st->dim + 31) / 32 * 32;
  P.st = *st;
  P.coarse = coarse;
  P.pair_idx = pairs;
  P.pstart = pstart;
  P.items = items;
  P.n_items = n_items;
  P.counter = counter;
  P.part_s = part_s;
  P.part_id = part_id;
  P.qcnt = qcnt;
  P.thr_key = thr_key;
  P.q_hi = q_hi;
  P.q_lo = q_lo;
  P.levels = levels;
  P.n_p = n_p;
  P.k = depth;
  P.d = st->dim;
  P.qcap = qcap;
  P.NS = vq_stages(DP, st->words_per_vec, depth);
  P.t_scale = ldexpf(1.0f, 12);
  P.inv_scale = ldexpf(1.0f, -(12 + 14));
  P.lo = vq::make_layout(DP, st->words_per_vec, P.NS, depth);
  const size_t smem = P.lo.total + 1024;
  const int grid = device_sm_count();
  const int fb = st->field_bits;
  int rc = IVFTQ_ERR_UNSUPPORTED;
#define VQ_DP(FBV)                                                   \
  switch (DP) {                                                      \
    case 32: rc = launch_vq_t<FBV, 32>(P, smem, grid, s); break;     \
    case 64: rc = launch_vq_t<FBV, 64>(P, smem, grid, s); break;     \
    case 96: rc = launch_vq_t<FBV, 96>(P, smem, grid, s); break;     \
    default: rc = launch_vq_t<FBV, 128>(P, smem, grid, s); break;    \
  }
  if (fb == 3) { VQ_DP(3) }
  else if (fb == 4) { VQ_DP(4) }
  else if (fb == 5) { VQ_DP(5) }
  else set_error("scan_vq: field width %d", fb);
#undef VQ_DP
  if (P.trace) {
    static long long h[vq::kTraceTiles * 8 + 8 + vq::kTraceItems * 4];
    cudaMemcpyAsync(h, P.trace, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (FILE* f = fopen(trace_path, "w")) {
      fprintf(f, "# vq NS=%d survivors=%lld inserts=%lld\n# t prod dec_end mma_s mma_e epi_s epi_e dec_s tile nt nq\n",
              P.NS, h[vq::kTraceTiles * 8], h[vq::kTraceTiles * 8 + 1]);
      const long long b = h[0];
      for (int t = 0; t < vq::kTraceTiles && h[t * 8]; ++t) {
        fprintf(f, "%d", t);
        for (int k = 0; k < 7; ++k) fprintf(f, " %lld", h[t * 8 + k] ? h[t * 8 + k] - b : -1);
        fprintf(f, " %lld %lld %lld\n", h[t * 8 + 7] & 4095, (h[t * 8 + 7] >> 12) & 4095, h[t * 8 + 7] >> 24);
      }
      fclose(f);
    }
    std::string ip = std::string(trace_path) + ".items";
    if (FILE* f = fopen(ip.c_str(), "w")) {
      fprintf(f, "# j - - emitted slot_ready (rel. first TMA)\n");
      const long long b = h[0];
      const long long* it = h + vq::kTraceTiles * 8 + 8;
      for (int j = 0; j < vq::kTraceItems && (it[j * 4] || it[j * 4 + 3]); ++j)
        fprintf(f, "%d %lld %lld %lld %lld\n", j, it[j * 4] ? it[j * 4] - b : -1,
                it[j * 4 + 1] ? it[j * 4 + 1] - b : -1, it[j * 4 + 2] ? it[j * 4 + 2] - b : -1,
                it[j * 4 + 3] ? it[j * 4 + 3] - b : -1);
      fclose(f);
    }
    cudaFree(P.trace);
  }
  return rc;
}

}  // namespace ivftq
