/*
 * ivftq_b200.h -- C ABI of the B200-native IVF-TQ search + ingest hot path.
 *
 * The reference (`ivftq`, pure Python/numpy, /root/reference/pkg/src/ivftq)
 * has no FFI; its boundary is the Python `IvfTqIndex` API (index.py:162-500).
 * Every entry point below replaces one numpy stage of that path and is what
 * a host binding (ctypes here) calls. Conventions:
 *
 *   - all array pointers are DEVICE pointers unless the name says `host`;
 *   - the library never allocates or frees caller memory: scratch is passed
 *     in, sized by the matching *_scratch_bytes query;
 *   - every launch is asynchronous on the caller's `stream` (cudaStream_t
 *     passed as void*, NULL = legacy default stream);
 *   - return value 0 = success, < 0 = an IVFTQ_ERR_* code; the message is in
 *     ivftq_last_error() (thread-local);
 *   - concurrency: calls from different host threads, on different streams
 *     or different devices, are independent. The library's only internal
 *     state is per device (SM count, shared-memory opt-ins; mutex-guarded)
 *     or per (host thread, device) (the side stream and fork/join events a
 *     scan uses internally, the kernel-timing events). Internal forks are
 *     joined back into the caller's stream on every return path, so a call
 *     inside a stream capture never leaves the capture forked. Process-wide
 *     switches: ivftq_set_coarse_mode (configuration, atomic).
 */
#ifndef IVFTQ_B200_H
#define IVFTQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IVFTQ_ABI_VERSION 3  /* 3: + k-means (seed, assign_tc64, sums), tensor-core encoder tail */

#define IVFTQ_OK 0
#define IVFTQ_ERR_ARG (-1)
#define IVFTQ_ERR_CUDA (-2)
#define IVFTQ_ERR_SCRATCH (-3)
#define IVFTQ_ERR_UNSUPPORTED (-4)

#define IVFTQ_F32 0
#define IVFTQ_F64 1

/* Device-resident inverted lists (replaces CoarsePartition.lists +
 * IvfTqIndex._bins/_signs/_norms, index.py:177-185, partition.py:34).
 * List l owns slots [list_offset[l], list_offset[l] + list_cap[l]); offsets and
 * capacities are multiples of 128 slots. Codes of 32 consecutive slots form a
 * block: word w of slot s is codes[((s/32)*words_per_vec + w)*32 + s%32].
 * Each word packs `fields_per_word` coordinates of field_bits = bits+1 bits
 * (field value bin*2+sign; the sign is stored even when use_sign is 0, as the
 * reference stores `signs` unconditionally), coordinate j of the word at bit
 * field_bits*j. levels[] tables are indexed by the field value. Slot order inside a list is arbitrary: every result is
 * ordered by (score desc, internal id asc), never by slot. */
typedef struct ivftq_store {
  int32_t dim;
  int32_t bits;
  int32_t use_sign;
  int32_t n_lists;
  int32_t field_bits;
  int32_t fields_per_word;
  int32_t words_per_vec;
  int32_t max_list_size; /* host-maintained upper bound of list_size[] */
  const int64_t* list_offset; /* [n_lists] */
  const int32_t* list_size;   /* [n_lists] */
  uint32_t* codes;            /* [capacity/32][words_per_vec][32] */
  uint16_t* norms;            /* [capacity] binary16 residual norms */
  int32_t* ids;               /* [capacity] internal id, -1 = empty slot */
  int64_t capacity;           /* slots */
} ivftq_store;

/* ---- host-only utilities (no GPU needed) -------------------------------- */
const char* ivftq_last_error(void);
int ivftq_abi_version(void);
/* Number of kernels this library has launched in the process (bench evidence). */
unsigned long long ivftq_launch_count(void);
/* Adds n to that count: the host side calls it on each CUDA-graph replay of
 * a captured search (n = kernels captured), since a replay launches them
 * without passing through this library. */
void ivftq_note_graph_launches(unsigned long long n);
/* Code layout for (dim, bits, use_sign). */
int ivftq_code_layout(int dim, int bits, int use_sign, int* field_bits,
                      int* fields_per_word, int* words_per_vec);
/* float64 -> binary16 bits, round-to-nearest-even, the rule of
 * `rnorm.astype(np.float16)` (index.py:255). Host memory. */
int ivftq_host_double_to_half(const double* host_x, int64_t n, uint16_t* host_out);
/* Pairwise sum-of-squares row norms, numpy's np.linalg.norm(axis=1) order
 * (index.py:241). Host memory; used to pin the device routine on the CPU. */
int ivftq_host_row_norms(const double* host_x, int64_t n, int dim, double* host_out);

/* ---- ingest: IvfTqIndex._encode_batch (index.py:231-267) ---------------- */
/* x (n, dim) f32 or f64 -> xn = x/||x|| f64 (index.py:238-245).
 * *bad_row (device) receives the first row with ||x|| < 1e-12, or n. */
int ivftq_normalize_rows(const void* x, int x_dtype, int64_t n, int dim,
                         double* xn, int64_t* bad_row, void* stream);
/* C = A . B^T, A (M,K) f64 row-major, B (N,K) f32/f64 row-major, C (M,N)
 * f64/f32: coarse scores (index.py:436), rotations (rotation.py:40). */
int ivftq_gemm_nt(const double* A, const void* B, int b_dtype, int64_t M, int N,
                  int K, void* C, int c_dtype, void* stream);
/* Max-IP list per row, ties -> lowest list (partition.py:45-55), f64 DFMA. */
int ivftq_assign(const double* xn, const float* centroids, int64_t n, int n_lists,
                 int dim, int32_t* list_out, void* stream);
/* Same decision on the tensor cores: error-compensated fp16 tcgen05 GEMM keeps
 * each row's best four approximate scores, then every centroid within the
 * error band of the maximum is re-scored in exact f64 (identical values and
 * tie rule to ivftq_assign). Falls back to ivftq_assign when unsupported. */
size_t ivftq_assign_tc_scratch_bytes(int64_t n, int n_lists, int dim);
int ivftq_assign_tc(const double* xn, const float* centroids, int64_t n, int n_lists,
                    int dim, int32_t* list_out, void* scratch, size_t scratch_bytes,
                    void* stream);
/* ---- GPU spherical k-means for the partition refresh (partition.py:64-178,
 * refresh.py:171-175): seeding, Lloyd assignment, Lloyd sums -------------- */
/* Lloyd-step assignment on f64 centroids (partition.py:149-150): the same
 * tensor-core pass + exact f64 decision as ivftq_assign_tc, ties to the lower
 * list. scratch >= ivftq_assign_tc_scratch_bytes(n, n_lists, dim). */
int ivftq_assign_tc64(const double* xn, const double* centroids, int64_t n, int n_lists,
                      int dim, int32_t* list_out, void* scratch, size_t scratch_bytes,
                      void* stream);
/* k-means++ seeding (partition.py:_kmeanspp, 83-113) entirely on the device.
 * X (n, dim) f64 unit rows; `first` = the host's rng.integers(n);
 * host_uniforms (k-1, nc) = the host's rng.random(nc) of every step in order,
 * nc = ivftq_kmeanspp_candidates(k) = 2 + floor(log2 k). chosen_out[k]
 * (device) receives the centre rows; totals_out[k] (device) the potential
 * total before each step (entry 0 unused): a total <= 1e-12 means the
 * reference's degenerate branch applies and the caller must seed on its
 * checked path instead. */
int ivftq_kmeanspp_candidates(int k);
size_t ivftq_kmeanspp_scratch_bytes(int64_t n, int dim, int k);
int ivftq_kmeanspp_seed(const double* X, int64_t n, int dim, int k, int64_t first,
                        const double* host_uniforms, int64_t* chosen_out,
                        double* totals_out, void* scratch, size_t scratch_bytes,
                        void* stream);
/* Lloyd update (partition.py:153-160): counts_out[l] rows per list and
 * sums_out[l] = the list's rows, in ascending row order, added in the order
 * of np.add.reduceat over the stably sorted rows (first row + numpy's pairwise
 * sum of the rest): bit-identical f64 sums. */
size_t ivftq_kmeans_sums_scratch_bytes(int64_t n, int n_lists);
int ivftq_kmeans_sums(const double* X, const int32_t* list_ids, int64_t n, int dim,
                      int n_lists, double* sums_out, int32_t* counts_out, void* scratch,
                      size_t scratch_bytes, void* stream);
/* out[i] = x_i . C[list_ids[i]] (partition.py:162, the empty-list rule's key). */
int ivftq_rowdot64(const double* X, const double* C, const int32_t* list_ids, int64_t n,
                   int dim, double* out, void* stream);
/* *differ (device) = 1 when the two assignments differ anywhere (partition.py:151). */
int ivftq_lists_differ(const int32_t* a, const int32_t* b, int64_t n, int32_t* differ,
                       void* stream);
/* Coarse-scoring path selection (results are identical in every mode):
 * 0 = default: assignment and probes on tensor cores with the exact f64 guard
 *     band whenever the shape is supported (padded dim <= 256, n_p <= 128),
 *     else the f64 GEMM + exact select;
 * 1 = f64 CUDA-core GEMMs only (parity reference);
 * 2 = same as 0 (kept for ABI compatibility; also IVFTQ_PROBE_TC=1). */
int ivftq_set_coarse_mode(int mode);
int ivftq_coarse_tc_supported(int dim, int n_lists);
/* Pre-split centroid operand images for the tensor-core coarse GEMM. */
size_t ivftq_coarse_prep_bytes(int n_lists, int dim);
int ivftq_coarse_prepare(const float* centroids, int n_lists, int dim, void* prep,
                         void* stream);
/* Residual r = xn - c_l (or xn when flat), ||r|| -> binary16 (index.py:247-255). */
int ivftq_residuals(const double* xn, const float* centroids, const int32_t* list_ids,
                    int64_t n, int dim, int flat, double* resid_out,
                    uint16_t* norm_out, void* stream);
/* unit = rot/||rot||, Lloyd-Max bin + half-bin sign (lloydmax.py:129-144),
 * packed into words_per_vec words per row; rows whose binary16 norm is 0
 * get all-zero codes (index.py:257-262). */
int ivftq_quantize_pack(const double* rot, const uint16_t* norms, int64_t n, int dim,
                        int bits, int use_sign, const double* boundaries,
                        const double* qcent, uint32_t* words_out, void* stream);
/* Tensor-core encoder tail (index.py:247-262 after the assignment), used by
 * ivftq_encode whenever ivftq_encode_supported_tc(dim): one kernel forms
 * r = xn - c_l, ||r|| -> binary16 (both bit-exact) and the unit row r/||r|| as
 * fp16 hi/lo tensor-core operands (no f64 intermediate returns to HBM); the
 * rotation u' = (r/||r||).R^T runs on tcgen05 (error-compensated fp16, f32
 * accumulation in TMEM); Lloyd-Max bins and signs are taken from u', and
 * every row with a coordinate within the guard width (2^-18) of a bin boundary
 * or half-bin centroid is re-encoded by an exact f64 pass, so the codes equal
 * the f64 path's. ivftq_rotate_unit_tc exposes the first two steps (U (n, dim)
 * f32 on the device) so the guard can be pinned against an f64 rotation. */
int ivftq_encode_supported_tc(int dim);
size_t ivftq_encode_tc_scratch_bytes(int64_t n, int dim);
int ivftq_rotate_unit_tc(const double* xn, const float* centroids, const int32_t* list_ids,
                         int64_t n, int dim, int flat, const double* R, float* U_out,
                         uint16_t* norm_out, void* scratch, size_t scratch_bytes,
                         void* stream);
int ivftq_encode_tail_tc(const double* xn, const float* centroids, const int32_t* list_ids,
                         int64_t n, int dim, int bits, int use_sign, int flat,
                         const double* R, const double* boundaries, const double* qcent,
                         uint16_t* norm_out, uint32_t* words_out, void* scratch,
                         size_t scratch_bytes, void* stream);
/* Whole encoder: normalize -> assign -> residual -> rotate -> quantize/pack.
 * scratch >= ivftq_encode_scratch_bytes(n, dim, n_lists). Outputs per row: xn (f64, for
 * the raw store; may alias nothing), list id, binary16 norm, code words. */
size_t ivftq_encode_scratch_bytes(int64_t n, int dim, int n_lists);
int ivftq_encode(const void* x, int x_dtype, int64_t n, int dim, int bits, int use_sign,
                 int flat, const float* centroids, int n_lists, const double* R,
                 const double* boundaries, const double* qcent, double* xn_out,
                 int64_t* bad_row, int32_t* list_out, uint16_t* norm_out,
                 uint32_t* words_out, void* scratch, size_t scratch_bytes,
                 void* stream);
/* Re-pack per-vector unpacked bins/signs (n, dim) u8 into code words
 * (storage load path, storage.py:152-158). */
int ivftq_pack_codes(const uint8_t* bins, const uint8_t* signs, int64_t n, int dim,
                     int bits, int use_sign, uint32_t* words_out, void* stream);

/* ---- list store (index.py:300-308 per-row list append) ------------------ */
int ivftq_histogram(const int32_t* list_ids, int64_t n, int n_lists, int32_t* counts,
                    void* stream);
/* Append n encoded rows with internal ids first_id.. into their lists.
 * cursor: [n_lists] int32 zeroed by the call. slot_of: [>= first_id+n]. */
int ivftq_append(const ivftq_store* store, const uint32_t* words, const uint16_t* norms,
                 const int32_t* list_ids, int64_t n, int64_t first_id,
                 int32_t* cursor, int64_t* slot_of, void* stream);
/* Move every list from src's segments to dst's (capacity growth). */
int ivftq_relayout(const ivftq_store* src, const ivftq_store* dst, int64_t* slot_of,
                   void* stream);
/* Unpack rows [first, first+n) by internal id to (n, dim) bins / signs u8
 * (the `bins`/`signs` views, index.py:319-325). signs may be NULL. */
int ivftq_export_codes(const ivftq_store* store, const int64_t* slot_of, int64_t first,
                       int64_t n, uint8_t* bins, uint8_t* signs, void* stream);
/* Apply XOR masks to stored codes in place, by internal id (bit_flip_ablation,
 * index.py:578-594): mask (n, dim) u8 of field bits to flip. */
int ivftq_xor_codes(const ivftq_store* store, const int64_t* slot_of, int64_t n,
                    const uint8_t* mask, int which /*0 bins,1 signs*/, int flip,
                    void* stream);

/* ---- search: IvfTqIndex.search_batch (index.py:409-483) ------------------ */
/* Per row of `scores` (rows, cols) f64: the n largest by (value desc, col asc)
 * -> idx_out/val_out (rows, n), the stable argsort probe order (index.py:438). */
int ivftq_select_topn(const double* scores, int64_t rows, int cols, int n,
                      int32_t* idx_out, double* val_out, void* stream);
/* Coarse probes (index.py:436-438): stable top-n_p of qn.C^T. Tensor-core
 * scores + exact f64 re-scoring of the guard band when supported, else the
 * f64 GEMM + select; both return identical probes, and exact f64 coarse
 * values that differ only in summation order (a few ulps). The path depends
 * only on the shape (and ivftq_set_coarse_mode), never on the batch size. */
size_t ivftq_probe_scratch_bytes(int64_t nq, int n_lists, int dim);
int ivftq_probe(const double* qn, const float* centroids, int64_t nq, int n_lists,
                int dim, int n_p, int32_t* probe_out, double* coarse_out,
                void* scratch, size_t scratch_bytes, void* stream);
/* The same with the centroids' tensor-core operand images already made by
 * ivftq_coarse_prepare (ivftq_coarse_prep_bytes(n_lists, dim) bytes) for this
 * centroid set: a caller that searches one index many times prepares once.
 * `centroids` is still read by the f64 fallback. */
int ivftq_probe_prepared(const double* qn, const float* centroids, const void* prepared,
                         int64_t nq, int n_lists, int dim, int n_p, int32_t* probe_out,
                         double* coarse_out, void* scratch, size_t scratch_bytes,
                         void* stream);
/* List scan + per-query top-`depth` (index.py:441-483): score =
 * coarse + (double)(||r|| * sum_j qrot_j * levels[code_j]). levels: f64
 * flattened reconstruction table (lloydmax.py:146-150). ids are internal. */
size_t ivftq_scan_scratch_bytes(int64_t nq, int n_p, int depth, int n_lists);
int ivftq_scan_topk(const ivftq_store* store, const int32_t* probe, const double* coarse,
                    const float* qrot, const double* levels, int64_t nq, int n_p,
                    int depth, int64_t* ids_out, double* scores_out, void* scratch,
                    size_t scratch_bytes, void* stream);
/* Query-major LUT scan (any bits, depth <= 7936): one CTA per (query, probe
 * split) builds lut[j][c] = qrot_j * T[c] in shared memory. */
int ivftq_scan_topk_lut(const ivftq_store* store, const int32_t* probe, const double* coarse,
                        const float* qrot, const double* levels, int64_t nq, int n_p,
                        int depth, int64_t* ids_out, double* scores_out, void* scratch,
                        size_t scratch_bytes, void* stream);
/* List-major tensor-core scan (bits 2..4, depth <= 32): probes regrouped by
 * list; per (list, 128-query tile) the decoded codes meet the queries in
 * tcgen05.mma (fp16 hi/lo error-compensated, fp32 accumulate in TMEM). */
int ivftq_scan_tc_supported(int dim, int bits, int depth);
size_t ivftq_scan_tc_scratch_bytes(int64_t nq, int n_p, int n_lists, int depth);
int ivftq_scan_topk_tc(const ivftq_store* store, const int32_t* probe, const double* coarse,
                       const float* qrot, const double* levels, int64_t nq, int n_p,
                       int depth, int64_t* ids_out, double* scores_out, void* scratch,
                       size_t scratch_bytes, void* stream);
/* Instrumentation: bracket the tensor-core scan kernel with CUDA events on its
 * stream; ivftq_last_scan_kernel_ms() syncs and returns the last duration. */
int ivftq_set_kernel_timing(int on);
/* Current timing switch (a captured search graph records the events only if
 * it was captured with timing on; the host keys its graphs on this). */
int ivftq_get_kernel_timing(void);
double ivftq_last_scan_kernel_ms(void);
/* Name of the list-scan kernel the calling thread's last tensor-core scan ran
 * ("scan_vq_kernel" or "scan_tc_kernel"); "" before the first. */
const char* ivftq_last_scan_kernel(void);
/* Exact re-score of the top-depth candidates against the raw f32 store and
 * re-order to top-k (index.py:470-473). */
int ivftq_rerank(const float* raw, const double* qn, const int64_t* cand_ids,
                 int64_t nq, int depth, int dim, int k, int64_t* ids_out,
                 double* scores_out, void* stream);
/* Decode rows by internal id: c_l + ||r|| R^T T[code], optionally renormalised
 * (refresh.reconstruct_all, refresh.py:63-81). R_T is the TRANSPOSED rotation
 * (row-major R^T), so the device GEMM computes T[code] . R. */
int ivftq_decode(const ivftq_store* store, const int64_t* slot_of,
                 const int32_t* list_of, int64_t n, const float* centroids,
                 const double* R_T, const double* levels, int flat, int renormalize,
                 double* out, void* scratch, size_t scratch_bytes, void* stream);
size_t ivftq_decode_scratch_bytes(int64_t n, int dim);
/* out[i] = <a_i, c_{l_i}> in f64 (refresh report IPs, refresh.py:179-187). */
int ivftq_rowdot(const double* a, const float* centroids, const int32_t* list_ids,
                 int64_t n, int dim, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* IVFTQ_B200_H */
