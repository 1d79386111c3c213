/*
 * dpq.h — C ABI of libdpq.so, the B200 (sm_100a) implementation of the
 * two-pass derived-codebook PQ search of arXiv 1905.06900.
 *
 * The reference (`derivedpq`, /root/reference/pkg) is pure Python/numpy and
 * has no FFI layer; its drop-in boundary is the public search API:
 *
 *   FlatIndex.search(Y, r, mode, r2, capped, return_timings)   flat.py:54-108
 *   IVFIndex.search(Y, r, ma, mode, r2, capped, return_timings) ivf.py:125-160
 *
 * Every entry point below replaces the arithmetic of one of those calls (or of
 * one of the unit-level seams the reference tests call), with plain pointers
 * and sizes, no torch types.  Argument validation that produces the
 * reference's Python exceptions stays in the Python mirror
 * (paper_1905_06900_b200/flat.py, ivf.py); the C side returns a status code
 * and a thread-local message (dpq_last_error).
 *
 * Conventions
 *  - All host pointers are plain C-contiguous arrays.  "_dev" variants take
 *    device pointers on the index's device and run on the index's stream.
 *  - Codes are (n, m) little-endian uint8 (b <= 8) or uint16 (b <= 16),
 *    row-major, exactly quantizer.py:78 / :169.
 *  - Results are (nq, r) float64 distances padded with +inf and int64 ids
 *    padded with -1 (flat.py:16-29).
 *  - Return value: DPQ_OK (0) or a DPQ_ERR_* code; dpq_last_error() explains.
 */
#ifndef DPQ_H_
#define DPQ_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DPQ_OK 0
#define DPQ_ERR_ARG 1    /* invalid argument (maps to ValueError)      */
#define DPQ_ERR_CUDA 2   /* CUDA runtime / kernel failure              */
#define DPQ_ERR_NOMEM 3  /* device or pinned allocation failed         */
#define DPQ_ERR_STATE 4  /* wrong index kind / not initialised         */

typedef struct dpq_index dpq_index_t;

/* Thread-local description of the last failure on this thread. */
const char* dpq_last_error(void);
/* ABI version (bumped on any signature change). */
int dpq_abi_version(void);
/* Number of visible CUDA devices (0 on a CPU-only host, never an error). */
int dpq_device_count(void);
/* Host-side finiteness scan of n float32 values (the input check of
 * sklearn check_array that flat.py:71 / ivf.py:125 run on the queries):
 * 0 = all finite, 1 = contains NaN, 2 = contains +-inf (NaN wins).  No GPU. */
int dpq_all_finite(const float* x, int64_t n);

/* quantizer.rotate (quantizer.py:235-239) in the reference's call shapes,
 * for n rows of x (n, d) f32: rows_per_call = 1 is the per-query (1, d) @ R
 * of the flat search (twopass.py:334), rows_per_call = ma the per-query
 * (ma, d) @ R of the IVF residuals (ivf.py:202).  sgemv / sgemm are the
 * CBLAS entry points of the BLAS numpy itself links (ilp64 = 1 for 64-bit
 * integer builds); every call is numpy's own (sgemv RowMajor/Trans for one
 * row, sgemm RowMajor/NoTrans for a block), so the bits are the reference's,
 * and the calls run on `threads` host threads.  No GPU.                   */
int dpq_rotate_rows(const float* x, int64_t n, int64_t rows_per_call, int d,
                    const float* rotation, float* out, void* sgemv,
                    void* sgemm, int ilp64, int threads);

/* ---------------------------------------------------------------- flat --
 * Replaces the fitted state FlatIndex holds after fit (flat.py:45-52):
 * quantizer.codebooks_ (m,k,dsub) f32, quantizer.derived_codebooks_
 * (m,kbar,dsub) f32 and codes_ (n,m).  The handle owns device copies; the
 * caller's buffers may be freed after the call.  id_base is added to every
 * returned id (0 for an unsharded index; the shard's first global row when a
 * database is split across GPUs).
 * prefix_codes/n_prefix: the rows qmax is estimated from
 * (twopass.py:83-84 uses codes[:min(r2,n)]).  Pass NULL/0 to use the
 * handle's own first rows; a shard passes the replicated global prefix.    */
int dpq_flat_create(int device, int m, int k, int kbar, int dsub,
                    const float* codebooks, const float* derived_codebooks,
                    const void* codes, int code_bytes, int64_t n,
                    int64_t id_base, const void* prefix_codes,
                    int64_t n_prefix, dpq_index_t** out);

/* ----------------------------------------------------------------- ivf --
 * Replaces IVFIndex's fitted state (ivf.py:63-103): centers_ (K,d) f32,
 * offsets_ (K+1) i64, sorted_codes_ (n,m), sorted_ids_ (n) i64, plus the
 * residual quantizer's codebooks.                                         */
int dpq_ivf_create(int device, int m, int k, int kbar, int dsub,
                   const float* codebooks, const float* derived_codebooks,
                   int n_cells, const float* centers, const int64_t* offsets,
                   const void* sorted_codes, int code_bytes,
                   const int64_t* sorted_ids, int64_t n, dpq_index_t** out);

void dpq_destroy(dpq_index_t* index);

/* Use an external CUDA stream (cudaStream_t as void*); NULL = own stream. */
int dpq_set_stream(dpq_index_t* index, void* stream);
/* Query batch size used internally (default 1024). */
int dpq_set_batch(dpq_index_t* index, int batch);
/* Enable per-phase CUDA-event timing (dpq_last_phase_ms). */
int dpq_set_timing(dpq_index_t* index, int enabled);
/* Validate host query buffers inside the flat searches (the finiteness part of
 * sklearn check_array that flat.py:71 runs first): the scan rides on the
 * staging copy of each batch.  A NaN or +-inf makes the search return
 * DPQ_ERR_ARG with a dpq_last_error() that starts with "non-finite query"
 * before any result is written; the caller then raises the reference's error
 * (paper_1905_06900_b200/flat.py re-runs check_array for its message). */
int dpq_set_check_finite(dpq_index_t* index, int enabled);

/* ------------------------------------------------------ flat searches --
 * dpq_flat_search_derived: FlatIndex.search(..., mode="derived", r2)
 * (flat.py:94-104 -> nns_derived, twopass.py:311-353) for nq queries.
 *   yr        (nq, d) f32 host, queries AFTER quantizer.rotate in the
 *             reference's call shape (identity for plain PQ).
 *   phase_us  optional (nq, 4) f64 host: index/tables/scan/refine µs per
 *             query (batched phases amortised per query), or NULL.
 * `capped` is accepted for signature parity; the retained candidate set is
 * identical either way (SURVEY Appendix A rule 8).                        */
int dpq_flat_search_derived(dpq_index_t* index, const float* yr, int64_t nq,
                            int r, int r2, int capped, double* dists,
                            int64_t* ids, double* phase_us);
/* Device-pointer twin: yr/dists/ids on the index's device. */
int dpq_flat_search_derived_dev(dpq_index_t* index, const float* yr,
                                int64_t nq, int r, int r2, double* dists,
                                int64_t* ids);

/* FlatIndex.search(..., mode="conventional") (flat.py:82-93): full
 * (m,k) tables, adc over all n codes, exact top-r.                        */
int dpq_flat_search_conventional(dpq_index_t* index, const float* yr,
                                 int64_t nq, int r, double* dists,
                                 int64_t* ids, double* phase_us);

/* ------------------------------------------------------- ivf searches --
 * IVFIndex.probe (ivf.py:107-120): the ma nearest cells (f64 distances,
 * ties to the lower cell id).  cells (nq, ma) i64 host.                   */
int dpq_ivf_probe(dpq_index_t* index, const float* y, int64_t nq, int ma,
                  int64_t* cells);
/* IVFIndex.search(..., mode="derived") (ivf.py:195-277).
 *   y         (nq, d) raw queries (host).
 *   res_rot   optional (nq, ma, d) rotated residuals computed by the caller
 *             with quantizer.rotate in the (ma, d) call shape (OPQ); NULL
 *             means identity rotation (residual y - center formed on
 *             device in f32, exactly ivf.py:120).
 *   cells     optional (nq, ma) probe result matching res_rot; NULL probes
 *             on device.                                                  */
int dpq_ivf_search_derived(dpq_index_t* index, const float* y, int64_t nq,
                           int r, int ma, int r2, int capped,
                           const float* res_rot, const int64_t* cells,
                           double* dists, int64_t* ids, double* phase_us);
int dpq_ivf_search_conventional(dpq_index_t* index, const float* y,
                                int64_t nq, int r, int ma,
                                const float* res_rot, const int64_t* cells,
                                double* dists, int64_t* ids,
                                double* phase_us);

/* ----------------------------------------------------- sharded (flat) --
 * Split form of dpq_flat_search_derived for a database split into
 * contiguous row shards, one per GPU.  Each shard's handle is
 * created with its rows, id_base = its first global row and the replicated
 * global prefix (the first min(N, max r2) rows, twopass.py:83-84), so every
 * shard quantizes with the same global qmin/qmax.  The caller exchanges
 * two small histograms between the phases (sum over shards, e.g. an NCCL
 * all-reduce) and merges the per-shard top-r by (dist, id):
 *   1. dpq_shard_begin: small tables + a score histogram of a row sample of
 *      this shard (all rows when exact != 0)
 *        -> sample_hist (nq,256) i32 and *n_sampled      [sum over shards]
 *   2. dpq_shard_scan: guard per query from the summed sample histogram
 *      (identical on every shard), scan, local histogram of the emitted
 *      scores (all <= guard)  -> cand_hist (nq,256) i32  [sum over shards]
 *   3. dpq_shard_finish: b* per query from the summed candidate histogram;
 *      refine local candidates (score <= b*), local top-r with global ids
 *        -> dists/ids (nq,r), need_exact (nq) u8: 1 where the guard proved
 *      too tight; the caller then repeats 1-3 with exact = 1.
 * The union of the shards' candidates is the unsharded candidate set, so the
 * merged top-r equals the unsharded result bit for bit.  Host buffers.     */
int dpq_shard_begin(dpq_index_t* index, const float* yr, int64_t nq, int r2,
                    int64_t n_global, int exact, int32_t* sample_hist,
                    int64_t* n_sampled);
int dpq_shard_scan(dpq_index_t* index, const int32_t* sample_hist_sum,
                   int64_t n_global, int64_t sample_global, int r2,
                   int exact, int32_t* cand_hist);
int dpq_shard_finish(dpq_index_t* index, const int32_t* cand_hist_sum,
                     int r, int r2, double* dists, int64_t* ids,
                     uint8_t* need_exact);

/* Device-resident form of the same protocol: every buffer is a device
 * pointer on the index's device and every call only enqueues work on the
 * index stream (no host synchronisation), so the caller runs the two
 * histogram all-reduces in place on that stream (NCCL) between the calls.
 * Instead of redoing internally, a query whose guard proved too tight (1)
 * or whose emit list overflowed on this shard (2) is flagged in `flags`
 * (nq u8, device); the caller all-reduces the flags (max) and repeats a
 * flagged batch through the host-buffer protocol above (exact = 1).
 * n_sampled is written on the host at once (it depends only on the
 * shard's size).  The per-shard top-r of all shards, all-gathered as
 * (n_parts, nq, r), is merged by dpq_merge_topr_dev.                      */
int dpq_shard_begin_dev(dpq_index_t* index, const float* yr, int64_t nq,
                        int r2, int64_t n_global, int exact,
                        int32_t* sample_hist, int64_t* n_sampled);
int dpq_shard_scan_dev(dpq_index_t* index, const int32_t* sample_hist_sum,
                       int64_t n_global, int64_t sample_global, int r2,
                       int exact, int32_t* cand_hist);
int dpq_shard_finish_dev(dpq_index_t* index, const int32_t* cand_hist_sum,
                         int r, int r2, double* dists, int64_t* ids,
                         uint8_t* flags);
/* Exact (dist, id) top-r of n_parts per-shard top-r lists, each sorted and
 * padded with (+inf, -1): part_dists/part_ids (n_parts, nq, r) device ->
 * dists/ids (nq, r) device (ResultSet.from_arrays over the union,
 * search.py:115-124).  Enqueued on the index stream.                      */
int dpq_merge_topr_dev(dpq_index_t* index, const double* part_dists,
                       const int64_t* part_ids, int n_parts, int64_t nq,
                       int r, double* dists, int64_t* ids);
/* Wait for everything enqueued on the index stream. */
int dpq_sync(dpq_index_t* index);

/* ------------------------------------------------- sharded (ivf) --
 * IVF list-split sharding: every inverted list is cut evenly
 * across the shards, keeping cell order; each shard's handle is created
 * with dpq_ivf_create over its slice of every list (sorted_ids = GLOBAL
 * ids) and then told the global lists: global_offsets (K+1) and, per list,
 * its first min(prefix_rows, len) global rows (prefix_codes, row offsets
 * prefix_offsets (K+1)) — the rows qmax is estimated from (ivf.py:205-217;
 * r2 <= prefix_rows).  The protocol mirrors the flat one, host buffers:
 *   1. dpq_ivf_shard_begin: probe (identical on every shard), per-cell
 *      tables, bounds from the first non-empty GLOBAL probed list, score
 *      histogram of this shard's sampled rows -> sample_hist (nq,256),
 *      n_sampled (nq) [sum both over shards]; n_rows (nq) = rows of the
 *      probed global lists (identical on every shard); exact != 0 samples
 *      every row.
 *   2. dpq_ivf_shard_scan: guards from the sums, scan of the local slices
 *      -> cand_hist (nq,256) [sum over shards]
 *   3. dpq_ivf_shard_finish: b*, refine of the local candidates in their
 *      own cell frames, local top-r with global ids; need_exact (nq) = 1
 *      where the guard proved too tight (repeat 1-3 with exact = 1).
 * The merged top-r (dpq_merge_topr_dev or the host merge) equals the
 * unsharded IVFIndex.search result bit for bit.                          */
int dpq_ivf_set_shard(dpq_index_t* index, const int64_t* global_offsets,
                      const void* prefix_codes, const int64_t* prefix_offsets,
                      int64_t prefix_rows);
int dpq_ivf_shard_begin(dpq_index_t* index, const float* y, int64_t nq,
                        int ma, int r2, int exact, const float* res_rot,
                        const int64_t* cells, int32_t* sample_hist,
                        int64_t* n_sampled, int64_t* n_rows);
int dpq_ivf_shard_scan(dpq_index_t* index, const int32_t* sample_hist_sum,
                       const int64_t* sampled_sum, const int64_t* rows_sum,
                       int r2, int32_t* cand_hist);
int dpq_ivf_shard_finish(dpq_index_t* index, const int32_t* cand_hist_sum,
                         int r, int r2, double* dists, int64_t* ids,
                         uint8_t* need_exact);

/* ------------------------------------------------ unit seams (debug) --
 * Replace compute_tables(yr, derived_codebooks_) + quantize_tables
 * (search.py:28-48, twopass.py:63-85) for nq queries: small (nq,m,kbar) f32,
 * q (nq,m,kbar) u8, qmin/qmax (nq) f64.                                   */
int dpq_debug_quantize_tables(dpq_index_t* index, const float* yr,
                              int64_t nq, int r2, float* small, uint8_t* q,
                              double* qmin, double* qmax);
/* adc_low_batch (twopass.py:99-106) of every code for nq queries, with
 * the tables quantize_tables (twopass.py:63-85) builds from the first
 * min(r2, n) codes: scores (nq, n) u8 in the caller's row order.          */
int dpq_debug_low_scores(dpq_index_t* index, const float* yr, int64_t nq,
                         int r2, uint8_t* scores);
/* The candidate ids refine scores (scan_derived -> CappedBuckets ->
 * refine's bucket walk, twopass.py:171-217, 276-302), in walk order:
 * ascending score, ties by ascending id.  For query q, counts[q] = number
 * of candidates; the first min(counts[q], cap) ids go to ids[q*cap ...]
 * and, when scores != NULL, their 8-bit scores to scores[q*cap ...].
 * Call with cap = 0 to size the buffers.                                  */
int dpq_debug_candidate_ids(dpq_index_t* index, const float* yr, int64_t nq,
                            int r2, int64_t cap, int64_t* ids,
                            uint8_t* scores, int64_t* counts);
/* CappedBuckets bound + refine walk (twopass.py:171-201, 276-308):
 * bstar (nq) i32 and ncand (nq) i64 = |{s <= b*, s < 255}|.               */
int dpq_debug_candidates(dpq_index_t* index, const float* yr, int64_t nq,
                         int r2, int32_t* bstar, int64_t* ncand);
/* compute_tables(yr, codebooks_) (search.py:28-48), full (nq,m,k) f32.    */
int dpq_debug_full_tables(dpq_index_t* index, const float* yr, int64_t nq,
                          float* tables);

/* Tensor-core full tables (tcgen05 kind::tf32, 3xTF32 with centred
 * operands and cached centroid norms): the approximation of
 * compute_tables(yr, codebooks_) (search.py:28-48) that the derived refine
 * uses when dsub >= 64 (env DPQ_TC_TABLES=0/1 overrides).  tables (nq, m, k)
 * f32 in centroid order, eps (nq, m) f64: a rigorous bound on
 * |tables - numpy's entry| for every entry of (query, subspace).  The search
 * stays bit-exact: candidates within the bound of the r-th best are
 * re-ranked with exact entries.                                           */
int dpq_debug_tc_tables(dpq_index_t* index, const float* yr, int64_t nq,
                        float* tables, double* eps);

/* ------------------------------------------------------------ encoder --
 * Nearest-centroid encoding on the tensor cores (tcgen05, 3xTF32): replaces
 * ProductQuantizer._encode_with (quantizer.py:75-83) -> nearest_centroids
 * (clustering.py:53-77): code[i,j] = argmin_c ||x[i, j*dsub:(j+1)*dsub] -
 * codebooks[j,c]||^2, ties to the lowest index.  Also the IVF coarse
 * assignment (ivf.py:83-101) with m = 1.  The reference's cross term is an
 * f32 BLAS GEMM, so near-ties (equal at f32 rounding) may pick a different
 * minimiser; every other row agrees.  dsub <= 32: one K = 32 GEMM per
 * tile; 32 < dsub <= 128 (4 | k): the K-chunked GEMM of the tensor-core
 * tables (dpq_tctab.cu) with an argmin epilogue.
 *   dpq_encoder_create: codebooks (m,k,dsub) f32 host; the handle owns the
 *     prepared device operand.
 *   dpq_encode:     x (n, m*dsub) f32 host -> codes (n, m) u16 host (k <= 65536).
 *   dpq_encode_dev: x device (n rows, row stride ldx floats) -> codes (n, m)
 *     i32 device, enqueued on `stream` (NULL: the encoder's own stream).   */
typedef struct dpq_encoder dpq_encoder_t;
int dpq_encoder_create(int device, int m, int k, int dsub,
                       const float* codebooks, dpq_encoder_t** out);
void dpq_encoder_destroy(dpq_encoder_t* enc);
int dpq_encode(dpq_encoder_t* enc, const float* x, int64_t n,
               uint16_t* codes);
int dpq_encode_dev(dpq_encoder_t* enc, const float* x, int64_t n,
                   int64_t ldx, int32_t* codes, void* stream);

/* ---------------------------------------------------------- containers --
 * Model/index containers straight to the device: replaces the bulk half of
 * derivedpq.vecio.load_model (vecio.py:156-198).  The Python mirror
 * (container.py) parses the JSON header (vecio.py:177-183) and passes each
 * array's byte range; arrays are read by `threads` host threads into pinned
 * buffers and copied to freshly allocated device buffers (dev_out[a], free
 * with dpq_dev_free) while the next piece is read.  With verify, crc_out[a]
 * is the zlib CRC-32 of array a computed ON THE DEVICE (vecio.py:141,188-192
 * compares it with the header).  stats4 (nullable): bytes read, host read
 * seconds, total seconds, arrays.                                          */
int dpq_container_read(int device, const char* path, int n_arrays,
                       const int64_t* offsets, const int64_t* nbytes,
                       int verify, int threads, void** dev_out,
                       uint32_t* crc_out, double* stats4);
/* zlib CRC-32 of a 16-byte-aligned device buffer (zlib.crc32 semantics). */
int dpq_crc32_dev(int device, const void* data, int64_t len, uint32_t* crc);
int dpq_dev_free(int device, void* p);
int dpq_dev_download(int device, const void* src, int64_t nbytes, void* dst);
/* Device halves of validate() on bulk arrays (flat.py:112-118,
 * ivf.py:280-292): the largest code (-1 if count == 0); ids out of [0, n)
 * (out2[0]) and rows no id maps to (out2[1]) — both 0 iff ids is a
 * permutation of arange(n); counts[c] = |{i : cells[i] == c}| with cells
 * outside [0, n_cells) counted in *n_bad.                                  */
int dpq_dev_codes_max(int device, const void* codes, int64_t count,
                      int code_bytes, int64_t* out_max);
int dpq_dev_check_permutation(int device, const int64_t* ids, int64_t n,
                              int64_t* out2);
int dpq_dev_bincount(int device, const int32_t* cells, int64_t n,
                     int n_cells, int64_t* counts, int64_t* n_bad);

/* ------------------------------------------------------- measurement --
 * Milliseconds of the last batch's phases when timing is enabled:
 * [0] tables (K1), [1] sample+guard, [2] scan (K2), [3] threshold (K3),
 * [4] refine+top-r (K6), [5] fallback, [6] whole batch.                    */
int dpq_last_phase_ms(dpq_index_t* index, float* ms7);
/* Counters since creation (8 x i64): kernel launches, queries searched,
 * code rows scanned (sum over queries), candidates refined, exact-redo
 * rounds, first-pass rows emitted (score <= guard), full-table entries
 * computed by the group-lazy table builder, scan units run by the wide
 * (5/6-bit, 16 queries per lane) loop.                                    */
int dpq_counters(dpq_index_t* index, int64_t* out8);
/* Extended counters (n of them; unknown slots read 0): [0..7] as
 * dpq_counters, [8] code-plane rows the first-pass scan read (summed over
 * query tiles; 4 or 8 B each), [9] LUT tile loads of the scan (128 KB each).
 * With [5] (emitted entries, 8 B each) they give the scan's bytes moved.
 * [10] candidates re-ranked exactly after tensor-core tables, [11] exact
 * f64 centre distances computed by the tensor-core IVF probe.           */
int dpq_counters_ex(dpq_index_t* index, int64_t* out, int n);

#ifdef __cplusplus
}
#endif
#endif /* DPQ_H_ */
