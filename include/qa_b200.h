/*
 * qa_b200.h -- C-ABI of the B200-native int8 exhaustive k-NN path.
 *
 * Drop-in boundary for the reference package's kernel seam
 * (quantann._backend, /root/reference/pkg/src/quantann/_backend.py:14-46).
 * Each entry point names the reference routine it replaces.  All functions:
 *
 *   * are plain C (no C++/torch types), thread-safe (an internal mutex
 *     serialises use of the per-device workspace);
 *   * return QA_OK (0) or a nonzero QA_E* code; the message for the last
 *     failure on the calling thread is available from qa_last_error();
 *   * take DEVICE pointers unless the name ends in _host, and a CUDA stream
 *     (cudaStream_t passed as void*, NULL = legacy default stream) on which
 *     all work is enqueued.  Device variants are asynchronous except where
 *     noted; _host variants are synchronous.
 *
 * Error mapping used by the Python shim (paper_2110_08919_b200/_lib.py):
 *   QA_EINVAL       -> ValueError with the reference's message
 *                      (_core.pyx:340-347, 357-358)
 *   QA_EUNSUPPORTED -> NotImplementedError (shape outside this build's limits)
 *   QA_ECUDA/ENOMEM -> RuntimeError
 *   QA_EIO          -> OSError; QA_ETRUNCATED / QA_ENONPOSITIVE / QA_EDIM ->
 *                      TruncatedRecord / NonPositiveDim / DimensionMismatch
 *                      with the reference's messages (dataset.py:160-209)
 *
 * Metric codes are the reference's (distances.py:22-27):
 *   0 = INNER_PRODUCT (score = -dot), 1 = L2_SQUARED, 2 = ANGULAR (1 - cos).
 */
#ifndef QA_B200_H
#define QA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    QA_OK = 0,
    QA_EINVAL = 1,
    QA_ECUDA = 2,
    QA_ENOMEM = 3,
    QA_EUNSUPPORTED = 4,
    QA_EIO = 5,          /* OSError (open/read/write failed) */
    QA_ETRUNCATED = 6,   /* TruncatedRecord (errors.py) */
    QA_ENONPOSITIVE = 7, /* NonPositiveDim */
    QA_EDIM = 8,         /* DimensionMismatch */
    QA_EZERONORM = 9     /* ZeroNorm: angular with a norm <= 0 (exact.py:67-69) */
};

/* Library identification. */
int qa_version(void);
const char *qa_last_error(void);
/* Number of visible CUDA devices (0 when no driver/GPU); never fails. */
int qa_device_count(void);
/* Row stride (bytes) this build uses for int8 code matrices of width d:
 * 32, 64 or a multiple of 128 -- the K granularity of the tcgen05 kind::i8
 * MMA and the TMA swizzle width.  Pad columns are zero. */
int64_t qa_code_stride(int64_t d);

/* ---- calibration (quantizer.py:176-267; BASELINE min/max + symmetric) ----
 * Per-dimension min and max of a float32 matrix x[n, ldx] (first d columns).
 * Exact (order-free); NaN entries are ignored like numpy's fmin/fmax would
 * NOT -- they propagate as in numpy min/max (result NaN for that column). */
int qa_minmax_f32(const float *x, int64_t n, int64_t d, int64_t ldx,
                  float *out_min, float *out_max, void *stream);

/* The reference's full calibration statistics, estimate_stats
 * (quantizer.py:176-222), bit-exact with its numpy evaluation: per-dimension
 * mean and MLE sigma (sequential float64 sums over rows), min, max, the
 * 0.1% / 99.9% order statistics (qlo/qhi, may be NULL) and the trimmed
 * abs-max; pooled mean/sigma by numpy's pairwise summation over 64-column
 * blocks.  x: DEVICE float32 [n, ldx]; every output a HOST array of d doubles
 * (two scalars for pooled).  Synchronous.  n < 2 -> QA_EINVAL (TooFewSamples
 * is raised one level up, quantizer.py:181-182). */
int qa_estimate_stats_f32(const float *x, int64_t n, int64_t d, int64_t ldx, double *mu,
                          double *sigma, double *mn, double *mx, double *tam, double *qlo,
                          double *qhi, double *pooled_mu, double *pooled_sigma, void *stream);

/* ---- encode (quantizer.py:291-300 _quantize_matrix; 303-320 callers) ----
 * codes[i, j] = Eq. 1 code of x[i, j] under per-dim window (k, sb, se) with
 * `bits` in [1, 8], bit-exact with numpy's float32 evaluation order.  codes
 * has row stride ldc >= d (bytes); columns [d, ldc) are written as zero.
 * Optional (may be NULL) per-row outputs of the encoded vector:
 *   sqnorm[i] = sum_j codes[i,j]^2 (int32), norm[i] = float(sqrt(double(sqnorm)))
 * (_core.pyx:137-157 norms, int8 branch). */
int qa_encode_i8(const float *x, int64_t n, int64_t d, int64_t ldx,
                 const float *k, const float *sb, const float *se, int bits,
                 int8_t *codes, int64_t ldc, int32_t *sqnorm, float *norm,
                 void *stream);

/* ---- norms (_core.pyx:137-157, int8 branch) ---- */
int qa_norms_i8(const int8_t *codes, int64_t n, int64_t d, int64_t ldc,
                int32_t *sqnorm, float *norm, void *stream);

/* ---- distances to listed rows (the service a graph traversal calls) ----
 * out_scores[q, j] = the reference's pair score _pair_i(query q, row
 * cand[q, j]) (_core.pyx:88-96) -- what HnswCore._dq / _dist_rows compute one
 * pair at a time (_core.pyx:472-494): L2 -> (double)l2, IP -> -dot, angular ->
 * 1 - dot / (qn * xn).  cand is int32 [nq, ldcand] (m used per row); an id
 * outside [0, n) yields +inf (padding of ragged neighbour lists).
 * row_of_id (int32 [n] or NULL) maps a caller id to its stored row when the
 * database is kept in an index layout.  Code rows as produced by
 * qa_encode_i8 (stride a multiple of 16, zero padded). */
int qa_gather_scores_i8(const int8_t *db, int64_t n, int64_t d, int64_t ldd,
                        const int32_t *db_sqnorm, const float *db_norm,
                        const int32_t *row_of_id,
                        const int8_t *q, int64_t nq, int64_t ldq,
                        const int32_t *q_sqnorm, const float *q_norm,
                        const int32_t *cand, int64_t m, int64_t ldcand, int metric,
                        double *out_scores, void *stream);

/* ---- exhaustive top-k (_core.pyx:301-365 scan_topk/_scan_i8) ----
 * db[n, ldd] and q[nq, ldq] are int8 codes with ldd, ldq == qa_code_stride(d)
 * (zero padded).  db_sqnorm/q_sqnorm (int32) are required for metric 1,
 * db_norm/q_norm (float32, strictly positive) for metric 2; others may be
 * NULL.  row_ids (optional, int32[n]) maps stored row -> reported id; it lets
 * an index keep its rows in a different order (e.g. sorted by norm, see
 * qa_order_rows_by_norm) and still report, and break ties by, the caller's
 * ids.  Writes keff = min(k, n) entries per query, ascending by
 * (score, id): out_scores float64[nq, keff], out_ids int32[nq, keff] where
 * id = (row_ids ? row_ids[row] : row) + id_offset.  Synchronises `stream`
 * once at the end (overflow check of the candidate buffers).  Angular with a
 * norm <= 0 returns QA_EZERONORM (the reference's exact.py raises ZeroNorm
 * before its scan; its raw _core would order NaN/inf scores).  keff <= 2048
 * runs the tensor-core filter + select; 2048 < keff <= 15360 runs the
 * float64-exact scan on the codes (bit-identical results, slower); larger
 * keff returns QA_EUNSUPPORTED. */
int qa_scan_topk_i8(const int8_t *db, int64_t n, int64_t d, int64_t ldd,
                    const int32_t *db_sqnorm, const float *db_norm,
                    const int32_t *row_ids,
                    const int8_t *q, int64_t nq, int64_t ldq,
                    const int32_t *q_sqnorm, const float *q_norm,
                    int64_t k, int metric, int64_t id_offset,
                    double *out_scores, int32_t *out_ids, void *stream);

/* Asynchronous form of qa_scan_topk_i8 (same arguments and results): returns
 * once the search is enqueued on `stream`, with no host synchronisation.
 * Queries whose candidate list overflowed or whose threshold estimate failed
 * are recomputed on the device (a full exact scan, still in stream order), so
 * the outputs are final when the stream reaches them.  Differences: a zero
 * angular norm is not reported (callers check norms, as exact.py does), and
 * the per-call candidate statistics are not collected.  Calls sharing a
 * device's workspace must use one stream. */
int qa_scan_topk_i8_async(const int8_t *db, int64_t n, int64_t d, int64_t ldd,
                          const int32_t *db_sqnorm, const float *db_norm,
                          const int32_t *row_ids,
                          const int8_t *q, int64_t nq, int64_t ldq,
                          const int32_t *q_sqnorm, const float *q_norm,
                          int64_t k, int metric, int64_t id_offset,
                          double *out_scores, int32_t *out_ids, void *stream);

/* Host-buffer form of the reference call scan_topk(data, queries, k, metric,
 * data_norms, query_norms) for int8 inputs: data[n, d] and queries[nq, d]
 * C-contiguous int8 in HOST memory; data_norms/query_norms host float32,
 * required for metric 2 and used as given (the reference takes them from
 * the caller too), ignored otherwise.  Output host arrays sized
 * nq*min(k,n).  Synchronous. */
int qa_scan_topk_i8_host(const int8_t *data, int64_t n, int64_t d,
                         const int8_t *queries, int64_t nq, int64_t k,
                         int metric, const float *data_norms,
                         const float *query_norms, double *out_scores,
                         int32_t *out_ids);

/* ---- float32 exhaustive search (_core.pyx:270-298 _scan_f32) ----
 * Replaces scan_topk() with float32 data/queries (_core.pyx:333-365, the
 * dtype == float32 branch 361-362) and norms() on float32 rows
 * (_core.pyx:150-153).  Scores are the reference's float64 values bit for
 * bit: each pair is summed sequentially over j (product exact in float64,
 * explicit round-to-nearest adds); rows ascending by (score, id), ids + id_offset.
 * db_norm/q_norm (float32, the caller's) are read for metric 2 only.  Inputs
 * must be finite (the reference's heap order with NaN scores is
 * insertion-order dependent).  keff = min(k, n) <= 15360.  Asynchronous. */
int qa_scan_topk_f32(const float *db, int64_t n, int64_t d, int64_t ldd,
                     const float *db_norm, const float *q, int64_t nq, int64_t ldq,
                     const float *q_norm, int64_t k, int metric, int64_t id_offset,
                     double *out_scores, int32_t *out_ids, void *stream);
/* out[i] = (float)sqrt(sequential float64 sum of x[i, j]^2). */
int qa_norms_f32(const float *x, int64_t n, int64_t d, int64_t ldx, float *out, void *stream);

/* ---- on-disk vector files (dataset.py:160-275) ----
 * fvecs/ivecs (itemsize 4), i8vecs/bvecs (itemsize 1): records of an int32
 * little-endian d followed by d items.  qa_vecs_probe validates the framing
 * of the whole file exactly as the reference's _load_records/_walk_records
 * (dataset.py:160-209) and returns n, d (0, 0 for an empty file).
 * qa_vecs_read copies the payloads of records [row_lo, row_hi) -- e.g. one
 * rank's row shard -- to dst with row stride ld_bytes: into HBM (dst_on_device,
 * pinned double-buffered staging, header-stripping 2-D DMA on `stream`;
 * returns after the copies complete) or into host memory.  recenter_u8 maps
 * bvecs bytes v -> int8 v - 128 (load_bvecs, dataset.py:231-237).
 * qa_vecs_write writes n host rows (stride ld_bytes) with d-headers
 * (save_fvecs/save_ivecs/save_i8vecs, dataset.py:249-275). */
int qa_vecs_probe(const char *path, int itemsize, int64_t *n, int64_t *d);
int qa_vecs_read(const char *path, int itemsize, int64_t d, int64_t row_lo, int64_t row_hi,
                 void *dst, int64_t ld_bytes, int dst_on_device, int recenter_u8, void *stream);
int qa_vecs_write(const char *path, int itemsize, const void *src, int64_t n, int64_t d,
                  int64_t ld_bytes);

/* ---- index layout ----
 * perm = the stored row order of an index (qa_layout.cu): rows stably sorted
 * by squared norm, cut into 4096-row norm bands stored interleaved (tight
 * per-unit filter bounds, every prefix spread over the bands); with
 * `stratify` the first 32768 stored rows are a stratified sample of all bands
 * (the search's threshold estimate treats that prefix as a sample; used for
 * L2).  qa_permute_rows_i8 applies it to codes + norms (norm/norm_out may be
 * NULL). */
int qa_order_rows_by_norm(const int32_t *sqnorm, int64_t n, int stratify, int32_t *perm,
                          void *stream);
int qa_permute_rows_i8(const int8_t *codes, const int32_t *sqnorm, const float *norm,
                       int64_t n, int64_t ldc, const int32_t *perm, int8_t *codes_out,
                       int32_t *sqnorm_out, float *norm_out, void *stream);

/* ---- multi-shard merge (row-sharded search, §8e) ----
 * in_scores/in_ids: [G, nq, kin] per-shard sorted lists with GLOBAL ids;
 * writes the first k of the (score, id)-merged list per query. */
int qa_merge_topk(const double *in_scores, const int32_t *in_ids, int64_t G,
                  int64_t nq, int64_t kin, int64_t k, double *out_scores,
                  int32_t *out_ids, void *stream);

/* ---- diagnostics (tests) ----
 * Full int32 dot matrix out[nq, n] (row stride n) through one filter pass
 * with the threshold disabled: impl 0 = the production tensor-core pass
 * (tcgen05 kind::i8), impl 1 = the CUDA-core dp4a pass.  Used to validate
 * the MMA path in isolation. */
int qa_debug_dots_i8(const int8_t *db, int64_t n, const int8_t *q, int64_t nq,
                     int64_t d, int impl, int32_t *out, void *stream);

/* Per-call statistics of the last qa_scan_topk_i8 on this thread: filter
 * rounds, kernel launches, overflow retries, the algorithmic int8 ops of the
 * filter passes (2 * queries * rows * d, unpadded d), and -- when profiling
 * is enabled -- CUDA-event durations measured on the launch stream around
 * every filter / select launch. */
typedef struct {
    int64_t rounds;
    int64_t candidates;
    int64_t launches;
    int64_t retries;
    int64_t filter_launches;
    double filter_ops;
    double filter_ms;
    double select_ms;
} qa_scan_stats;
int qa_last_scan_stats(qa_scan_stats *out);
/* Sums of qa_scan_stats over every scan since the last reset (a step that
 * issues several query batches reports them together). */
int qa_scan_totals(qa_scan_stats *out);
int qa_reset_scan_totals(void);
/* Enable (1) / disable (0) event timing of filter and select launches. */
int qa_set_profiling(int on);

#ifdef __cplusplus
}
#endif

#endif /* QA_B200_H */
