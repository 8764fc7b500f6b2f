// qa_internal.h -- launcher declarations shared between the translation units.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "qa_common.cuh"

namespace qa {

int num_sms();

cudaError_t launch_encode(const float *x, int64_t n, int64_t d, int64_t ldx, const float *k,
                          const float *sb, const float *se, int bits, int8_t *codes, int64_t ldc,
                          int32_t *sqnorm, float *norm, cudaStream_t st);
cudaError_t launch_norms(const int8_t *codes, int64_t n, int64_t d, int64_t ldc, int32_t *sqnorm,
                         float *norm, cudaStream_t st);
cudaError_t launch_minmax(const float *x, int64_t n, int64_t d, int64_t ldx, float *out_min,
                          float *out_max, float *scratch, int64_t scratch_floats,
                          cudaStream_t st);

// Everything one filter pass needs.  Rows [r_lo, r_hi) of the database are
// scored against queries [0, nq) of the current query chunk; every
// (query, row) whose dot passes the query's threshold is appended to that
// query's candidate list (capacity cap; count keeps counting past cap so
// overflow is detectable).
struct FilterArgs {
    const int8_t *db;
    int64_t ldd;
    const int8_t *q;
    int64_t ldq;
    int64_t kdim;  // padded reduction length (== ldd == ldq, multiple of 32)
    int64_t nq;
    int64_t r_lo, r_hi;
    const int32_t *db_sqnorm;
    const float *db_norm;
    // per 32-row group norm range (launch_group_ranges): L2 grp_lo = min
    // sqnorm; angular grp_lo/grp_hi = float bits of min/max norm
    const int32_t *grp_lo;
    const int32_t *grp_hi;
    const int32_t *thr;
    Cand *cand;
    int32_t *ccount;
    int64_t cap;
    int metric;
    // 0 = filter (threshold test + append), 1 = dense (every row is a
    // candidate: cand[q, row - r_lo]; the round-0 pass), 2 = diagnostics
    // (every dot to dots_out[q, row]), 3 = masked dense, 4 = sampled
    // estimate (per-bucket best goodness to est_keys; no candidates).
    int mode;
    int32_t *dots_out;
    int64_t ld_dots;
    // expected candidates per query in this pass (mode 0; sizes the work
    // units so their survivors fit the on-chip staging)
    double exp_cands;
    // zeroed work-unit counter of this launch (dynamic scheduling)
    unsigned *sched = nullptr;
    // mode 4 (sampled threshold estimate): per query, the best "goodness" of
    // every row bucket, est_keys[q * est_ld + bucket] (see
    // filter_est_buckets); goodness is an order-preserving int32, larger is
    // better: IP dot, L2 2*dot - xx, angular the float dot/xn mapped to int
    int32_t *est_keys = nullptr;
    int64_t est_ld = 0;
    // mode 4: the pass reads every sample_stride-th 128-row tile of
    // [r_lo, r_hi), max_tpu sample tiles per work unit (filter_est_layout)
    int64_t sample_stride = 0;
    // cap on the tiles per work unit (0 = the launcher's choice)
    int max_tpu = 0;
    // mode 0: work units from a table (launch_unit_table) instead of fixed
    // runs of tiles: unit_table[2*i] = first tile (relative to r_lo),
    // [2*i+1] = tile count (<= 32); *unit_count units
    const int32_t *unit_table = nullptr;
    const int32_t *unit_count = nullptr;
};

// The work-unit table of a mode-0 pass over tiles [tile_lo, tile_lo + n_tiles)
// (global 128-row tile indices): aligned runs of `tpu` tiles, except runs
// whose norm range is wide (the index's sparse norm tails), which are split
// into short units (8 tiles) with tighter bounds; the split units come first so
// their extra cost starts early.  table needs 2 * n_tiles ints, scratch
// 2 * ceil(n_tiles / tpu) doubles; *ticket must be 0 (the kernel leaves it 0).
cudaError_t launch_unit_table(int metric, const int32_t *grp_lo, const int32_t *grp_hi,
                              int64_t tile_lo, int64_t n_tiles, int tpu, int32_t *table,
                              int32_t *count, unsigned *ticket, double *scratch, cudaStream_t st);
// tiles per unit the launcher picks for a mode-0 pass
int filter_tiles_per_unit(int64_t rows, int64_t nq, int64_t kdim);

// Work-unit size (sample tiles) and buckets per query of a mode-4 pass over
// `tiles` sample tiles: ~2 units per CTA, halved until there are at least
// `min_buckets` buckets per query (*tpu = 0: no tensor-core pass for the shape).
void filter_est_layout(int64_t tiles, int64_t nq, int64_t kdim, int64_t min_buckets, int *tpu,
                       int64_t *buckets);
// thr[q] / est[q] from the est_j-th best bucket of a mode-4 pass (qa_select.cu);
// est[q] = ~0 when fewer than j buckets hold a row
cudaError_t launch_est_select(const int32_t *keys, int64_t ld, int64_t nb, int64_t nq, int64_t j,
                              int metric, const int32_t *q_sqnorm, const float *q_norm,
                              int32_t *thr, unsigned long long *est, cudaStream_t st);



// Tensor-core (tcgen05 kind::i8) filter pass.  Returns cudaErrorNotSupported
// when the shape is outside what the kernel handles.
cudaError_t launch_filter_tc(const FilterArgs &a, cudaStream_t st);
// Plain CUDA-core (dp4a) filter pass, the bring-up path.
cudaError_t launch_filter_simt(const FilterArgs &a, cudaStream_t st);

struct SelectArgs {
    Entry *state;        // [nq, k] sorted (score,row) prefix of length state_cnt[q]
    int32_t *state_cnt;  // [nq]
    const Cand *cand;    // [nq, cap]
    const int32_t *ccount;
    int64_t cap;
    int64_t nq;
    int64_t k;
    int metric;
    const int32_t *db_sqnorm;
    const float *db_norm;
    const int32_t *q_sqnorm;
    const float *q_norm;
    const int32_t *row_ids;  // stored row -> reported id (NULL: identity)
    int32_t *thr;        // out: next-round threshold
    int32_t *overflow;   // [nq] sticky per-query flag: candidate list overflowed
    int32_t *any_overflow;
    unsigned long long *cand_count;  // statistics: valid candidates seen (may be NULL)
    // fused threshold estimate (0 = none; the register select only): after
    // the merge, thr := threshold of the est_j-th kept entry and est[q] := its
    // order key (with est_combine, the tighter of that and the previous one)
    int64_t est_j = 0;
    unsigned long long *est = nullptr;
    int est_combine = 0;
    // fused fill (register select only): ccount_reset[q] := next_fill once the
    // round's candidates are consumed (-1 = leave)
    int32_t next_fill = -1;
    int32_t *ccount_reset = nullptr;
};

cudaError_t launch_select(const SelectArgs &a, cudaStream_t st);

// Device-side exact recompute of the flagged queries (flag[q] != 0) of a
// search: a full scan per flagged query, results into out_* (qa_select.cu).
struct RepairArgs {
    const int8_t *db;
    int64_t n, ld;
    const int32_t *db_sqnorm;
    const float *db_norm;
    const int32_t *row_ids;
    const int8_t *q;
    int64_t nq;
    const int32_t *q_sqnorm;
    const float *q_norm;
    int64_t keff;
    int metric;
    int64_t id_offset;
    const int32_t *flag;
    double *out_scores;
    int32_t *out_ids;
    // workspace (repair_scratch_bytes): compacted flag list, counters, the
    // per-part partial lists
    void *scratch;
};
size_t repair_scratch_bytes(int64_t n, int64_t nq, int64_t keff);
cudaError_t launch_repair(const RepairArgs &r, cudaStream_t st);
cudaError_t launch_init_state(int32_t *state_cnt, int32_t *thr, int64_t nq, int metric,
                              cudaStream_t st);
cudaError_t launch_fill(int32_t *p, int64_t n, int32_t v, cudaStream_t st);
// thr[q] := threshold of the j-th kept entry; est[q] := its order key, or with
// `combine` the tighter of that and the previous est[q] (two-level estimate)
cudaError_t launch_estimate(const Entry *state, const int32_t *state_cnt, int32_t *thr,
                            unsigned long long *est, int64_t nq, int64_t k, int64_t j, int metric,
                            const int32_t *q_sqnorm, const float *q_norm, bool combine,
                            cudaStream_t st);
// redo[q] := 1 where the k-th kept entry is worse than est[q]
cudaError_t launch_check_estimate(const Entry *state, const int32_t *state_cnt,
                                  const unsigned long long *est, int64_t nq, int64_t k,
                                  int32_t *redo, int32_t *any_redo, cudaStream_t st);
// est != NULL: also the estimate check of launch_check_estimate (fused)
cudaError_t launch_finalize(const Entry *state, int64_t nq, int64_t k, int64_t keff, int metric,
                            int64_t id_offset, double *out_scores, int32_t *out_ids,
                            cudaStream_t st, const int32_t *state_cnt = nullptr,
                            const unsigned long long *est = nullptr, int32_t *redo = nullptr,
                            int32_t *any_redo = nullptr);
// state_cnt := 0, thr := pass-all for nq queries; also zeroes ovf[nq] and
// flags[16] when given (fused memsets)
// (and zeroes sched[nsched], the filter passes' work-unit counters)
cudaError_t launch_init_state_full(int32_t *state_cnt, int32_t *thr, int64_t nq, int metric,
                                   int32_t *ovf, int32_t *flags, int32_t *ccount, int32_t fill0,
                                   cudaStream_t st, unsigned *sched = nullptr, int nsched = 0);
// Norm range of every 32-row group, padded to `groups` entries (groups past
// n never pass a filter bound).
cudaError_t launch_group_ranges(int metric, const int32_t *sqnorm, const float *norm, int64_t n,
                                int32_t *lo, int32_t *hi, int64_t groups, cudaStream_t st);
// stable ascending order of rows by int32 key (CUB radix sort); perm[i] = row
cudaError_t launch_order_by_key(const int32_t *key, int64_t n, bool stratify, int32_t *perm,
                                void *scratch,
                                size_t scratch_bytes, size_t *needed, cudaStream_t st);
cudaError_t launch_permute_rows(const int8_t *src, const int32_t *sq_in, const float *n_in,
                                int64_t n, int64_t ld, const int32_t *perm, int8_t *dst,
                                int32_t *sq_out, float *n_out, cudaStream_t st);
// scratch bytes launch_merge needs (0: the shared-memory merge serves k)
size_t merge_scratch_bytes(int64_t G, int64_t nq, int64_t kin, int64_t k);
cudaError_t launch_merge(const double *in_scores, const int32_t *in_ids, int64_t G, int64_t nq,
                         int64_t kin, int64_t k, double *out_scores, int32_t *out_ids,
                         cudaStream_t st, void *scratch = nullptr);

// float32 exhaustive search (qa_exact_f32.cu), bit-exact with _scan_f32.
cudaError_t launch_f32_scores(const float *db, int64_t ldd, const float *q, int64_t ldq, int64_t d,
                              int64_t nq, int64_t r_lo, int64_t rows, int metric,
                              const float *db_norm, const float *q_norm, double *out, int64_t ldo,
                              cudaStream_t st);
cudaError_t launch_f32_select(const double *scores, int64_t lds, int64_t rows, int64_t id0,
                              double *st_s, int32_t *st_i, int32_t *st_n, int64_t nq, int64_t k,
                              cudaStream_t st);
cudaError_t launch_f32_finalize(const double *st_s, const int32_t *st_i, int64_t nq, int64_t k,
                                int64_t id_offset, double *out_s, int32_t *out_i, cudaStream_t st);
// scores of listed (query, row id) pairs (qa_gather.cu)
cudaError_t launch_gather_scores(const int8_t *db, int64_t n, int64_t ldd,
                                 const int32_t *db_sqnorm, const float *db_norm,
                                 const int32_t *row_of_id, const int8_t *q, int64_t nq,
                                 int64_t ldq, const int32_t *q_sqnorm, const float *q_norm,
                                 const int32_t *cand, int64_t m, int64_t ldcand, int metric,
                                 double *out, cudaStream_t st);

cudaError_t launch_norms_f32(const float *x, int64_t n, int64_t d, int64_t ldx, float *out,
                             cudaStream_t st);
size_t f32_select_smem(int64_t k);
// any k: all n scores of m queries sorted per query (CUB segmented radix sort);
// scratch of f32_fullsort_bytes(m, n) bytes
size_t f32_fullsort_bytes(int64_t m, int64_t n);
cudaError_t launch_f32_fullsort(const float *db, int64_t ldd, const float *q, int64_t ldq,
                                int64_t d, int64_t m, int64_t n, int metric, const float *db_norm,
                                const float *q_norm, int64_t keff, int64_t id_offset,
                                double *out_s, int32_t *out_i, void *scratch, size_t bytes,
                                cudaStream_t st);

// estimate_stats (qa_stats.cu): x on the device, every output on the HOST;
// synchronous on st.  qlo/qhi: the trimming quantiles per dimension.
cudaError_t launch_estimate_stats(const float *x, int64_t n, int64_t d, int64_t ldx, double *mu,
                                  double *sigma, double *mn, double *mx, double *tam,
                                  double *qlo, double *qhi, double *pooled_mu,
                                  double *pooled_sigma, cudaStream_t st);

// Largest list the select kernel sorts in shared memory at once.
constexpr int64_t kSortMax = 8192;
// Largest k served by the int8 select (k + one candidate chunk must fit
// kSortMax); larger k (up to kMaxKF32) take the float64-exact scan on the
// codes, which sorts state + a 1024-candidate chunk of 12-byte entries in
// shared memory (16384 entries = 192 KiB).
constexpr int64_t kMaxK = 2048;
constexpr int64_t kMaxKF32 = 16384 - 1024;

}  // namespace qa
