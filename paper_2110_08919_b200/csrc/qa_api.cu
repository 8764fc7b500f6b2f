// qa_api.cu -- the C-ABI (include/qa_b200.h) and the search orchestration.
//
// Search algorithm for one query chunk (all of it stays on the device; the
// only host synchronisation is the final overflow check):
//
//   round 0   rows [0, r0)          dense pass: every row is a candidate
//   round i   rows [r_{i-1}, r_i)   filter pass with each query's current
//                                   k-th score as threshold, r_i = ratio*r_{i-1}
//   after every round: select (exact float64 scores, (score, id) sort, keep
//   k, next threshold); at the end: finalize (scores + ids to the output).
//
// Any k rows' k-th best score bounds the final k-th best score, so a filter
// pass never discards a row of the final top-k; rows whose threshold test
// passes are re-scored exactly, so the output equals the reference's full
// lexicographic sort truncated to keff (_core.pyx:301-330, 349).  Candidate
// lists are bounded (cap per query); a query that overflows its list in any
// round is recomputed with a larger cap.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/qa_b200.h"
#include "qa_common.cuh"
#include "qa_internal.h"

namespace qa {

namespace {

thread_local std::string g_err;
thread_local qa_scan_stats g_stats;
thread_local qa_scan_stats g_totals;
bool g_profiling = false;

// Event pairs recorded around filter / select launches when profiling.
struct EventTimer {
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<int, int>> spans;  // (kind, index of start event)
    size_t used = 0;
    cudaEvent_t next() {
        if (used == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        return pool[used++];
    }
    void reset() {
        used = 0;
        spans.clear();
    }
    void begin(int kind, cudaStream_t st) {
        if (!g_profiling) return;
        spans.emplace_back(kind, (int)used);
        cudaEventRecord(next(), st);
    }
    void end(cudaStream_t st) {
        if (!g_profiling) return;
        cudaEventRecord(next(), st);
    }
    // sums the recorded spans into s (waits for the last event) and resets
    void accumulate(qa_scan_stats &s) {
        if (used > 0) cudaEventSynchronize(pool[used - 1]);
        static const bool print = getenv("QA_B200_TIMES") != nullptr;  // diagnostics
        for (auto &sp : spans) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, pool[sp.second], pool[sp.second + 1]);
            if (print) std::fprintf(stderr, "qa_time %s %.1f us\n", sp.first == 0 ? "filter" : "select", ms * 1e3f);
            if (sp.first == 0)
                s.filter_ms += ms;
            else
                s.select_ms += ms;
        }
        reset();
    }
};
thread_local EventTimer g_timer;

int set_err(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

}  // namespace

int set_error_message(int code, const char *msg) {
    g_err = msg;
    return code;
}

namespace {

int cuda_err(cudaError_t e, const char *what) {
    if (e == cudaErrorNotSupported)
        return set_err(QA_EUNSUPPORTED, "%s: shape not supported by this build", what);
    if (e == cudaErrorMemoryAllocation) return set_err(QA_ENOMEM, "%s: out of device memory", what);
    return set_err(QA_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define QA_TRY(expr, what)                         \
    do {                                           \
        cudaError_t _e = (expr);                   \
        if (_e != cudaSuccess) return cuda_err(_e, what); \
    } while (0)

// Grow-only device buffers, one set per device, guarded by a mutex.
struct Buf {
    void *ptr = nullptr;
    size_t bytes = 0;
    cudaError_t reserve(size_t want) {
        if (want <= bytes) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        size_t b = std::max(want, (size_t)256);
        cudaError_t e = cudaMalloc(&ptr, b);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
};

struct Workspace {
    std::mutex mu;
    Buf state, state_cnt, thr, cand, ccount, ovf, flags, scratch, grp, est;
    Buf ekeys;                       // bucket keys of the sampled estimate pass
    Buf units;                       // work-unit table of the final pass (+ count)
    Buf sched;                       // [kSchedSlots] work-unit counters of the filter passes
    Buf f32_scores, f32_ss, f32_si, f32_sn;  // float32 exact search (qa_exact_f32.cu)
    Buf f32_full;                            // any-k full sort scratch
    Buf f32_x, f32_q, f32_xn;                // codes as float32 (large k / wide rows)
    Buf r_idx, r_q, r_qsq, r_qn, r_s, r_ids;  // overflow retry
    Buf merge;                                // large-k shard merge
    Buf repair;                               // device-side recompute (async scans)
};

constexpr int kMaxDevices = 64;
constexpr int kSchedSlots = 64;  // filter passes per query chunk with a preset counter
Workspace g_ws[kMaxDevices];

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

bool use_simt_filter(int64_t kdim) {
    static int forced = -1;
    if (forced < 0) {
        const char *v = getenv("QA_B200_FILTER");
        forced = (v && strcmp(v, "simt") == 0) ? 1 : 0;
    }
    return forced == 1 || kdim > 1024;
}

bool trace_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *v = getenv("QA_B200_TRACE");
        on = (v && *v && strcmp(v, "0") != 0) ? 1 : 0;
    }
    return on == 1;
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

struct ScanPlan {
    int64_t r0, ratio, cap, qchunk;
    // Threshold estimate (0 = off): the sample is every est_stride-th 128-row
    // tile of the index (est_tiles tiles, est_rows rows); the est_j-th best
    // sample score bounds ONE pass over every row.
    int64_t est_rows, est_j, est_stride, est_tiles;
};

// Smallest j with P(Poisson(lambda) >= j) <= tail.
int64_t poisson_quantile(double lambda, double tail) {
    double pmf = std::exp(-lambda), cdf = pmf;
    int64_t j = 0;
    while (1.0 - cdf > tail && j < 100000) {
        ++j;
        pmf *= lambda / (double)j;
        cdf += pmf;
    }
    return j + 1;
}

ScanPlan plan_scan(int64_t n, int64_t nq, int64_t keff, int64_t cap_min, bool allow_estimate) {
    ScanPlan p;
    // a power of two >= 256: with ratio 2 every round boundary >= 4096 is a
    // multiple of the index's 4096-row norm blocks (qa_layout.cu).  1024
    // measured best for cfg1 (a dense round is cheaper than two doubling
    // rounds of a few hundred rows each).
    int64_t r0 = 1024;
    if (const char *v = getenv("QA_B200_R0")) r0 = std::max<int64_t>(128, atoll(v));
    while (r0 < keff) r0 *= 2;
    p.r0 = std::min(n, r0);
    // Row growth per round: every round adds ~k*(ratio-1) survivors per query;
    // small ratios cost more rounds (launches), large ones more survivors.
    // Small batches: few, wide rounds (each round costs a select launch;
    // the filter is HBM-bound there, not survivor-bound).
    p.ratio = nq >= 256 ? 2 : 32;
    if (const char *v = getenv("QA_B200_RATIO")) p.ratio = std::max(2, atoi(v));
    p.cap = std::max<int64_t>({2048, p.r0, 2 * keff * p.ratio, cap_min});
    // Threshold estimate.  In a sample of P rows (every stride-th tile: the
    // index interleaves narrow norm blocks, so the sample spans every band)
    // about k*P/n rows beat the final k-th score; taking the j-th sample
    // score with j a high quantile of that count makes ">= k rows pass"
    // near-certain, and the check after the pass proves it per query (the
    // rare misses are recomputed without the estimate).  The pass then admits
    // ~j*n/P candidates per query instead of ~k per doubling round.
    p.est_rows = 0;
    p.est_j = 0;
    p.est_stride = 0;
    p.est_tiles = 0;
    if (allow_estimate) {
        // sample rows: a larger sample costs a longer sampled pass and buys a
        // tighter estimate (fewer candidates in the final pass and the
        // select).  Batches up to ~2k queries gain from 65536 (cfg2 +1.4 %,
        // cfg4 2-5 %); a 10k-query chunk loses (cfg1 -15 %: its bucket
        // arrays and their select grow with the query count)
        int64_t P = nq <= 2048 ? 65536 : 32768;
        if (const char *v = getenv("QA_B200_EST_ROWS")) P = std::max<int64_t>(128, atoll(v));
        while (P < 64 * keff) P *= 2;
        // small indexes (e.g. one GPU's row shard): a smaller sample rather
        // than no estimate at all (which costs a doubling round per 2x rows)
        if (!getenv("QA_B200_EST_ROWS"))
            while (4 * P > n && P / 2 >= std::max<int64_t>(64 * keff, 4096)) P /= 2;
        if (4 * P <= n) {
            const int64_t T = (n + 127) / 128;
            const int64_t stride = std::max<int64_t>(1, T / (P / 128));
            const int64_t S = (T + stride - 1) / stride;
            // rows sampled (the last index tile may be partial and sampled)
            int64_t rows = S * 128;
            if ((S - 1) * stride == T - 1) rows -= T * 128 - n;
            const double lambda = (double)keff * (double)rows / (double)n;
            double tail = 1e-4;
            if (const char *v = getenv("QA_B200_EST_TAIL")) tail = atof(v);
            int64_t j = std::max<int64_t>(8, poisson_quantile(lambda, tail));
            // diagnostics/tests: force j (small j makes the estimate fail often)
            if (const char *v = getenv("QA_B200_EST_J")) j = std::max<int64_t>(1, atoll(v));
            if (j < keff) {
                p.est_rows = rows;
                p.est_j = j;
                p.est_stride = stride;
                p.est_tiles = S;
                p.cap = std::max<int64_t>(p.cap, 4 * j * (n / rows));
            }
        }
    }
    const int64_t per_q = p.cap * (int64_t)sizeof(Cand) + keff * (int64_t)sizeof(Entry) + 64;
    const int64_t budget = (int64_t)1 << 30;
    p.qchunk = std::max<int64_t>(1, std::min<int64_t>(nq, budget / per_q));
    p.qchunk = std::min<int64_t>(p.qchunk, 65535 * 16);
    return p;
}

__global__ void gather_rows_kernel(const int8_t *__restrict__ src, int64_t ld,
                                   const int32_t *__restrict__ idx, int64_t m,
                                   int8_t *__restrict__ dst) {
    int64_t r = blockIdx.x;
    if (r >= m) return;
    const int8_t *s = src + (int64_t)idx[r] * ld;
    for (int64_t j = threadIdx.x; j < ld; j += blockDim.x) dst[r * ld + j] = s[j];
}

template <typename T>
__global__ void gather_vals_kernel(const T *__restrict__ src, const int32_t *__restrict__ idx,
                                   int64_t m, T *__restrict__ dst) {
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < m) dst[r] = src[idx[r]];
}

__global__ void scatter_results_kernel(const double *__restrict__ s, const int32_t *__restrict__ i,
                                       const int32_t *__restrict__ idx, int64_t m, int64_t keff,
                                       double *__restrict__ out_s, int32_t *__restrict__ out_i) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m * keff) return;
    int64_t r = t / keff, j = t - r * keff;
    out_s[(int64_t)idx[r] * keff + j] = s[t];
    out_i[(int64_t)idx[r] * keff + j] = i[t];
}

// flag[0] := 1 when any angular norm is <= 0 (or NaN): the reference raises
// ZeroNorm before scanning (exact.py:67-69); here the check rides on the
// scan's one end-of-search readback
__global__ void zero_norm_kernel(const float *__restrict__ a, int64_t na,
                                 const float *__restrict__ b, int64_t nb, int32_t *flag) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const float v = i < na ? a[i] : (i < na + nb ? b[i - na] : 1.0f);
    if (!(v > 0.0f)) *flag = 1;
}

// One query chunk with the sampled estimate: the bucket-best pass over the
// sample tiles, the per-query est_j-th best bucket as the bound, then ONE
// filter pass over every row and one select.  The check in finalize flags the
// queries whose k-th score the bound did not cover.
cudaError_t sampled_chunk(const ScanPlan &pl, int64_t n, int64_t d_alg, int64_t ld,
                          const int8_t *db, const int32_t *db_sqnorm, const float *db_norm,
                          const int32_t *row_ids, const int8_t *q, int64_t m,
                          const int32_t *q_sqnorm, const float *q_norm, int64_t keff, int metric,
                          const int32_t *grp_lo, const int32_t *grp_hi, int32_t *thr, Cand *cand,
                          int32_t *ccount, Entry *state, int32_t *state_cnt,
                          unsigned long long *est, int32_t *ekeys, int32_t *units,
                          unsigned *sched, int32_t *ovf, int32_t *flags, cudaStream_t st) {
    FilterArgs fa{};
    fa.db = db;
    fa.ldd = ld;
    fa.q = q;
    fa.ldq = ld;
    fa.kdim = ld;
    fa.nq = m;
    fa.db_sqnorm = db_sqnorm;
    fa.db_norm = db_norm;
    fa.grp_lo = grp_lo;
    fa.grp_hi = grp_hi;
    fa.thr = thr;
    fa.cand = cand;
    fa.ccount = ccount;
    fa.cap = pl.cap;
    fa.metric = metric;
    // the bucket-best pass over the sample tiles
    int tpu = 0;
    int64_t nb = 0;
    filter_est_layout(pl.est_tiles, m, ld, 8 * pl.est_j, &tpu, &nb);
    fa.mode = 4;
    fa.r_lo = 0;
    fa.r_hi = n;
    fa.sample_stride = pl.est_stride;
    fa.max_tpu = tpu;
    fa.est_keys = ekeys;
    fa.est_ld = nb;
    fa.sched = sched + 0;
    g_timer.begin(0, st);
    cudaError_t e = launch_filter_tc(fa, st);
    g_timer.end(st);
    if (e != cudaSuccess) return e;
    g_stats.filter_launches += 1;
    g_stats.filter_ops += 2.0 * (double)m * (double)pl.est_rows * (double)d_alg;
    e = launch_est_select(ekeys, nb, nb, m, pl.est_j, metric, q_sqnorm, q_norm, thr, est, st);
    if (e != cudaSuccess) return e;
    // the pass over every row, bounded by the estimate
    fa.mode = 0;
    fa.sample_stride = 0;
    fa.max_tpu = 0;
    if (const char *v = getenv("QA_B200_FINAL_TPU")) fa.max_tpu = atoi(v);  // diagnostics
    // L2: the norm tails of the index are sparse, so their runs of tiles span
    // wide norm ranges (cfg2: the lowest 4096-row block spans 180x the median
    // block), their bound admits nearly every element to the exact test, and
    // one such unit outlasted the rest of the pass (538 -> 291 us per cfg2
    // batch as single-tile units; 8-tile units since the epilogue parks its
    // candidates: qa_layout.cu).  Angular tests survivors in the select,
    // not the epilogue: there the extra units cost more (cfg1 +16 %); so do
    // they for a handful of queries, whose exact tests are few (cfg4 batch
    // 1 / 8: +25 us, batch 64: -15 us).
    static const bool tables = [] {
        const char *v = getenv("QA_B200_UNIT_TABLE");  // diagnostics: 0 = off
        return !(v && strcmp(v, "0") == 0);
    }();
    if (tables && metric == kL2 && m > 16 && fa.max_tpu == 0) {
        const int tpu = filter_tiles_per_unit(n, m, ld);
        if (tpu > 1) {
            const int64_t nt = (n + 127) / 128;
            e = launch_unit_table(metric, grp_lo, grp_hi, 0, nt, tpu, units, units + 2 * nt,
                                  sched + kSchedSlots - 1, (double *)(units + 2 * nt + 2), st);
            if (e != cudaSuccess) return e;
            fa.unit_table = units;
            fa.unit_count = units + 2 * nt;
            g_stats.launches += 1;
        }
    }
    fa.est_keys = nullptr;
    fa.est_ld = 0;
    fa.sched = sched + 1;
    fa.exp_cands = (double)pl.est_j * (double)n / (double)pl.est_rows;
    g_timer.begin(0, st);
    e = launch_filter_tc(fa, st);
    g_timer.end(st);
    if (e != cudaSuccess) return e;
    g_stats.filter_launches += 1;
    g_stats.filter_ops += 2.0 * (double)m * (double)n * (double)d_alg;
    SelectArgs sa;
    sa.state = state;
    sa.state_cnt = state_cnt;
    sa.cand = cand;
    sa.ccount = ccount;
    sa.cap = pl.cap;
    sa.nq = m;
    sa.k = keff;
    sa.metric = metric;
    sa.db_sqnorm = db_sqnorm;
    sa.db_norm = db_norm;
    sa.q_sqnorm = q_sqnorm;
    sa.q_norm = q_norm;
    sa.row_ids = row_ids;
    sa.thr = thr;
    sa.overflow = ovf;
    sa.any_overflow = flags;
    sa.cand_count = reinterpret_cast<unsigned long long *>(flags + 4);
    sa.next_fill = -1;
    sa.ccount_reset = ccount;
    g_timer.begin(1, st);
    e = launch_select(sa, st);
    g_timer.end(st);
    if (e != cudaSuccess) return e;
    g_stats.launches += 5;  // estimate pass, est_select, filter, select
    g_stats.rounds += 2;
    return cudaSuccess;
}

// One complete search with a given minimum candidate capacity.  Returns
// QA_OK; *overflowed receives the list of queries whose lists overflowed
// (their output rows are invalid and must be recomputed).
int scan_impl(Workspace &ws, const int8_t *db, int64_t n, int64_t d_alg, int64_t ld,
              const int32_t *db_sqnorm,
              const float *db_norm, const int32_t *row_ids, const int8_t *q, int64_t nq,
              const int32_t *q_sqnorm,
              const float *q_norm, int64_t keff, int metric, int64_t id_offset,
              double *out_scores, int32_t *out_ids, int64_t cap_min, bool allow_estimate,
              cudaStream_t st, std::vector<int32_t> *overflowed, bool async_ = false) {
    ScanPlan pl = plan_scan(n, nq, keff, cap_min, allow_estimate);
    const int64_t qc = pl.qchunk;
    const bool simt = use_simt_filter(ld);
    // the estimate needs the tensor-core pass (filter mode 4); the CUDA-core
    // bring-up path scans in doubling rounds
    if (simt) pl.est_rows = 0;
    if (pl.est_rows > 0) {
        int64_t nb_max = 0;
        for (int64_t mm : {std::min(qc, nq), nq - (nq - 1) / qc * qc}) {
            int tpu = 0;
            int64_t nb = 0;
            filter_est_layout(pl.est_tiles, mm, ld, 8 * pl.est_j, &tpu, &nb);
            nb_max = std::max(nb_max, nb);
        }
        QA_TRY(ws.ekeys.reserve((size_t)qc * nb_max * 4), "workspace");
        // table [2 * tiles] + count + pad, then the per-run ranges (2 doubles per run)
        QA_TRY(ws.units.reserve(((size_t)(n + 127) / 128 * 2 + 2) * 4 + (size_t)(n + 127) / 128 * 16),
               "workspace");
    }
    QA_TRY(ws.state.reserve((size_t)qc * keff * sizeof(Entry)), "workspace");
    QA_TRY(ws.state_cnt.reserve((size_t)qc * 4), "workspace");
    QA_TRY(ws.thr.reserve((size_t)qc * 4), "workspace");
    QA_TRY(ws.cand.reserve((size_t)qc * pl.cap * sizeof(Cand)), "workspace");
    QA_TRY(ws.ccount.reserve((size_t)qc * 4), "workspace");
    QA_TRY(ws.ovf.reserve((size_t)nq * 4), "workspace");
    QA_TRY(ws.flags.reserve(64), "workspace");
    QA_TRY(ws.est.reserve((size_t)qc * 8), "workspace");
    QA_TRY(ws.sched.reserve((size_t)kSchedSlots * 4), "workspace");
    unsigned *sched = (unsigned *)ws.sched.ptr;
    unsigned long long *est = (unsigned long long *)ws.est.ptr;
    Entry *state = (Entry *)ws.state.ptr;
    int32_t *state_cnt = (int32_t *)ws.state_cnt.ptr;
    int32_t *thr = (int32_t *)ws.thr.ptr;
    Cand *cand = (Cand *)ws.cand.ptr;
    int32_t *ccount = (int32_t *)ws.ccount.ptr;
    int32_t *ovf = (int32_t *)ws.ovf.ptr;
    int32_t *flags = (int32_t *)ws.flags.ptr;  // [0] any overflow, [4:6) candidate counter
    // norm range of every 128-row tile (per-unit filter bounds)
    const int64_t groups = (n + 127) / 128;
    QA_TRY(ws.grp.reserve((size_t)groups * 8), "workspace");
    int32_t *grp_lo = (int32_t *)ws.grp.ptr, *grp_hi = grp_lo + groups;
    QA_TRY(launch_group_ranges(metric, db_sqnorm, db_norm, n, grp_lo, grp_hi, groups, st),
           "group ranges");
    if (metric != kIP && groups) g_stats.launches += 1;

    unsigned long long trace_prev = 0;
    for (int64_t c0 = 0; c0 < nq; c0 += qc) {
        const int64_t m = std::min(qc, nq - c0);
        // state, thresholds, this chunk's overflow flags and (chunk 0) the
        // search flags in one launch
        QA_TRY(launch_init_state_full(state_cnt, thr, m, metric, ovf + c0, c0 == 0 ? flags : nullptr,
                                      ccount, pl.est_rows > 0 ? 0 : (int32_t)std::min(n, pl.r0), st,
                                      sched, kSchedSlots),
               "init");
        int pass = 0;  // filter passes of this chunk (work-unit counter slot)
        g_stats.launches += 1;
        if (c0 == 0 && metric == kAngular && !async_) {
            zero_norm_kernel<<<(unsigned)((n + nq + 255) / 256), 256, 0, st>>>(db_norm, n, q_norm,
                                                                               nq, flags + 2);
            QA_TRY(cudaGetLastError(), "norm check");
            g_stats.launches += 1;
        }
        if (pl.est_rows > 0) {
            QA_TRY(sampled_chunk(pl, n, d_alg, ld, db, db_sqnorm, db_norm, row_ids, q + c0 * ld, m,
                                 q_sqnorm ? q_sqnorm + c0 : nullptr, q_norm ? q_norm + c0 : nullptr,
                                 keff, metric, grp_lo, grp_hi, thr, cand, ccount, state, state_cnt,
                                 est, (int32_t *)ws.ekeys.ptr, (int32_t *)ws.units.ptr, sched,
                                 ovf + c0, flags, st),
                   "sampled scan");
            QA_TRY(launch_finalize(state, m, keff, keff, metric, id_offset, out_scores + c0 * keff,
                                   out_ids + c0 * keff, st, state_cnt, est, ovf + c0, flags),
                   "finalize");
            g_stats.launches += 1;
            continue;
        }
        int64_t r_lo = 0, r_hi = pl.r0;
        bool first = true;
        bool counts_preset = true;  // init set round 0's (dense) counts
        for (;;) {
            FilterArgs fa{};
            fa.db = db;
            fa.ldd = ld;
            fa.q = q + c0 * ld;
            fa.ldq = ld;
            fa.kdim = ld;
            fa.nq = m;
            fa.r_lo = r_lo;
            fa.r_hi = r_hi;
            fa.db_sqnorm = db_sqnorm;
            fa.db_norm = db_norm;
            fa.grp_lo = grp_lo;
            fa.grp_hi = grp_hi;
            fa.thr = thr;
            fa.cand = cand;
            fa.ccount = ccount;
            fa.cap = pl.cap;
            fa.metric = metric;
            // round 0: dense (every row); survivor-dense early rounds whose
            // rows fit the candidate list: masked dense (no atomics); then the
            // filter with staged survivors
            static const int64_t masked_max = [] {
                const char *v = getenv("QA_B200_MASKED_MAX");  // diagnostics knob
                return v ? (int64_t)atoll(v) : (int64_t)1024;
            }();
            const bool masked = !first && (r_hi - r_lo) <= std::min<int64_t>(pl.cap, masked_max);
            const int mode = first ? 1 : (masked ? 3 : 0);
            fa.mode = mode;
            fa.dots_out = nullptr;
            fa.ld_dots = 0;
            if (pass >= kSchedSlots) QA_TRY(cudaMemsetAsync(sched + pass % kSchedSlots, 0, 4, st), "sched");
            fa.sched = sched + pass % kSchedSlots;
            ++pass;
            // ~k new candidates per doubling of the rows seen
            fa.exp_cands = (double)keff * (double)(r_hi - r_lo) / (double)std::max<int64_t>(r_lo, 1);
            // candidate counts of this round: preset by init (round 0) or by
            // the previous round's register select; otherwise here
            if (!counts_preset) {
                QA_TRY(launch_fill(ccount, m, mode != 0 ? (int32_t)(r_hi - r_lo) : 0, st), "fill");
                g_stats.launches += 1;
            }
            cudaError_t e = cudaErrorNotSupported;
            g_timer.begin(0, st);
            if (!simt) e = launch_filter_tc(fa, st);
            if (e == cudaErrorNotSupported) e = launch_filter_simt(fa, st);
            g_timer.end(st);
            QA_TRY(e, "filter");
            g_stats.filter_launches += 1;
            g_stats.filter_ops += 2.0 * (double)m * (double)(r_hi - r_lo) * (double)d_alg;
            SelectArgs sa;
            sa.state = state;
            sa.state_cnt = state_cnt;
            sa.cand = cand;
            sa.ccount = ccount;
            sa.cap = pl.cap;
            sa.nq = m;
            sa.k = keff;
            sa.metric = metric;
            sa.db_sqnorm = db_sqnorm;
            sa.db_norm = db_norm;
            sa.q_sqnorm = q_sqnorm ? q_sqnorm + c0 : nullptr;
            sa.q_norm = q_norm ? q_norm + c0 : nullptr;
            sa.row_ids = row_ids;
            sa.thr = thr;
            sa.overflow = ovf + c0;
            sa.any_overflow = flags;
            sa.cand_count = reinterpret_cast<unsigned long long *>(flags + 4);
            // the next round's rows (and so its candidate-count preset, which
            // the register select writes when it is done with this round's)
            const int64_t next_hi = std::min(n, round_up(r_hi * pl.ratio, 128));
            const bool next_masked = (next_hi - r_hi) <= std::min<int64_t>(pl.cap, masked_max);
            const int32_t next_fill = next_masked ? (int32_t)(next_hi - r_hi) : 0;
            const bool fill_fused = keff <= 128 && r_hi < n;
            sa.next_fill = fill_fused ? next_fill : -1;
            sa.ccount_reset = ccount;
            g_timer.begin(1, st);
            QA_TRY(launch_select(sa, st), "select");
            g_timer.end(st);
            counts_preset = fill_fused;
            g_stats.launches += 2;  // filter + select
            g_stats.rounds += 1;
            if (trace_enabled()) {  // diagnostics: per-round survivors (synchronises)
                unsigned long long cnt = 0;
                QA_TRY(cudaMemcpyAsync(&cnt, flags + 4, 8, cudaMemcpyDeviceToHost, st), "trace");
                QA_TRY(cudaStreamSynchronize(st), "trace");
                std::fprintf(stderr, "qa_trace chunk=%lld rows=[%lld,%lld) mode=%d cands=%llu\n",
                             (long long)c0, (long long)r_lo, (long long)r_hi, mode,
                             cnt - trace_prev);
                trace_prev = cnt;
            }
            if (r_hi >= n) break;
            r_lo = r_hi;
            first = false;
            r_hi = next_hi;
        }
        QA_TRY(launch_finalize(state, m, keff, keff, metric, id_offset, out_scores + c0 * keff,
                               out_ids + c0 * keff, st, state_cnt, nullptr, ovf + c0, flags),
               "finalize");
        g_stats.launches += 1;
    }
    overflowed->clear();
    if (async_) {
        // no host round trip: the flagged queries (overflow, failed estimate
        // check) are recomputed on the device, in stream order
        QA_TRY(ws.repair.reserve(repair_scratch_bytes(n, nq, keff)), "workspace");
        RepairArgs rp{db, n, ld, db_sqnorm, db_norm, row_ids, q, nq, q_sqnorm, q_norm, keff,
                      metric, id_offset, ovf, out_scores, out_ids, ws.repair.ptr};
        QA_TRY(launch_repair(rp, st), "repair");
        g_stats.launches += 2;
        return QA_OK;
    }
    int32_t hflags[6] = {0, 0, 0, 0, 0, 0};
    QA_TRY(cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, st),
           "overflow check");
    QA_TRY(cudaStreamSynchronize(st), "sync");
    if (hflags[2])
        return set_err(QA_EZERONORM, "angular metric needs nonzero corpus and query vectors");
    const int32_t any = hflags[0];
    unsigned long long cands = 0;
    std::memcpy(&cands, hflags + 4, sizeof(cands));
    g_stats.candidates += (int64_t)cands;
    g_timer.accumulate(g_stats);
    if (any) {
        std::vector<int32_t> h(nq);
        QA_TRY(cudaMemcpy(h.data(), ovf, (size_t)nq * 4, cudaMemcpyDeviceToHost), "overflow list");
        for (int64_t i = 0; i < nq; ++i)
            if (h[i]) overflowed->push_back((int32_t)i);
    }
    return QA_OK;
}

// Body of qa_scan_topk_f32 (validated arguments, workspace lock held).
int f32_impl(Workspace &ws, const float *db, int64_t n, int64_t d, int64_t ldd,
             const float *db_norm, const float *q, int64_t nq, int64_t ldq, const float *q_norm,
             int64_t keff, int metric, int64_t id_offset, double *out_scores, int32_t *out_ids,
             cudaStream_t st) {
    if (n > INT32_MAX || d > INT32_MAX) return set_err(QA_EUNSUPPORTED, "shape above this build's limit");
    if (keff > kMaxKF32) {
        // any k: every score of a query chunk, stable-sorted per query
        // (keff rows of the full (score, id) order, _core.pyx:348-365)
        int64_t m = std::max<int64_t>(1, ((int64_t)2 << 30) / (32 * n));
        m = std::min<int64_t>({m, nq, (int64_t)INT32_MAX / n, 65535});
        const size_t need = f32_fullsort_bytes(m, n);
        QA_TRY(ws.f32_full.reserve(need), "workspace");
        for (int64_t c0 = 0; c0 < nq; c0 += m) {
            const int64_t mm = std::min(m, nq - c0);
            QA_TRY(launch_f32_fullsort(db, ldd, q + c0 * ldq, ldq, d, mm, n, metric, db_norm,
                                       q_norm ? q_norm + c0 : nullptr, keff, id_offset,
                                       out_scores + c0 * keff, out_ids + c0 * keff, ws.f32_full.ptr,
                                       ws.f32_full.bytes, st),
                   "f32 full sort");
        }
        return QA_OK;
    }
    constexpr int64_t kF32Rows = 16384, kF32Queries = 1024;
    const int64_t R = std::min(n, kF32Rows);
    const int64_t qc = std::min(nq, kF32Queries);
    QA_TRY(ws.f32_scores.reserve((size_t)qc * R * 8), "workspace");
    QA_TRY(ws.f32_ss.reserve((size_t)qc * keff * 8), "workspace");
    QA_TRY(ws.f32_si.reserve((size_t)qc * keff * 4), "workspace");
    QA_TRY(ws.f32_sn.reserve((size_t)qc * 4), "workspace");
    double *sc = (double *)ws.f32_scores.ptr, *ss = (double *)ws.f32_ss.ptr;
    int32_t *si = (int32_t *)ws.f32_si.ptr, *sn = (int32_t *)ws.f32_sn.ptr;
    for (int64_t c0 = 0; c0 < nq; c0 += qc) {
        const int64_t m = std::min(qc, nq - c0);
        QA_TRY(cudaMemsetAsync(sn, 0, (size_t)m * 4, st), "memset");
        for (int64_t r0 = 0; r0 < n; r0 += R) {
            const int64_t rows = std::min(R, n - r0);
            QA_TRY(launch_f32_scores(db, ldd, q + c0 * ldq, ldq, d, m, r0, rows, metric, db_norm,
                                     q_norm ? q_norm + c0 : nullptr, sc, R, st),
                   "f32 scores");
            QA_TRY(launch_f32_select(sc, R, rows, r0, ss, si, sn, m, keff, st), "f32 select");
        }
        QA_TRY(launch_f32_finalize(ss, si, m, keff, id_offset, out_scores + c0 * keff,
                                   out_ids + c0 * keff, st),
               "f32 finalize");
    }
    return QA_OK;
}

// int8 codes [n, ld] (stored order, row_ids -> caller order) as float32
// [n, d] rows in CALLER order; norms likewise.  Every int8 dot, l2 and
// angular score is an exact float64 computation on these values, so the
// float32 scan reproduces the int8 path bit for bit (used for k beyond the
// int8 select's limit).
__global__ void codes_to_f32_kernel(const int8_t *__restrict__ codes, int64_t n, int64_t d,
                                    int64_t ld, const int32_t *__restrict__ row_ids,
                                    const float *__restrict__ norm_in, float *__restrict__ out,
                                    float *__restrict__ norm_out) {
    const int64_t r = blockIdx.x;
    if (r >= n) return;
    const int64_t dst = row_ids ? (int64_t)row_ids[r] : r;
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) out[dst * d + j] = (float)codes[r * ld + j];
    if (threadIdx.x == 0 && norm_in) norm_out[dst] = norm_in[r];
}

int scan_entry(const int8_t *db, int64_t n, int64_t d, int64_t ldd, const int32_t *db_sqnorm,
               const float *db_norm, const int32_t *row_ids, const int8_t *q, int64_t nq, int64_t ldq,
               const int32_t *q_sqnorm, const float *q_norm, int64_t k, int metric,
               int64_t id_offset, double *out_scores, int32_t *out_ids, cudaStream_t st,
               bool async_ = false) {
    g_stats = qa_scan_stats{};
    if (metric < 0 || metric > 2) return set_err(QA_EINVAL, "unknown metric %d", metric);
    if (k < 0) return set_err(QA_EINVAL, "k must be >= 0");
    if (n < 0 || nq < 0 || d < 0) return set_err(QA_EINVAL, "negative shape");
    const int64_t ld = qa_code_stride(d);
    if (ldd != ld || ldq != ld)
        return set_err(QA_EINVAL, "code row stride must be qa_code_stride(d)=%lld",
                       (long long)ld);
    const int64_t keff = std::min(k, n);
    if (n == 0 || nq == 0 || keff == 0) return QA_OK;
    if (metric == kAngular && (!db_norm || !q_norm))
        return set_err(QA_EINVAL, "angular metric needs data and query norms");
    if (metric == kL2 && (!db_sqnorm || !q_sqnorm))
        return set_err(QA_EINVAL, "L2 metric needs data and query squared norms");
    if (n > INT32_MAX) return set_err(QA_EUNSUPPORTED, "n exceeds int32 ids");
    // Widths whose worst-case int32 sum could wrap (|dot| <= d*128^2, l2 <=
    // d*255^2; the reference accumulates in C int, _core.pyx:49-63) take the
    // float64-exact route below, like large k: identical to the reference
    // whenever its int32 sums do not overflow.
    const bool wide_d = d > 131071 || (metric == kL2 && d > 33025);
    Workspace &ws = g_ws[current_device() % kMaxDevices];
    std::lock_guard<std::mutex> lock(ws.mu);
    if (keff > kMaxK || wide_d) {
        // large k (or wide rows): the float64-exact scan on the codes as
        // float32 (bit-exact with the int8 path, see codes_to_f32_kernel),
        // caller row order
        QA_TRY(ws.f32_x.reserve((size_t)n * d * 4 + 16), "workspace");
        QA_TRY(ws.f32_q.reserve((size_t)nq * d * 4 + 16), "workspace");
        QA_TRY(ws.f32_xn.reserve((size_t)n * 4 + 16), "workspace");
        float *xf = (float *)ws.f32_x.ptr, *qf = (float *)ws.f32_q.ptr, *xn = (float *)ws.f32_xn.ptr;
        codes_to_f32_kernel<<<(unsigned)n, 128, 0, st>>>(db, n, d, ld, row_ids,
                                                         metric == kAngular ? db_norm : nullptr,
                                                         xf, xn);
        codes_to_f32_kernel<<<(unsigned)nq, 128, 0, st>>>(q, nq, d, ld, nullptr, nullptr, qf,
                                                          nullptr);
        QA_TRY(cudaGetLastError(), "large-k path");
        if (metric == kAngular) {
            int32_t zf = 0;
            QA_TRY(ws.flags.reserve(64), "workspace");
            int32_t *dflag = (int32_t *)ws.flags.ptr + 2;
            QA_TRY(cudaMemsetAsync(dflag, 0, 4, st), "large-k path");
            zero_norm_kernel<<<(unsigned)((n + nq + 255) / 256), 256, 0, st>>>(db_norm, n, q_norm,
                                                                               nq, dflag);
            QA_TRY(cudaMemcpyAsync(&zf, dflag, 4, cudaMemcpyDeviceToHost, st), "large-k path");
            QA_TRY(cudaStreamSynchronize(st), "large-k path");
            if (zf) return set_err(QA_EZERONORM, "angular metric needs nonzero corpus and query vectors");
        }
        const int rc = f32_impl(ws, xf, n, d, d, metric == kAngular ? xn : nullptr, qf, nq, d,
                                metric == kAngular ? q_norm : nullptr, keff, metric, id_offset,
                                out_scores, out_ids, st);
        if (rc != QA_OK) return rc;
        // the workspace is reused by the next call on any stream
        QA_TRY(cudaStreamSynchronize(st), "large-k path");
        return QA_OK;
    }
    std::vector<int32_t> ovf;
    if (!async_) g_timer.reset();
    int rc = scan_impl(ws, db, n, d, ld, db_sqnorm, db_norm, row_ids, q, nq, q_sqnorm, q_norm, keff, metric,
                       id_offset, out_scores, out_ids, 0, true, st, &ovf, async_);
    if (rc != QA_OK) return rc;
    int64_t cap = plan_scan(n, nq, keff, 0, true).cap;
    while (!ovf.empty()) {
        // Recompute the overflowed queries with 4x the candidate capacity;
        // once cap >= n no list can overflow.
        g_stats.retries += 1;
        cap = std::min<int64_t>(cap * 4, std::max<int64_t>(n, 2048));
        const int64_t m = (int64_t)ovf.size();
        QA_TRY(ws.r_idx.reserve((size_t)m * 4), "workspace");
        QA_TRY(ws.r_q.reserve((size_t)m * ld), "workspace");
        QA_TRY(ws.r_qsq.reserve((size_t)m * 4), "workspace");
        QA_TRY(ws.r_qn.reserve((size_t)m * 4), "workspace");
        QA_TRY(ws.r_s.reserve((size_t)m * keff * 8), "workspace");
        QA_TRY(ws.r_ids.reserve((size_t)m * keff * 4), "workspace");
        int32_t *idx = (int32_t *)ws.r_idx.ptr;
        int8_t *qsub = (int8_t *)ws.r_q.ptr;
        int32_t *qsq = (int32_t *)ws.r_qsq.ptr;
        float *qn = (float *)ws.r_qn.ptr;
        double *s = (double *)ws.r_s.ptr;
        int32_t *ids = (int32_t *)ws.r_ids.ptr;
        QA_TRY(cudaMemcpyAsync(idx, ovf.data(), m * 4, cudaMemcpyHostToDevice, st), "retry");
        gather_rows_kernel<<<(unsigned)m, 128, 0, st>>>(q, ld, idx, m, qsub);
        if (q_sqnorm)
            gather_vals_kernel<int32_t><<<(unsigned)((m + 255) / 256), 256, 0, st>>>(q_sqnorm, idx,
                                                                                   m, qsq);
        if (q_norm)
            gather_vals_kernel<float><<<(unsigned)((m + 255) / 256), 256, 0, st>>>(q_norm, idx, m,
                                                                                 qn);
        std::vector<int32_t> ovf2;
        rc = scan_impl(ws, db, n, d, ld, db_sqnorm, db_norm, row_ids, qsub, m, q_sqnorm ? qsq : nullptr,
                       q_norm ? qn : nullptr, keff, metric, id_offset, s, ids, cap, false, st,
                       &ovf2);
        if (rc == QA_OK) {
            scatter_results_kernel<<<(unsigned)((m * keff + 255) / 256), 256, 0, st>>>(
                s, ids, idx, m, keff, out_scores, out_ids);
            cudaError_t e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) rc = cuda_err(e, "retry");
        }
        // map second-level overflow indices back to original query ids
        std::vector<int32_t> next;
        for (int32_t i : ovf2) next.push_back(ovf[i]);
        if (rc != QA_OK) return rc;
        ovf.swap(next);
        if (cap >= n && !ovf.empty())
            return set_err(QA_ECUDA, "internal: overflow at full capacity");
    }
    return QA_OK;
}

void add_totals() {
    g_totals.rounds += g_stats.rounds;
    g_totals.candidates += g_stats.candidates;
    g_totals.launches += g_stats.launches;
    g_totals.retries += g_stats.retries;
    g_totals.filter_launches += g_stats.filter_launches;
    g_totals.filter_ops += g_stats.filter_ops;
    g_totals.filter_ms += g_stats.filter_ms;
    g_totals.select_ms += g_stats.select_ms;
}

}  // namespace

int num_sms() {
    static int cached[kMaxDevices] = {0};
    int dev = current_device() % kMaxDevices;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

}  // namespace qa

using namespace qa;

extern "C" {

int qa_version(void) { return 1; }

const char *qa_last_error(void) { return g_err.c_str(); }

int qa_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

int64_t qa_code_stride(int64_t d) {
    if (d <= 32) return 32;
    if (d <= 64) return 64;
    return (d + 127) / 128 * 128;
}

int qa_set_profiling(int on) {
    g_profiling = on != 0;
    return QA_OK;
}

int qa_last_scan_stats(qa_scan_stats *out) {
    if (!out) return set_err(QA_EINVAL, "null stats pointer");
    *out = g_stats;
    return QA_OK;
}

int qa_scan_totals(qa_scan_stats *out) {
    if (!out) return set_err(QA_EINVAL, "null stats pointer");
    g_timer.accumulate(g_totals);  // timing spans of asynchronous scans
    *out = g_totals;
    return QA_OK;
}

int qa_reset_scan_totals(void) {
    g_timer.reset();
    g_totals = qa_scan_stats{};
    return QA_OK;
}

int qa_minmax_f32(const float *x, int64_t n, int64_t d, int64_t ldx, float *out_min,
                  float *out_max, void *stream) {
    if (n < 0 || d < 1 || ldx < d) return set_err(QA_EINVAL, "bad shape");
    cudaStream_t st = (cudaStream_t)stream;
    Workspace &ws = g_ws[current_device() % kMaxDevices];
    std::lock_guard<std::mutex> lock(ws.mu);
    int64_t floats = (int64_t)num_sms() * 4 * 2 * d;
    QA_TRY(ws.scratch.reserve((size_t)floats * 4), "workspace");
    QA_TRY(launch_minmax(x, n, d, ldx, out_min, out_max, (float *)ws.scratch.ptr, floats, st),
           "minmax");
    // the shared scratch is free for the next caller (any stream) only once
    // this call's kernels are done (build-time entry: the sync is cheap)
    QA_TRY(cudaStreamSynchronize(st), "minmax");
    return QA_OK;
}

int qa_encode_i8(const float *x, int64_t n, int64_t d, int64_t ldx, const float *k,
                 const float *sb, const float *se, int bits, int8_t *codes, int64_t ldc,
                 int32_t *sqnorm, float *norm, void *stream) {
    if (bits < 1 || bits > 8) return set_err(QA_EINVAL, "bits must be between 1 and 8");
    if (n < 0 || d < 0 || ldx < d || ldc < d) return set_err(QA_EINVAL, "bad shape");
    QA_TRY(launch_encode(x, n, d, ldx, k, sb, se, bits, codes, ldc, sqnorm, norm,
                         (cudaStream_t)stream),
           "encode");
    return QA_OK;
}

int qa_norms_i8(const int8_t *codes, int64_t n, int64_t d, int64_t ldc, int32_t *sqnorm,
                float *norm, void *stream) {
    if (n < 0 || d < 0 || ldc < d) return set_err(QA_EINVAL, "bad shape");
    QA_TRY(launch_norms(codes, n, d, ldc, sqnorm, norm, (cudaStream_t)stream), "norms");
    return QA_OK;
}

int qa_gather_scores_i8(const int8_t *db, int64_t n, int64_t d, int64_t ldd,
                        const int32_t *db_sqnorm, const float *db_norm, const int32_t *row_of_id,
                        const int8_t *q, int64_t nq, int64_t ldq, const int32_t *q_sqnorm,
                        const float *q_norm, const int32_t *cand, int64_t m, int64_t ldcand,
                        int metric, double *out_scores, void *stream) {
    if (metric < 0 || metric > 2) return set_err(QA_EINVAL, "unknown metric %d", metric);
    if (n < 0 || nq < 0 || d < 0 || m < 0) return set_err(QA_EINVAL, "negative shape");
    if (ldd < d || ldq < d || ldcand < m) return set_err(QA_EINVAL, "bad stride");
    if (nq == 0 || m == 0) return QA_OK;
    if (ldd % 16 != 0 || ldq % 16 != 0 || ((uintptr_t)db % 16) != 0 || ((uintptr_t)q % 16) != 0)
        return set_err(QA_EINVAL, "code rows must be 16-byte aligned (qa_code_stride)");
    if (metric == kL2 && (!db_sqnorm || !q_sqnorm))
        return set_err(QA_EINVAL, "the L2 metric needs the squared code norms");
    if (metric == kAngular && (!db_norm || !q_norm))
        return set_err(QA_EINVAL, "angular metric needs data and query norms");
    if (metric == kL2 && d > 33025)
        return set_err(QA_EUNSUPPORTED, "rows wider than the int32-safe range");
    QA_TRY(launch_gather_scores(db, n, ldd, db_sqnorm, db_norm, row_of_id, q, nq, ldq, q_sqnorm,
                                q_norm, cand, m, ldcand, metric, out_scores, (cudaStream_t)stream),
           "gather scores");
    return QA_OK;
}

int qa_scan_topk_i8(const int8_t *db, int64_t n, int64_t d, int64_t ldd, const int32_t *db_sqnorm,
                    const float *db_norm, const int32_t *row_ids, const int8_t *q, int64_t nq,
                    int64_t ldq,
                    const int32_t *q_sqnorm, const float *q_norm, int64_t k, int metric,
                    int64_t id_offset, double *out_scores, int32_t *out_ids, void *stream) {
    const int rc = scan_entry(db, n, d, ldd, db_sqnorm, db_norm, row_ids, q, nq, ldq, q_sqnorm,
                              q_norm, k, metric, id_offset, out_scores, out_ids,
                              (cudaStream_t)stream);
    add_totals();
    return rc;
}

int qa_scan_topk_i8_async(const int8_t *db, int64_t n, int64_t d, int64_t ldd,
                          const int32_t *db_sqnorm, const float *db_norm, const int32_t *row_ids,
                          const int8_t *q, int64_t nq, int64_t ldq, const int32_t *q_sqnorm,
                          const float *q_norm, int64_t k, int metric, int64_t id_offset,
                          double *out_scores, int32_t *out_ids, void *stream) {
    const int rc = scan_entry(db, n, d, ldd, db_sqnorm, db_norm, row_ids, q, nq, ldq, q_sqnorm,
                              q_norm, k, metric, id_offset, out_scores, out_ids,
                              (cudaStream_t)stream, true);
    add_totals();
    return rc;
}

int qa_scan_topk_i8_host(const int8_t *data, int64_t n, int64_t d, const int8_t *queries,
                         int64_t nq, int64_t k, int metric, const float *data_norms,
                         const float *query_norms, double *out_scores, int32_t *out_ids) {
    if (metric < 0 || metric > 2) return set_err(QA_EINVAL, "unknown metric %d", metric);
    if (k < 0) return set_err(QA_EINVAL, "k must be >= 0");
    if (n < 0 || nq < 0 || d < 0) return set_err(QA_EINVAL, "negative shape");
    const int64_t keff = std::min(k, n);
    if (n == 0 || nq == 0 || keff == 0) return QA_OK;
    if (metric == kAngular && (!data_norms || !query_norms))
        return set_err(QA_EINVAL, "angular metric needs data and query norms");
    const int64_t ld = qa_code_stride(d);
    cudaStream_t st = nullptr;
    QA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    int8_t *ddb = nullptr, *dq = nullptr;
    int32_t *dsq = nullptr, *qsq = nullptr, *dids = nullptr;
    float *dn = nullptr, *qn = nullptr;
    double *ds = nullptr;
    int rc = QA_OK;
    auto fail = [&](cudaError_t e, const char *w) { rc = cuda_err(e, w); };
    do {
        cudaError_t e;
        if ((e = cudaMalloc(&ddb, n * ld)) != cudaSuccess) { fail(e, "alloc"); break; }
        if ((e = cudaMalloc(&dq, nq * ld)) != cudaSuccess) { fail(e, "alloc"); break; }
        if ((e = cudaMalloc(&dsq, n * 4)) != cudaSuccess) { fail(e, "alloc"); break; }
        if ((e = cudaMalloc(&qsq, nq * 4)) != cudaSuccess) { fail(e, "alloc"); break; }
        if ((e = cudaMalloc(&dn, n * 4)) != cudaSuccess) { fail(e, "alloc"); break; }
        if ((e = cudaMalloc(&qn, nq * 4)) != cudaSuccess) { fail(e, "alloc"); break; }
        if ((e = cudaMalloc(&ds, nq * keff * 8)) != cudaSuccess) { fail(e, "alloc"); break; }
        if ((e = cudaMalloc(&dids, nq * keff * 4)) != cudaSuccess) { fail(e, "alloc"); break; }
        if (ld != d) {
            cudaMemsetAsync(ddb, 0, n * ld, st);
            cudaMemsetAsync(dq, 0, nq * ld, st);
        }
        if (d > 0) {
            cudaMemcpy2DAsync(ddb, ld, data, d, d, n, cudaMemcpyHostToDevice, st);
            cudaMemcpy2DAsync(dq, ld, queries, d, d, nq, cudaMemcpyHostToDevice, st);
        }
        launch_norms(ddb, n, d, ld, dsq, nullptr, st);
        launch_norms(dq, nq, d, ld, qsq, nullptr, st);
        if (metric == kAngular) {
            cudaMemcpyAsync(dn, data_norms, n * 4, cudaMemcpyHostToDevice, st);
            cudaMemcpyAsync(qn, query_norms, nq * 4, cudaMemcpyHostToDevice, st);
        }
        if ((e = cudaGetLastError()) != cudaSuccess) { fail(e, "upload"); break; }
        rc = scan_entry(ddb, n, d, ld, dsq, dn, nullptr, dq, nq, ld, qsq, qn, k, metric, 0, ds, dids, st);
        if (rc != QA_OK) break;
        cudaMemcpyAsync(out_scores, ds, nq * keff * 8, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(out_ids, dids, nq * keff * 4, cudaMemcpyDeviceToHost, st);
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { fail(e, "download"); break; }
    } while (0);
    cudaFree(ddb);
    cudaFree(dq);
    cudaFree(dsq);
    cudaFree(qsq);
    cudaFree(dn);
    cudaFree(qn);
    cudaFree(ds);
    cudaFree(dids);
    cudaStreamDestroy(st);
    return rc;
}

int qa_norms_f32(const float *x, int64_t n, int64_t d, int64_t ldx, float *out, void *stream) {
    if (n < 0 || d < 0 || ldx < d) return set_err(QA_EINVAL, "bad shape");
    QA_TRY(launch_norms_f32(x, n, d, ldx, out, (cudaStream_t)stream), "norms");
    return QA_OK;
}

// float32 exhaustive search: rows in rounds of kF32Rows; every round scores
// (query chunk x round rows) in float64 exactly as _scan_f32 does, then the
// select kernel merges the round into each query's (score, id) state.
int qa_scan_topk_f32(const float *db, int64_t n, int64_t d, int64_t ldd, const float *db_norm,
                     const float *q, int64_t nq, int64_t ldq, const float *q_norm, int64_t k,
                     int metric, int64_t id_offset, double *out_scores, int32_t *out_ids,
                     void *stream) {
    if (metric < 0 || metric > 2) return set_err(QA_EINVAL, "unknown metric %d", metric);
    if (k < 0) return set_err(QA_EINVAL, "k must be >= 0");
    if (n < 0 || nq < 0 || d < 0 || ldd < d || ldq < d) return set_err(QA_EINVAL, "bad shape");
    const int64_t keff = std::min(k, n);
    if (n == 0 || nq == 0 || keff == 0) return QA_OK;
    if (metric == kAngular && (!db_norm || !q_norm))
        return set_err(QA_EINVAL, "angular metric needs data and query norms");
    Workspace &ws = g_ws[current_device() % kMaxDevices];
    std::lock_guard<std::mutex> lock(ws.mu);
    return f32_impl(ws, db, n, d, ldd, db_norm, q, nq, ldq, q_norm, keff, metric, id_offset,
                    out_scores, out_ids, (cudaStream_t)stream);
}

int qa_estimate_stats_f32(const float *x, int64_t n, int64_t d, int64_t ldx, double *mu,
                          double *sigma, double *mn, double *mx, double *tam, double *qlo,
                          double *qhi, double *pooled_mu, double *pooled_sigma, void *stream) {
    if (n < 2) return set_err(QA_EINVAL, "need at least 2 vectors, got %lld", (long long)n);
    if (d < 1 || ldx < d) return set_err(QA_EINVAL, "bad shape");
    if (!mu || !sigma || !mn || !mx || !tam || !pooled_mu || !pooled_sigma)
        return set_err(QA_EINVAL, "null output");
    std::vector<double> lo_buf, hi_buf;
    if (!qlo) {
        lo_buf.resize((size_t)d);
        qlo = lo_buf.data();
    }
    if (!qhi) {
        hi_buf.resize((size_t)d);
        qhi = hi_buf.data();
    }
    QA_TRY(launch_estimate_stats(x, n, d, ldx, mu, sigma, mn, mx, tam, qlo, qhi, pooled_mu,
                                 pooled_sigma, (cudaStream_t)stream),
           "estimate_stats");
    return QA_OK;
}

int qa_order_rows_by_norm(const int32_t *sqnorm, int64_t n, int stratify, int32_t *perm,
                          void *stream) {
    if (n < 0 || n > INT32_MAX) return set_err(QA_EINVAL, "bad shape");
    if (n == 0) return QA_OK;
    cudaStream_t st = (cudaStream_t)stream;
    Workspace &ws = g_ws[current_device() % kMaxDevices];
    std::lock_guard<std::mutex> lock(ws.mu);
    size_t need = 0;
    QA_TRY(launch_order_by_key(sqnorm, n, stratify != 0, perm, nullptr, 0, &need, st), "order");
    QA_TRY(ws.scratch.reserve(need), "workspace");
    QA_TRY(launch_order_by_key(sqnorm, n, stratify != 0, perm, ws.scratch.ptr, ws.scratch.bytes,
                              &need, st),
           "order");
    QA_TRY(cudaStreamSynchronize(st), "order");  // shared scratch (see qa_minmax_f32)
    return QA_OK;
}

int qa_permute_rows_i8(const int8_t *codes, const int32_t *sqnorm, const float *norm, int64_t n,
                       int64_t ldc, const int32_t *perm, int8_t *codes_out, int32_t *sqnorm_out,
                       float *norm_out, void *stream) {
    if (n < 0 || ldc % 16 != 0) return set_err(QA_EINVAL, "bad shape");
    QA_TRY(launch_permute_rows(codes, sqnorm, norm, n, ldc, perm, codes_out, sqnorm_out, norm_out,
                               (cudaStream_t)stream),
           "permute");
    return QA_OK;
}

int qa_merge_topk(const double *in_scores, const int32_t *in_ids, int64_t G, int64_t nq,
                  int64_t kin, int64_t k, double *out_scores, int32_t *out_ids, void *stream) {
    if (G < 1 || nq < 0 || kin < 0 || k < 0) return set_err(QA_EINVAL, "bad shape");
    if (k > G * kin) return set_err(QA_EINVAL, "k exceeds the number of merged entries");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t need = merge_scratch_bytes(G, nq, kin, k);
    if (need == 0) {
        QA_TRY(launch_merge(in_scores, in_ids, G, nq, kin, k, out_scores, out_ids, st), "merge");
        return QA_OK;
    }
    // large k: merge-path tree through a workspace buffer
    Workspace &ws = g_ws[current_device() % kMaxDevices];
    std::lock_guard<std::mutex> lock(ws.mu);
    QA_TRY(ws.merge.reserve(need), "workspace");
    QA_TRY(launch_merge(in_scores, in_ids, G, nq, kin, k, out_scores, out_ids, st, ws.merge.ptr),
           "merge");
    QA_TRY(cudaStreamSynchronize(st), "merge");  // the buffer is shared per device
    return QA_OK;
}

int qa_debug_dots_i8(const int8_t *db, int64_t n, const int8_t *q, int64_t nq, int64_t d,
                     int impl, int32_t *out, void *stream) {
    if (n < 1 || nq < 1 || d < 0) return set_err(QA_EINVAL, "bad shape");
    const int64_t ld = qa_code_stride(d);
    FilterArgs fa{};
    fa.db = db;
    fa.ldd = ld;
    fa.q = q;
    fa.ldq = ld;
    fa.kdim = ld;
    fa.nq = nq;
    fa.r_lo = 0;
    fa.r_hi = n;
    fa.metric = kIP;
    fa.mode = 2;
    fa.dots_out = out;
    fa.ld_dots = n;
    cudaStream_t st = (cudaStream_t)stream;
    Workspace &ws = g_ws[current_device() % kMaxDevices];
    std::lock_guard<std::mutex> lock(ws.mu);
    QA_TRY(ws.flags.reserve(64), "workspace");
    QA_TRY(ws.sched.reserve((size_t)kSchedSlots * 4), "workspace");
    fa.sched = (unsigned *)ws.sched.ptr;
    QA_TRY(cudaMemsetAsync(fa.sched, 0, 4, st), "sched");
    cudaError_t e = impl == 0 ? launch_filter_tc(fa, st)
                              : launch_filter_simt(fa, st);
    QA_TRY(e, "debug dots");
    return QA_OK;
}

}  // extern "C"
