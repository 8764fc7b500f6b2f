/*
 * qa_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file: it is the checker that tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg compare the CUDA path against.
 *
 * Every function restates one reference routine (paths relative to
 * /root/reference/pkg/src/quantann):
 *
 *   qo_encode_i8     quantizer.py:291-300  (_quantize_matrix, Eq. 1)
 *   qo_norms_i8      _core.pyx:137-157     (norms, int8 branch via _sumsq_i 66-74)
 *   qo_minmax_f32    per-dim min/max (quantizer.py:196-197 block.min/max)
 *   qo_scan_topk_i8  _core.pyx:301-365     (_scan_i8 + scan_topk; pair kernel 49-96)
 *   qo_norms_f32     _core.pyx:150-153     (norms, float32 branch via _dot_f 32-37)
 *   qo_scan_topk_f32 _core.pyx:270-298     (_scan_f32; pair kernel 32-46, 75-84)
 *
 * Pinned against the reference's own compiled _core (oracle/_ref) and against
 * the golden vectors in tests/golden/ -- see tests/test_oracle.py.
 *
 * Build: oracle/Makefile (gcc -O2 -fno-fast-math -ffp-contract=off; fp32
 * arithmetic must stay IEEE round-to-nearest exactly as numpy's).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* quantizer.py:291-300.  All arithmetic in the order numpy evaluates it:
 *   ratio = fp32(fp32(x - k) / fp32(se - sb))
 *   q     = clip(floor(double(fp32(2^bits * ratio))), lo, hi)
 *   code  = in_window ? q : (x > se ? hi : lo)    (window tests in float64,
 *           so NaN is neither in-window nor above: it maps to lo). */
void qo_encode_i8(const float *x, int64_t n, int64_t d, const float *k,
                  const float *sb, const float *se, int bits, int8_t *out) {
    const double lo = -(double)(1 << (bits - 1));
    const double hi = (double)((1 << (bits - 1)) - 1);
    const float scale = (float)(1 << bits);
    for (int64_t i = 0; i < n; ++i) {
        const float *row = x + i * d;
        int8_t *orow = out + i * d;
        for (int64_t j = 0; j < d; ++j) {
            volatile float w = se[j] - sb[j];
            volatile float num = row[j] - k[j];
            volatile float ratio = num / w;
            volatile float t = scale * ratio;
            double q = floor((double)t);
            if (q < lo) q = lo;
            if (q > hi) q = hi;
            double xv = (double)row[j];
            double code;
            if (xv >= (double)sb[j] && xv <= (double)se[j])
                code = q;
            else if (xv > (double)se[j])
                code = hi;
            else
                code = lo;
            orow[j] = (int8_t)(int)code;
        }
    }
}

/* _core.pyx:154-156: float32(sqrt(double(int64 sum c^2))); n==0 or d==0 -> 0. */
void qo_norms_i8(const int8_t *x, int64_t n, int64_t d, float *out) {
    for (int64_t i = 0; i < n; ++i) {
        long long acc = 0;
        for (int64_t j = 0; j < d; ++j) {
            int t = (int)x[i * d + j];
            acc += (long long)(t * t);
        }
        out[i] = (float)sqrt((double)acc);
    }
}

/* Per-dimension min and max of a float32 matrix (float64 outputs; exact). */
void qo_minmax_f32(const float *x, int64_t n, int64_t d, double *mn, double *mx) {
    for (int64_t j = 0; j < d; ++j) {
        mn[j] = INFINITY;
        mx[j] = -INFINITY;
    }
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < d; ++j) {
            double v = (double)x[i * d + j];
            if (v < mn[j]) mn[j] = v;
            if (v > mx[j]) mx[j] = v;
        }
}

/* ---- (score, id) lexicographic order, _core.pyx:164-173 ---------------- */
static inline int lex_gt(double d1, int i1, double d2, int i2) {
    if (d1 != d2) return d1 > d2;
    return i1 > i2;
}

/* Bounded max-heap keyed on (score, id): the worst retained entry on top. */
static void heap_sift_down(double *hd, int *hi, int size, int c) {
    for (;;) {
        int l = 2 * c + 1, r = l + 1, m = c;
        if (l < size && lex_gt(hd[l], hi[l], hd[m], hi[m])) m = l;
        if (r < size && lex_gt(hd[r], hi[r], hd[m], hi[m])) m = r;
        if (m == c) return;
        double td = hd[c]; hd[c] = hd[m]; hd[m] = td;
        int ti = hi[c]; hi[c] = hi[m]; hi[m] = ti;
        c = m;
    }
}

static void heap_push(double *hd, int *hi, int size, double d, int id) {
    int c = size;
    hd[c] = d;
    hi[c] = id;
    while (c > 0) {
        int p = (c - 1) >> 1;
        if (!lex_gt(hd[c], hi[c], hd[p], hi[p])) break;
        double td = hd[c]; hd[c] = hd[p]; hd[p] = td;
        int ti = hi[c]; hi[c] = hi[p]; hi[p] = ti;
        c = p;
    }
}

/* _core.pyx:88-96 metric mapping of one int8 pair. */
static inline double pair_i8(const int8_t *a, const int8_t *b, int64_t d, int metric,
                             double na, double nb) {
    int acc = 0;
    if (metric == 1) {
        for (int64_t j = 0; j < d; ++j) {
            int t = (int)a[j] - (int)b[j];
            acc += t * t;
        }
        return (double)acc;
    }
    for (int64_t j = 0; j < d; ++j) acc += (int)a[j] * (int)b[j];
    if (metric == 0) return -(double)acc;
    return 1.0 - (double)acc / (na * nb);
}

/* _core.pyx:301-330 semantics: result row q = first keff entries of the
 * (score, id)-sorted list of all n rows.  keff = min(k, n); caller sizes
 * out_d/out_i as nq*keff.  Returns keff. */
int64_t qo_scan_topk_i8(const int8_t *X, int64_t n, int64_t d, const int8_t *Q,
                        int64_t nq, int64_t k, int metric, const float *xn,
                        const float *qn, double *out_d, int32_t *out_i) {
    int64_t keff = k < n ? k : n;
    if (n == 0 || nq == 0 || keff == 0) return keff;
#pragma omp parallel
    {
        double *hd = (double *)malloc(sizeof(double) * (size_t)(keff + 1));
        int *hi = (int *)malloc(sizeof(int) * (size_t)(keff + 1));
#pragma omp for schedule(dynamic, 1)
        for (int64_t q = 0; q < nq; ++q) {
            const int8_t *qp = Q + q * d;
            double qnorm = metric == 2 ? (double)qn[q] : 0.0;
            int size = 0;
            for (int64_t r = 0; r < n; ++r) {
                double dv = pair_i8(qp, X + r * d, d, metric, qnorm,
                                    metric == 2 ? (double)xn[r] : 0.0);
                if (size < keff) {
                    heap_push(hd, hi, size, dv, (int)r);
                    ++size;
                } else if (lex_gt(hd[0], hi[0], dv, (int)r)) {
                    hd[0] = dv;
                    hi[0] = (int)r;
                    heap_sift_down(hd, hi, size, 0);
                }
            }
            /* pop worst-first into descending slots -> ascending rows */
            for (int j = size - 1; j >= 0; --j) {
                out_d[q * keff + j] = hd[0];
                out_i[q * keff + j] = hi[0];
                --size;
                hd[0] = hd[size];
                hi[0] = hi[size];
                heap_sift_down(hd, hi, size, 0);
            }
        }
        free(hd);
        free(hi);
    }
    return keff;
}

/* ---- float32 path: _core.pyx:32-46 (_dot_f/_l2_f), 75-84 (_pair_f),
 * 150-153 (norms, float32 branch), 270-298 (_scan_f32).  Sequential float64
 * accumulation in j order; built with -ffp-contract=off so t*t and the adds
 * round separately exactly as the reference's C does (no FMA on x86-64
 * baseline). ------------------------------------------------------------ */
/* Scores of listed (query, row) pairs: out[q, j] = pair_i8(Q[q], X[cand[q, j]])
 * -- HnswCore._dq for an external int8 query (_core.pyx:483-494 -> _pair_i,
 * 88-96); an id outside [0, n) gives +inf (padding of ragged lists). */
void qo_pair_scores_i8(const int8_t *X, int64_t n, int64_t d, const int8_t *Q, int64_t nq,
                       const int32_t *cand, int64_t m, int metric, const float *xn,
                       const float *qn, double *out) {
    for (int64_t q = 0; q < nq; ++q)
        for (int64_t j = 0; j < m; ++j) {
            const int32_t id = cand[q * m + j];
            if (id < 0 || id >= n) {
                out[q * m + j] = INFINITY;
                continue;
            }
            out[q * m + j] = pair_i8(Q + q * d, X + (int64_t)id * d, d, metric,
                                     metric == 2 ? (double)qn[q] : 0.0,
                                     metric == 2 ? (double)xn[id] : 0.0);
        }
}

static inline double pair_f32(const float *a, const float *b, int64_t d, int metric,
                              double na, double nb) {
    double acc = 0.0;
    if (metric == 1) {
        for (int64_t j = 0; j < d; ++j) {
            double t = (double)a[j] - (double)b[j];
            acc += t * t;
        }
        return acc;
    }
    for (int64_t j = 0; j < d; ++j) acc += (double)a[j] * (double)b[j];
    if (metric == 0) return -acc;
    return 1.0 - acc / (na * nb);
}

void qo_norms_f32(const float *x, int64_t n, int64_t d, float *out) {
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t j = 0; j < d; ++j) acc += (double)x[i * d + j] * (double)x[i * d + j];
        out[i] = (float)sqrt(acc);
    }
}

int64_t qo_scan_topk_f32(const float *X, int64_t n, int64_t d, const float *Q, int64_t nq,
                         int64_t k, int metric, const float *xn, const float *qn,
                         double *out_d, int32_t *out_i) {
    int64_t keff = k < n ? k : n;
    if (n == 0 || nq == 0 || keff == 0) return keff;
#pragma omp parallel
    {
        double *hd = (double *)malloc(sizeof(double) * (size_t)(keff + 1));
        int *hi = (int *)malloc(sizeof(int) * (size_t)(keff + 1));
#pragma omp for schedule(dynamic, 1)
        for (int64_t q = 0; q < nq; ++q) {
            const float *qp = Q + q * d;
            double qnorm = metric == 2 ? (double)qn[q] : 0.0;
            int size = 0;
            for (int64_t r = 0; r < n; ++r) {
                double dv = pair_f32(qp, X + r * d, d, metric, qnorm,
                                     metric == 2 ? (double)xn[r] : 0.0);
                if (size < keff) {
                    heap_push(hd, hi, size, dv, (int)r);
                    ++size;
                } else if (lex_gt(hd[0], hi[0], dv, (int)r)) {
                    hd[0] = dv;
                    hi[0] = (int)r;
                    heap_sift_down(hd, hi, size, 0);
                }
            }
            for (int j = size - 1; j >= 0; --j) {
                out_d[q * keff + j] = hd[0];
                out_i[q * keff + j] = hi[0];
                --size;
                hd[0] = hd[size];
                hi[0] = hi[size];
                heap_sift_down(hd, hi, size, 0);
            }
        }
        free(hd);
        free(hi);
    }
    return keff;
}
