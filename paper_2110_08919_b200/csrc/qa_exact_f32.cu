// qa_exact_f32.cu -- float32 exhaustive search, bit-exact with the
// reference's _scan_f32 (the ground truth for recall).
//
// Reference arithmetic (_core.pyx:32-46, 75-84, 270-298):
//   dot  = sequential sum over j = 0..d-1 of (double)q[j] * (double)x[j],
//          accumulator starting at +0.0
//   l2   = sequential sum of t*t, t = (double)q[j] - (double)x[j]
//   score: IP -dot; L2 l2; ANGULAR 1.0 - dot / ((double)qn * (double)xn)
//   norms(float32 rows) = (float)sqrt(sequential sum of (double)x[j]^2)
// The product of two float32 values is exact in float64, so a DFMA on the
// dot path rounds exactly like the reference's multiply-then-add; the L2 path
// uses explicit __dsub_rn / __dmul_rn / __dadd_rn (no contraction).  Every
// pair is accumulated by ONE thread in the reference's j order, so each score
// is the reference's float64 value bit for bit; the top-k is the exact
// (score, id) lexicographic order.
//
// Shape of the work (B200: FP64 on the CUDA cores, ~64 DFMA/clk/SM):
//   scores kernel  CTA tile 64 queries x 128 rows, 256 threads, 4x8 float64
//                  accumulators per thread, float32 operands converted once
//                  while staged (double-buffered) into shared memory;
//   select kernel  one CTA per query: streams the round's scores in chunks of
//                  1024, keeps rows that beat the current k-th (score, id),
//                  and bitonic-sorts state + survivors in shared memory.
// The orchestration (rounds of kF32Rows rows, query chunks) is in qa_api.cu.
#include <cstdint>
#include <cub/device/device_segmented_radix_sort.cuh>
#include <cuda_runtime.h>

#include "qa_common.cuh"
#include "qa_internal.h"

namespace qa {

namespace {

constexpr int kFQ = 64;    // queries per CTA tile
constexpr int kFR = 128;   // rows per CTA tile
constexpr int kFK = 16;    // dimensions per shared-memory stage
constexpr int kFT = 256;   // threads

template <int M>
__global__ void __launch_bounds__(kFT, 2)
f32_scores_kernel(const float *__restrict__ db, int64_t ldd, const float *__restrict__ q,
                  int64_t ldq, int d, int nq, int64_t r_lo, int rows,
                  const float *__restrict__ db_norm, const float *__restrict__ q_norm,
                  double *__restrict__ out, int64_t ldo) {
    extern __shared__ __align__(16) double fsm[];
    double *Qs = fsm;                         // [2][kFK][kFQ]
    double *Xs = fsm + 2 * kFK * kFQ;         // [2][kFK][kFR]
    const int tid = threadIdx.x;
    const int tq = tid >> 4, tr = tid & 15;   // 16 x 16 thread grid
    const int q0 = blockIdx.y * kFQ;
    const int rt0 = blockIdx.x * kFR;         // tile start within the round
    const int64_t row0 = r_lo + rt0;

    // staging assignment: X 128 rows x 16 dims = 8 floats per thread,
    // Q 64 x 16 = 4 per thread
    const int xr = tid >> 1, xj = (tid & 1) * 8;
    const int qr = tid >> 2, qj = (tid & 3) * 4;
    const bool xrow_ok = rt0 + xr < rows;
    const bool qrow_ok = q0 + qr < nq;
    const float *xp = db + (row0 + xr) * ldd;
    const float *qp = q + (int64_t)(q0 + qr) * ldq;

    float xv[8], qv[4];
    auto load = [&](int j0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int j = j0 + xj + i;
            xv[i] = (xrow_ok && j < d) ? __ldg(xp + j) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int j = j0 + qj + i;
            qv[i] = (qrow_ok && j < d) ? __ldg(qp + j) : 0.f;
        }
    };
    auto store = [&](int buf) {
        double *xs = Xs + buf * kFK * kFR;
        double *qs = Qs + buf * kFK * kFQ;
#pragma unroll
        for (int i = 0; i < 8; ++i) xs[(xj + i) * kFR + xr] = (double)xv[i];
#pragma unroll
        for (int i = 0; i < 4; ++i) qs[(qj + i) * kFQ + qr] = (double)qv[i];
    };

    double acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int l = 0; l < 8; ++l) acc[i][l] = 0.0;

    const int nchunks = (d + kFK - 1) / kFK;
    load(0);
    store(0);
    __syncthreads();
    for (int c = 0; c < nchunks; ++c) {
        const int buf = c & 1;
        if (c + 1 < nchunks) load((c + 1) * kFK);
        const double *xs = Xs + buf * kFK * kFR;
        const double *qs = Qs + buf * kFK * kFQ;
        // zero-padded dimensions past d add +0 (dot) or 0*0 (l2): the
        // accumulator never holds -0.0, so they leave it unchanged
#pragma unroll
        for (int j = 0; j < kFK; ++j) {
            double a[4], b[8];
            const double2 a01 = *reinterpret_cast<const double2 *>(qs + j * kFQ + tq * 4);
            const double2 a23 = *reinterpret_cast<const double2 *>(qs + j * kFQ + tq * 4 + 2);
            a[0] = a01.x; a[1] = a01.y; a[2] = a23.x; a[3] = a23.y;
#pragma unroll
            for (int l = 0; l < 8; ++l) b[l] = xs[j * kFR + tr + 16 * l];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int l = 0; l < 8; ++l) {
                    if constexpr (M == kL2) {
                        const double t = __dsub_rn(a[i], b[l]);
                        acc[i][l] = __dadd_rn(acc[i][l], __dmul_rn(t, t));
                    } else {
                        acc[i][l] = __fma_rn(a[i], b[l], acc[i][l]);
                    }
                }
        }
        if (c + 1 < nchunks) {
            store(buf ^ 1);
        }
        __syncthreads();
    }

#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int qq = q0 + tq * 4 + i;
        if (qq >= nq) continue;
        double qn = 0.0;
        if constexpr (M == kAngular) qn = (double)q_norm[qq];
#pragma unroll
        for (int l = 0; l < 8; ++l) {
            const int r = rt0 + tr + 16 * l;
            if (r >= rows) continue;
            double s;
            if constexpr (M == kIP) {
                s = -acc[i][l];
            } else if constexpr (M == kL2) {
                s = acc[i][l];
            } else {
                const double den = __dmul_rn(qn, (double)db_norm[r_lo + r]);
                s = __dsub_rn(1.0, __ddiv_rn(acc[i][l], den));
            }
            out[(int64_t)qq * ldo + r] = s;
        }
    }
}

__device__ __forceinline__ bool lex_gt(double as, int ai, double bs, int bi) {
    return as > bs || (as == bs && ai > bi);
}

constexpr int kSelChunk = 1024;

// Merge one round's scores [rows] into each query's sorted (score, id) state.
__global__ void __launch_bounds__(512)
f32_select_kernel(const double *__restrict__ scores, int64_t lds, int rows, int64_t id0,
                  double *__restrict__ st_s, int32_t *__restrict__ st_i,
                  int32_t *__restrict__ st_n, int k, int sortn) {
    extern __shared__ __align__(16) unsigned char ssm[];
    double *ks = reinterpret_cast<double *>(ssm);
    int32_t *ki = reinterpret_cast<int32_t *>(ks + sortn);
    __shared__ int cnt;
    __shared__ double thr_s;
    __shared__ int thr_i;
    const int qi = blockIdx.x;
    const int tid = threadIdx.x, nt = blockDim.x;
    int cur = st_n[qi];
    for (int i = tid; i < cur; i += nt) {
        ks[i] = st_s[(int64_t)qi * k + i];
        ki[i] = st_i[(int64_t)qi * k + i];
    }
    if (tid == 0) {
        cnt = 0;
        if (cur == k) {
            thr_s = st_s[(int64_t)qi * k + k - 1];
            thr_i = st_i[(int64_t)qi * k + k - 1];
        }
    }
    __syncthreads();
    const double *sp = scores + (int64_t)qi * lds;
    for (int c0 = 0; c0 < rows; c0 += kSelChunk) {
        const int m = min(kSelChunk, rows - c0);
        const bool full = cur == k;
        const double ts = thr_s;
        const int ti = thr_i;
        for (int r = tid; r < m; r += nt) {
            const double s = sp[c0 + r];
            const int id = (int)(id0 + c0 + r);
            if (!full || lex_gt(ts, ti, s, id)) {
                const int p = atomicAdd(&cnt, 1);
                ks[cur + p] = s;
                ki[cur + p] = id;
            }
        }
        __syncthreads();
        const int added = cnt;
        __syncthreads();   // everyone has read cnt before the next chunk appends
        if (added == 0) continue;
        const int total = cur + added;
        int P = 1;
        while (P < total) P <<= 1;
        for (int i = total + tid; i < P; i += nt) {
            ks[i] = __longlong_as_double(0x7ff0000000000000ll);  // +inf
            ki[i] = INT32_MAX;
        }
        __syncthreads();
        for (int size = 2; size <= P; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int t = tid; t < (P >> 1); t += nt) {
                    const int i = 2 * t - (t & (stride - 1));
                    const int j = i + stride;
                    const bool up = (i & size) == 0;
                    const double si = ks[i], sj = ks[j];
                    const int ii = ki[i], ij = ki[j];
                    if (lex_gt(si, ii, sj, ij) == up) {
                        ks[i] = sj; ks[j] = si;
                        ki[i] = ij; ki[j] = ii;
                    }
                }
                __syncthreads();
            }
        }
        cur = total < k ? total : k;
        if (tid == 0) {
            cnt = 0;
            if (cur == k) {
                thr_s = ks[k - 1];
                thr_i = ki[k - 1];
            }
        }
        __syncthreads();
    }
    for (int i = tid; i < cur; i += nt) {
        st_s[(int64_t)qi * k + i] = ks[i];
        st_i[(int64_t)qi * k + i] = ki[i];
    }
    if (tid == 0) st_n[qi] = cur;
}

__global__ void f32_finalize_kernel(const double *__restrict__ st_s, const int32_t *__restrict__ st_i,
                                    int64_t nq, int k, int64_t id_offset,
                                    double *__restrict__ out_s, int32_t *__restrict__ out_i) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nq * k) return;
    out_s[t] = st_s[t];
    out_i[t] = (int32_t)(st_i[t] + id_offset);
}

// Any k (keff beyond the shared-memory select): every score of a query
// chunk, sorted per query by (score, id) with a stable segmented radix sort.
// Keys are order-preserving u64 maps of score + 0.0 (so -0.0 ties +0.0, the
// reference's double compare), values the row ids in ascending order -- the
// stable sort keeps ties in id order.
__global__ void fullsort_keys_kernel(const double *__restrict__ scores, int64_t total, int64_t n,
                                     unsigned long long *__restrict__ keys,
                                     int32_t *__restrict__ vals) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    keys[t] = skey_from_double(scores[t] + 0.0);
    vals[t] = (int32_t)(t % n);
}

__global__ void fullsort_out_kernel(const double *__restrict__ scores,
                                    const int32_t *__restrict__ vals, int64_t m, int64_t n,
                                    int64_t keff, int64_t id_offset, double *__restrict__ out_s,
                                    int32_t *__restrict__ out_i) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m * keff) return;
    const int64_t q = t / keff, j = t - q * keff;
    const int32_t id = vals[q * n + j];
    out_s[t] = scores[q * n + id];  // the score itself (keeps -0.0)
    out_i[t] = (int32_t)(id + id_offset);
}

__global__ void fullsort_offsets_kernel(int64_t m, int64_t n, int64_t *__restrict__ off) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t <= m) off[t] = t * n;
}

// (float)sqrt(sequential float64 sum of x^2), one thread per row
__global__ void norms_f32_kernel(const float *__restrict__ x, int64_t n, int64_t d, int64_t ldx,
                                 float *__restrict__ out) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const float *p = x + r * ldx;
    double acc = 0.0;
    for (int64_t j = 0; j < d; ++j) {
        const double v = (double)__ldg(p + j);
        acc = __fma_rn(v, v, acc);
    }
    out[r] = __double2float_rn(__dsqrt_rn(acc));
}

}  // namespace

size_t f32_select_smem(int64_t k) {
    int64_t P = 1;
    while (P < k + kSelChunk) P <<= 1;
    return (size_t)P * 12;
}

cudaError_t launch_f32_scores(const float *db, int64_t ldd, const float *q, int64_t ldq, int64_t d,
                              int64_t nq, int64_t r_lo, int64_t rows, int metric,
                              const float *db_norm, const float *q_norm, double *out, int64_t ldo,
                              cudaStream_t st) {
    if (rows <= 0 || nq <= 0) return cudaSuccess;
    const size_t smem = (size_t)2 * kFK * (kFQ + kFR) * sizeof(double);
    dim3 grid((unsigned)((rows + kFR - 1) / kFR), (unsigned)((nq + kFQ - 1) / kFQ));
    if (grid.y > 65535) return cudaErrorNotSupported;
    auto go = [&](auto kern) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        kern<<<grid, kFT, smem, st>>>(db, ldd, q, ldq, (int)d, (int)nq, r_lo, (int)rows, db_norm,
                                      q_norm, out, ldo);
        return cudaGetLastError();
    };
    if (metric == kIP) return go(f32_scores_kernel<kIP>);
    if (metric == kL2) return go(f32_scores_kernel<kL2>);
    return go(f32_scores_kernel<kAngular>);
}

cudaError_t launch_f32_select(const double *scores, int64_t lds, int64_t rows, int64_t id0,
                              double *st_s, int32_t *st_i, int32_t *st_n, int64_t nq, int64_t k,
                              cudaStream_t st) {
    if (rows <= 0 || nq <= 0) return cudaSuccess;
    const size_t smem = f32_select_smem(k);
    int64_t P = (int64_t)(smem / 12);
    cudaError_t e = cudaFuncSetAttribute(f32_select_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    f32_select_kernel<<<(unsigned)nq, 512, smem, st>>>(scores, lds, (int)rows, id0, st_s, st_i,
                                                       st_n, (int)k, (int)P);
    return cudaGetLastError();
}

cudaError_t launch_f32_finalize(const double *st_s, const int32_t *st_i, int64_t nq, int64_t k,
                                int64_t id_offset, double *out_s, int32_t *out_i,
                                cudaStream_t st) {
    const int64_t m = nq * k;
    if (m <= 0) return cudaSuccess;
    f32_finalize_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(st_s, st_i, nq, (int)k,
                                                                      id_offset, out_s, out_i);
    return cudaGetLastError();
}

cudaError_t launch_norms_f32(const float *x, int64_t n, int64_t d, int64_t ldx, float *out,
                             cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    norms_f32_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(x, n, d, ldx, out);
    return cudaGetLastError();
}

}  // namespace qa

namespace qa {

size_t f32_fullsort_bytes(int64_t m, int64_t n) {
    // scores (8) + keys in/out (16) + values in/out (8) per (query, row),
    // offsets, and CUB's temporary storage
    size_t temp = 0;
    const int64_t total = m * n;
    cub::DeviceSegmentedRadixSort::SortPairs(nullptr, temp, (unsigned long long *)nullptr,
                                             (unsigned long long *)nullptr, (int32_t *)nullptr,
                                             (int32_t *)nullptr, total, (int)m,
                                             (int64_t *)nullptr, (int64_t *)nullptr);
    return (size_t)total * 32 + (size_t)(m + 1) * 8 + temp + 1024;
}

cudaError_t launch_f32_fullsort(const float *db, int64_t ldd, const float *q, int64_t ldq,
                                int64_t d, int64_t m, int64_t n, int metric, const float *db_norm,
                                const float *q_norm, int64_t keff, int64_t id_offset,
                                double *out_s, int32_t *out_i, void *scratch, size_t bytes,
                                cudaStream_t st) {
    if (m == 0 || n == 0 || keff == 0) return cudaSuccess;
    if (bytes < f32_fullsort_bytes(m, n)) return cudaErrorInvalidValue;
    const int64_t total = m * n;
    char *p = (char *)scratch;
    auto take = [&](size_t b) {
        char *r = p;
        p += (b + 255) / 256 * 256;
        return r;
    };
    double *sc = (double *)take((size_t)total * 8);
    unsigned long long *k_in = (unsigned long long *)take((size_t)total * 8);
    unsigned long long *k_out = (unsigned long long *)take((size_t)total * 8);
    int32_t *v_in = (int32_t *)take((size_t)total * 4);
    int32_t *v_out = (int32_t *)take((size_t)total * 4);
    int64_t *off = (int64_t *)take((size_t)(m + 1) * 8);
    size_t temp = (size_t)((char *)scratch + bytes - p);
    cudaError_t e = launch_f32_scores(db, ldd, q, ldq, d, m, 0, n, metric, db_norm, q_norm, sc, n, st);
    if (e != cudaSuccess) return e;
    fullsort_keys_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(sc, total, n, k_in, v_in);
    fullsort_offsets_kernel<<<(unsigned)((m + 256) / 256), 256, 0, st>>>(m, n, off);
    e = cub::DeviceSegmentedRadixSort::SortPairs(p, temp, k_in, k_out, v_in, v_out, total, (int)m,
                                                 off, off + 1, 0, 64, st);
    if (e != cudaSuccess) return e;
    fullsort_out_kernel<<<(unsigned)((m * keff + 255) / 256), 256, 0, st>>>(sc, v_out, m, n, keff,
                                                                          id_offset, out_s, out_i);
    return cudaGetLastError();
}

}  // namespace qa
