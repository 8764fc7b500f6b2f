// qa_select.cu -- exact top-k maintenance between filter passes, final
// score materialisation and the cross-shard merge.
//
// Reference semantics (_core.pyx:301-330): the result for a query is the
// first keff entries of the full (score, id) lexicographic sort.  The filter
// pass only discards rows that provably cannot enter that prefix; this file
// turns the surviving candidates into the exact prefix: exact float64 scores
// (angular: one correctly rounded division + subtraction, _core.pyx:96),
// lexicographic sort, truncation to k, and the next pass's threshold.
#include <cfloat>

#include "qa_common.cuh"
#include "qa_internal.h"

namespace qa {

namespace {

template <typename T, typename Less>
__device__ void block_bitonic_sort(T *buf, int P, Less less) {
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (P >> 1); t += blockDim.x) {
                int i = 2 * t - (t & (stride - 1));
                int j = i + stride;
                bool up = ((i & size) == 0);
                T a = buf[i], b = buf[j];
                bool swap = up ? less(b, a) : less(a, b);
                if (swap) {
                    buf[i] = b;
                    buf[j] = a;
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

struct EntryLess {
    __device__ bool operator()(const Entry &a, const Entry &b) const { return entry_less(a, b); }
};

template <int M>
__device__ __forceinline__ Entry make_entry(Cand c, int32_t qq, float qn,
                                            const int32_t *__restrict__ db_sqnorm,
                                            const float *__restrict__ db_norm) {
    Entry e;
    e.row = c.row;
    e.dot = c.dot;
    if constexpr (M == kIP) {
        e.skey = skey_from_int((int32_t)(0u - (uint32_t)c.dot));
    } else if constexpr (M == kL2) {
        uint32_t s = (uint32_t)qq + (uint32_t)__ldg(db_sqnorm + c.row) - 2u * (uint32_t)c.dot;
        e.skey = skey_from_int((int32_t)s);
    } else {
        e.skey = skey_from_double(angular_score(c.dot, qn, __ldg(db_norm + c.row)));
    }
    return e;
}

template <int M>
__device__ __forceinline__ int32_t threshold_of(const Entry &e, int32_t qq,
                                                const float *__restrict__ db_norm) {
    if constexpr (M == kIP) {
        return e.dot;  // candidate iff dot >= dot_k (ties may win on id)
    } else if constexpr (M == kL2) {
        int32_t s = (int32_t)((uint32_t)(e.skey & 0xffffffffull) ^ 0x80000000u);
        return (int32_t)((uint32_t)s - (uint32_t)qq);  // xx - 2dot <= l2_k - qq
    } else {
        // c_k = dot_k / xn_k; the float proxy float(dot)*rcp(xn) is within
        // 3 * 2^-24 relative of dot/xn, and rows that tie the k-th score
        // after float64 rounding differ from c_k by < 2^-51 relative; a
        // 2^-20 relative band (plus an absolute 2^-40) covers both.
        double c = __ddiv_rn((double)e.dot, (double)__ldg(db_norm + e.row));
        double p = c - fabs(c) * 0x1p-20 - 0x1p-40;
        return __float_as_int(__double2float_rd(p));
    }
}

template <int M>
__global__ void __launch_bounds__(256) select_kernel(SelectArgs a, int sz) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Entry *buf = reinterpret_cast<Entry *>(smem_raw);
    const int64_t q = blockIdx.x;
    if (q >= a.nq) return;
    const int32_t total_cands = a.ccount[q];
    if (total_cands == 0) return;  // nothing new: state and threshold unchanged
    const int m = (int)min((int64_t)total_cands, a.cap);
    if (total_cands > a.cap && threadIdx.x == 0) {
        a.overflow[q] = 1;
        atomicExch(a.any_overflow, 1);
    }
    const int32_t qq = (M == kL2) ? a.q_sqnorm[q] : 0;
    const float qn = (M == kAngular) ? a.q_norm[q] : 1.0f;
    Entry *st = a.state + q * a.k;
    const Cand *cd = a.cand + q * a.cap;
    int cur = a.state_cnt[q];
    for (int i = threadIdx.x; i < cur; i += blockDim.x) buf[i] = st[i];
    int pos = 0;
    while (pos < m) {
        const int take = min(m - pos, sz - cur);
        for (int i = threadIdx.x; i < take; i += blockDim.x)
            buf[cur + i] = make_entry<M>(cd[pos + i], qq, qn, a.db_sqnorm, a.db_norm);
        const int tot = cur + take;
        const int P = next_pow2(tot);
        for (int i = tot + threadIdx.x; i < P; i += blockDim.x) {
            buf[i].skey = ~0ull;
            buf[i].row = INT32_MAX;
            buf[i].dot = 0;
        }
        __syncthreads();
        block_bitonic_sort(buf, P, EntryLess());
        cur = (int)min((int64_t)tot, a.k);
        pos += take;
    }
    for (int i = threadIdx.x; i < cur; i += blockDim.x) st[i] = buf[i];
    if (threadIdx.x == 0) {
        a.state_cnt[q] = cur;
        if (cur == a.k) a.thr[q] = threshold_of<M>(buf[cur - 1], qq, a.db_norm);
    }
}

__global__ void reset_kernel(int32_t *p, int64_t n, int32_t v) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void init_state_kernel(int32_t *state_cnt, int32_t *thr, int64_t nq,
                                  int32_t pass_all) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nq) {
        state_cnt[i] = 0;
        thr[i] = pass_all;
    }
}

template <int M>
__global__ void finalize_kernel(const Entry *__restrict__ state, int64_t nq, int64_t k,
                                int64_t keff, const int32_t *__restrict__ db_sqnorm,
                                const float *__restrict__ db_norm,
                                const int32_t *__restrict__ q_sqnorm,
                                const float *__restrict__ q_norm, int64_t id_offset,
                                double *__restrict__ out_scores, int32_t *__restrict__ out_ids) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nq * keff) return;
    int64_t q = t / keff, j = t - q * keff;
    Entry e = state[q * k + j];
    double s;
    if constexpr (M == kIP) {
        s = -(double)e.dot;  // dot == 0 gives -0.0, exactly as _core.pyx:95
    } else if constexpr (M == kL2) {
        uint32_t v = (uint32_t)q_sqnorm[q] + (uint32_t)db_sqnorm[e.row] - 2u * (uint32_t)e.dot;
        s = (double)(int32_t)v;
    } else {
        s = angular_score(e.dot, q_norm[q], db_norm[e.row]);
    }
    out_scores[t] = s;
    out_ids[t] = (int32_t)(e.row + id_offset);
}

struct MEntry {
    unsigned long long skey;
    int32_t id;
    int32_t pad;
    double score;
};
struct MEntryLess {
    __device__ bool operator()(const MEntry &a, const MEntry &b) const {
        return a.skey < b.skey || (a.skey == b.skey && a.id < b.id);
    }
};

__global__ void __launch_bounds__(256) merge_kernel(const double *__restrict__ in_scores,
                                                    const int32_t *__restrict__ in_ids, int64_t G,
                                                    int64_t nq, int64_t kin, int64_t k,
                                                    double *__restrict__ out_scores,
                                                    int32_t *__restrict__ out_ids, int sz) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MEntry *buf = reinterpret_cast<MEntry *>(smem_raw);
    const int64_t q = blockIdx.x;
    if (q >= nq) return;
    int cur = 0;
    for (int64_t g = 0; g < G; ++g) {
        const double *sg = in_scores + (g * nq + q) * kin;
        const int32_t *ig = in_ids + (g * nq + q) * kin;
        int64_t pos = 0;
        while (pos < kin) {
            const int take = (int)min(kin - pos, (int64_t)(sz - cur));
            for (int i = threadIdx.x; i < take; i += blockDim.x) {
                MEntry e;
                e.score = sg[pos + i];
                e.skey = skey_from_double(e.score + 0.0);  // -0.0 ties +0.0 (float64 ==)
                e.id = ig[pos + i];
                e.pad = 0;
                buf[cur + i] = e;
            }
            const int tot = cur + take;
            const int P = next_pow2(tot);
            for (int i = tot + threadIdx.x; i < P; i += blockDim.x) {
                buf[i].skey = ~0ull;
                buf[i].id = INT32_MAX;
            }
            __syncthreads();
            block_bitonic_sort(buf, P, MEntryLess());
            cur = (int)min((int64_t)tot, k);
            pos += take;
        }
    }
    for (int i = threadIdx.x; i < cur; i += blockDim.x) {
        out_scores[q * k + i] = buf[i].score;
        out_ids[q * k + i] = buf[i].id;
    }
}

int pow2_at_least(int64_t v, int64_t cap) {
    int64_t p = 32;
    while (p < v && p < cap) p <<= 1;
    return (int)p;
}

}  // namespace

cudaError_t launch_select(const SelectArgs &a, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    const int sz = pow2_at_least(a.k + a.cap, kSortMax);
    const size_t smem = (size_t)sz * sizeof(Entry);
    cudaError_t e = cudaSuccess;
    switch (a.metric) {
        case kIP:
            e = cudaFuncSetAttribute(select_kernel<kIP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
            if (e == cudaSuccess) select_kernel<kIP><<<(unsigned)a.nq, 256, smem, st>>>(a, sz);
            break;
        case kL2:
            e = cudaFuncSetAttribute(select_kernel<kL2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem);
            if (e == cudaSuccess) select_kernel<kL2><<<(unsigned)a.nq, 256, smem, st>>>(a, sz);
            break;
        default:
            e = cudaFuncSetAttribute(select_kernel<kAngular>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e == cudaSuccess)
                select_kernel<kAngular><<<(unsigned)a.nq, 256, smem, st>>>(a, sz);
            break;
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_fill(int32_t *p, int64_t n, int32_t v, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    reset_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, n, v);
    return cudaGetLastError();
}

cudaError_t launch_init_state(int32_t *state_cnt, int32_t *thr, int64_t nq, int metric,
                              cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    int32_t pass = metric == kIP ? kThrPassIP
                                 : (metric == kL2 ? kThrPassL2 : (int32_t)kThrPassAngBits);
    init_state_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(state_cnt, thr, nq, pass);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const Entry *state, const int32_t *state_cnt, int64_t nq, int64_t k,
                            int64_t keff, int metric, const int32_t *db_sqnorm,
                            const float *db_norm, const int32_t *q_sqnorm, const float *q_norm,
                            int64_t id_offset, double *out_scores, int32_t *out_ids,
                            cudaStream_t st) {
    (void)state_cnt;
    int64_t total = nq * keff;
    if (total == 0) return cudaSuccess;
    unsigned grid = (unsigned)((total + 255) / 256);
    switch (metric) {
        case kIP:
            finalize_kernel<kIP><<<grid, 256, 0, st>>>(state, nq, k, keff, db_sqnorm, db_norm,
                                                       q_sqnorm, q_norm, id_offset, out_scores,
                                                       out_ids);
            break;
        case kL2:
            finalize_kernel<kL2><<<grid, 256, 0, st>>>(state, nq, k, keff, db_sqnorm, db_norm,
                                                       q_sqnorm, q_norm, id_offset, out_scores,
                                                       out_ids);
            break;
        default:
            finalize_kernel<kAngular><<<grid, 256, 0, st>>>(state, nq, k, keff, db_sqnorm,
                                                            db_norm, q_sqnorm, q_norm, id_offset,
                                                            out_scores, out_ids);
    }
    return cudaGetLastError();
}

cudaError_t launch_merge(const double *in_scores, const int32_t *in_ids, int64_t G, int64_t nq,
                         int64_t kin, int64_t k, double *out_scores, int32_t *out_ids,
                         cudaStream_t st) {
    if (nq == 0 || k == 0) return cudaSuccess;
    const int sz = pow2_at_least(k + kin, kSortMax);
    const size_t smem = (size_t)sz * sizeof(MEntry);
    cudaError_t e = cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    merge_kernel<<<(unsigned)nq, 256, smem, st>>>(in_scores, in_ids, G, nq, kin, k, out_scores,
                                                  out_ids, sz);
    return cudaGetLastError();
}

}  // namespace qa
