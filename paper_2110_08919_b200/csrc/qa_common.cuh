// qa_common.cuh -- shared device helpers for the int8 exhaustive k-NN path.
//
// Ordering contract (reference _core.pyx:164-173): results are ascending by
// (score, id), score compared as float64, ties broken by the smaller id.
// Scores per metric (_core.pyx:88-96):
//   INNER_PRODUCT  score = -(double)dot
//   L2_SQUARED     score = (double)l2          (int32 accumulation)
//   ANGULAR        score = 1.0 - (double)dot / ((double)qn * (double)xn)
#pragma once

#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

namespace qa {

enum Metric : int { kIP = 0, kL2 = 1, kAngular = 2 };

// Candidate produced by a filter pass: stored database row and the exact
// int32 dot product with the query.
struct Cand {
    int32_t row;
    int32_t dot;
};

// One retained neighbour: order key, reported id (the row's position in the
// caller's corpus -- differs from the stored row when the index keeps its
// rows sorted by norm), stored row.  skey orders exactly like the float64
// score; ties are resolved by id, the reference's rule.
struct Entry {
    unsigned long long skey;
    int32_t id;
    int32_t row;
};

// Order-preserving map of an int32 score to an unsigned key.
__host__ __device__ __forceinline__ unsigned long long skey_from_int(int32_t s) {
    return (unsigned long long)((uint32_t)s ^ 0x80000000u);
}

// Order-preserving map of a float64 score (never NaN, never -0.0 here).
__host__ __device__ __forceinline__ unsigned long long skey_from_double(double s) {
#ifdef __CUDA_ARCH__
    long long b = __double_as_longlong(s);
#else
    long long b;
    memcpy(&b, &s, 8);
#endif
    return b < 0 ? ~(unsigned long long)b : ((unsigned long long)b | 0x8000000000000000ull);
}

// Inverses of the maps above.
__host__ __device__ __forceinline__ int32_t int_from_skey(unsigned long long k) {
    return (int32_t)((uint32_t)k ^ 0x80000000u);
}
__device__ __forceinline__ double double_from_skey(unsigned long long k) {
    long long b = (k & 0x8000000000000000ull) ? (long long)(k & 0x7fffffffffffffffull)
                                              : (long long)~k;
    return __longlong_as_double(b);
}

__device__ __forceinline__ double angular_score(int32_t dot, float qn, float xn) {
    // qn*xn is exact in float64 (24+24 significant bits); one correctly
    // rounded division and one correctly rounded subtraction, exactly as
    // _core.pyx:96.  Explicit _rn intrinsics forbid FMA contraction.
    double den = __dmul_rn((double)qn, (double)xn);
    return __dsub_rn(1.0, __ddiv_rn((double)dot, den));
}

__device__ __forceinline__ bool entry_less(const Entry &a, const Entry &b) {
    return a.skey < b.skey || (a.skey == b.skey && a.id < b.id);
}

// Filter thresholds (one 32-bit word per query, meaning depends on metric):
//   IP       int32 D : candidate iff dot >= D
//   L2       int32 T : candidate iff xx - 2*dot <= T      (T = l2_k - qq)
//   ANGULAR  float P : candidate iff float(dot) * inv_xn >= P
// The "pass everything" values:
constexpr int32_t kThrPassIP = INT32_MIN;
constexpr int32_t kThrPassL2 = INT32_MAX;
// angular pass-all is -inf (bit pattern 0xff800000)
constexpr uint32_t kThrPassAngBits = 0xff800000u;

template <int M>
__device__ __forceinline__ bool passes(int32_t dot, int32_t thr, int32_t xx, float inv_xn) {
    if constexpr (M == kIP) {
        return dot >= thr;
    } else if constexpr (M == kL2) {
        return xx - 2 * dot <= thr;
    } else {
        float p = __fmul_rn(__int2float_rn(dot), inv_xn);
        return p >= __int_as_float(thr);
    }
}

}  // namespace qa
