// qa_gather.cu -- batched int8 distances to listed rows (sm_100a).
//
// The distance service a graph traversal needs: for every query q and every
// listed candidate id c = cand[q, j], the reference's pair score
// _pair_i(query q, row c) (_core.pyx:88-96), i.e. what HnswCore._dq computes
// one pair at a time for an external int8 query (_core.pyx:483-494) and
// _dist_rows for a stored one (472-481).  The traversal itself (visited
// sets, candidate heaps: _core.pyx:505-754) is host logic and not part of
// this library; a host-side beam search hands the neighbour lists of a whole
// query batch to this kernel per hop.
//
// HBM-bound gather: each pair reads one code row (ld bytes) at a random
// position.  Eight lanes share a pair (16 bytes = 16 codes per lane and 128-
// byte step: a 128-byte row is one coalesced 128-byte request), dp4a
// accumulation in int32, a 3-step shuffle reduction; the L2 distance uses the
// exact integer identity |x|^2 + |q|^2 - 2 x.q with the stored squared norms
// (equal to the reference's sum of squared differences whenever that does not
// wrap a C int).  Scores are float64 exactly as the reference forms them.
#include "qa_common.cuh"
#include "qa_internal.h"

namespace qa {

namespace {

constexpr int kLanesPerPair = 8;
constexpr int kPairsPerWarp = 32 / kLanesPerPair;

__global__ void __launch_bounds__(256) gather_scores_kernel(
    const int8_t *__restrict__ db, int64_t n, int64_t ldd, const int32_t *__restrict__ db_sqnorm,
    const float *__restrict__ db_norm, const int32_t *__restrict__ row_of_id,
    const int8_t *__restrict__ q, int64_t nq, int64_t ldq, const int32_t *__restrict__ q_sqnorm,
    const float *__restrict__ q_norm, const int32_t *__restrict__ cand, int64_t m, int64_t ldcand,
    int metric, double *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int sub = lane & (kLanesPerPair - 1);
    const int slot = lane / kLanesPerPair;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t groups_per_q = (m + kPairsPerWarp - 1) / kPairsPerWarp;
    const int64_t total = nq * groups_per_q;
    for (int64_t g = warp; g < total; g += nwarps) {
        const int64_t qi = g / groups_per_q;
        const int64_t j = (g - qi * groups_per_q) * kPairsPerWarp + slot;
        int32_t id = -1;
        if (j < m) id = __ldg(cand + qi * ldcand + j);
        const bool ok = id >= 0 && (int64_t)id < n;
        int64_t row = 0;
        if (ok) row = row_of_id ? (int64_t)__ldg(row_of_id + id) : (int64_t)id;
        const int8_t *xr = db + row * ldd;
        const int8_t *qr = q + qi * ldq;
        int32_t dot = 0;
        if (ok) {
            // rows are padded with zeros to ld (a multiple of 16 bytes)
            const int64_t kd = ldd < ldq ? ldd : ldq;
            for (int64_t c = (int64_t)sub * 16; c < kd; c += 16 * kLanesPerPair) {
                const int4 a = __ldg(reinterpret_cast<const int4 *>(xr + c));
                const int4 b = __ldg(reinterpret_cast<const int4 *>(qr + c));
                dot = __dp4a(a.x, b.x, dot);
                dot = __dp4a(a.y, b.y, dot);
                dot = __dp4a(a.z, b.z, dot);
                dot = __dp4a(a.w, b.w, dot);
            }
        }
#pragma unroll
        for (int o = kLanesPerPair / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        if (sub == 0 && j < m) {
            double s;
            if (!ok) {
                s = __longlong_as_double(0x7ff0000000000000ll);  // +inf: not a row
            } else if (metric == kIP) {
                s = -(double)dot;
            } else if (metric == kL2) {
                const int32_t l2 = (int32_t)((uint32_t)__ldg(db_sqnorm + row) +
                                             (uint32_t)__ldg(q_sqnorm + qi) - 2u * (uint32_t)dot);
                s = (double)l2;
            } else {
                s = angular_score(dot, __ldg(q_norm + qi), __ldg(db_norm + row));
            }
            out[qi * m + j] = s;
        }
    }
}

}  // namespace

cudaError_t launch_gather_scores(const int8_t *db, int64_t n, int64_t ldd,
                                 const int32_t *db_sqnorm, const float *db_norm,
                                 const int32_t *row_of_id, const int8_t *q, int64_t nq,
                                 int64_t ldq, const int32_t *q_sqnorm, const float *q_norm,
                                 const int32_t *cand, int64_t m, int64_t ldcand, int metric,
                                 double *out, cudaStream_t st) {
    if (nq == 0 || m == 0) return cudaSuccess;
    const int64_t groups = nq * ((m + kPairsPerWarp - 1) / kPairsPerWarp);
    int64_t blocks = (groups + 7) / 8;
    const int64_t cap = (int64_t)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    gather_scores_kernel<<<(unsigned)blocks, 256, 0, st>>>(db, n, ldd, db_sqnorm, db_norm,
                                                           row_of_id, q, nq, ldq, q_sqnorm, q_norm,
                                                           cand, m, ldcand, metric, out);
    return cudaGetLastError();
}

}  // namespace qa
