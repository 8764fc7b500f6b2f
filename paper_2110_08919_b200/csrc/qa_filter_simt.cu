// qa_filter_simt.cu -- CUDA-core (dp4a) filter pass.
//
// The bring-up implementation of one filter pass: every (row, query) dot is
// computed with __dp4a on int32 words, tested against the query's threshold
// (qa_common.cuh passes<>) and appended to the query's candidate list.  It is
// kept as an independent cross-check of the tensor-core pass
// (qa_debug_dots_i8 compares both) and serves tiny shapes where a 128-row
// MMA tile would be mostly padding.
#include "qa_common.cuh"
#include "qa_internal.h"

namespace qa {

namespace {

constexpr int kRows = 128;   // rows per block (one per thread)
constexpr int kQTile = 16;   // queries staged in shared memory per block

template <int M>
__global__ void __launch_bounds__(kRows) filter_simt_kernel(FilterArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int32_t *qs = reinterpret_cast<int32_t *>(smem_raw);  // [kQTile][kdim/4]
    const int64_t words = a.kdim / 4;
    const int64_t q0 = (int64_t)blockIdx.y * kQTile;
    const int nqt = (int)min((int64_t)kQTile, a.nq - q0);
    for (int64_t i = threadIdx.x; i < (int64_t)nqt * words; i += blockDim.x) {
        int64_t qi = i / words, w = i - qi * words;
        qs[i] = *reinterpret_cast<const int32_t *>(a.q + (q0 + qi) * a.ldq + 4 * w);
    }
    __syncthreads();
    const int64_t row = a.r_lo + (int64_t)blockIdx.x * kRows + threadIdx.x;
    if (row >= a.r_hi) return;
    const int32_t *xr = reinterpret_cast<const int32_t *>(a.db + row * a.ldd);
    int32_t xx = 0;
    float inv_xn = 0.f;
    if constexpr (M == kL2) xx = __ldg(a.db_sqnorm + row);
    if constexpr (M == kAngular) inv_xn = __frcp_rn(__ldg(a.db_norm + row));
    for (int qi = 0; qi < nqt; ++qi) {
        const int32_t *qw = qs + qi * words;
        int32_t acc = 0;
        for (int64_t w = 0; w < words; ++w) acc = __dp4a(__ldg(xr + w), qw[w], acc);
        const int64_t q = q0 + qi;
        if (a.mode == 2) {
            a.dots_out[q * a.ld_dots + row] = acc;
            continue;
        }
        if (a.mode == 1) {
            a.cand[q * a.cap + (row - a.r_lo)] = Cand{(int32_t)row, acc};
            continue;
        }
        if (a.mode == 3) {  // masked dense: slot per row, row = -1 when filtered out
            a.cand[q * a.cap + (row - a.r_lo)] =
                passes<M>(acc, __ldg(a.thr + q), xx, inv_xn) ? Cand{(int32_t)row, acc} : Cand{-1, 0};
            continue;
        }
        if (passes<M>(acc, __ldg(a.thr + q), xx, inv_xn)) {
            int32_t slot = atomicAdd(a.ccount + q, 1);
            if (slot < a.cap) a.cand[q * a.cap + slot] = Cand{(int32_t)row, acc};
        }
    }
}

}  // namespace

cudaError_t launch_filter_simt(const FilterArgs &a, cudaStream_t st) {
    if (a.r_hi <= a.r_lo || a.nq == 0) return cudaSuccess;
    dim3 grid((unsigned)((a.r_hi - a.r_lo + kRows - 1) / kRows),
              (unsigned)((a.nq + kQTile - 1) / kQTile));
    size_t smem = (size_t)kQTile * a.kdim;
    if (smem > 200 * 1024) return cudaErrorNotSupported;
    cudaError_t e = cudaSuccess;
    switch (a.metric) {
        case kIP:
            e = cudaFuncSetAttribute(filter_simt_kernel<kIP>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e == cudaSuccess) filter_simt_kernel<kIP><<<grid, kRows, smem, st>>>(a);
            break;
        case kL2:
            e = cudaFuncSetAttribute(filter_simt_kernel<kL2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e == cudaSuccess) filter_simt_kernel<kL2><<<grid, kRows, smem, st>>>(a);
            break;
        default:
            e = cudaFuncSetAttribute(filter_simt_kernel<kAngular>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e == cudaSuccess) filter_simt_kernel<kAngular><<<grid, kRows, smem, st>>>(a);
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace qa
