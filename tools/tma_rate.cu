// tma_rate.cu -- microbenchmark: L2 -> shared memory streaming rate on B200.
//
// Every CTA (one per SM) streams 16 KiB tiles of an L2-resident buffer
// through an S-stage mbarrier ring (one thread issues, one thread consumes
// and releases), in three flavours:
//   tensor  : cp.async.bulk.tensor.2d, box 128 rows x 128 B, SWIZZLE_128B
//             (the filter kernel's database-tile load)
//   bulk    : cp.async.bulk (1-D, contiguous 16 KiB)
//   bulk4   : 4 x cp.async.bulk of 4 KiB
// Each CTA pair group of G CTAs may read the SAME tiles (G consumers per
// tile, like the query tiles sharing a row block) or distinct ones.
// Diagnostics only.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rate tma_rate.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(64, 1)
    tma_rate_kernel(const __grid_constant__ CUtensorMap tm, const int8_t *buf, int64_t n_tiles,
                    int iters, int stages, int group) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uintptr_t base = ((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023;
    unsigned char *ring = (unsigned char *)base;
    __shared__ uint64_t full[16], empty[16];
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // CTAs in the same group read the same tile sequence
    const int64_t start = (int64_t)(blockIdx.x / group) * 977;
    if (threadIdx.x == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            const int64_t tile = (start + i) % n_tiles;
            mbar_wait(empty + s, ph ^ 1);
            mbar_expect(full + s, 16384);
            unsigned char *dst = ring + (size_t)s * 16384;
            if (MODE == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
                    "l"((uint64_t)&tm), "r"(smem_u32(full + s)), "r"(0), "r"((int)(tile * 128))
                    : "memory");
            } else if (MODE == 1) {
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                    " [%0], [%1], 16384, [%2];" ::"r"(smem_u32(dst)),
                    "l"(buf + tile * 16384), "r"(smem_u32(full + s))
                    : "memory");
            } else {
                for (int j = 0; j < 4; ++j)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                        " [%0], [%1], 4096, [%2];" ::"r"(smem_u32(dst + j * 4096)),
                        "l"(buf + tile * 16384 + j * 4096), "r"(smem_u32(full + s))
                        : "memory");
            }
            if (++s == stages) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (threadIdx.x == 32) {
        int s = 0;
        uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            mbar_wait(full + s, ph);
            mbar_arrive(empty + s);
            if (++s == stages) {
                s = 0;
                ph ^= 1;
            }
        }
    }
    __syncthreads();
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t bytes = 64ll << 20;  // L2 resident
    const int64_t n_tiles = bytes / 16384;
    int8_t *buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, (cuuint64_t)(bytes / 128)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t estr[2] = {1, 1};
    ((PFN_cuTensorMapEncodeTiled_v12000)fn)(
        &tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int iters = 4000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[3] = {"tensor", "bulk", "bulk4"};
    for (int mode = 0; mode < 3; ++mode)
        for (int stages : {4, 8, 12})
            for (int group : {1, 8, 40}) {
                size_t smem = 1024 + (size_t)stages * 16384;
                auto k = mode == 0 ? tma_rate_kernel<0>
                                   : (mode == 1 ? tma_rate_kernel<1> : tma_rate_kernel<2>);
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                k<<<sms, 64, smem>>>(tm, buf, n_tiles, 200, stages, group);
                cudaEventRecord(e0);
                k<<<sms, 64, smem>>>(tm, buf, n_tiles, iters, stages, group);
                cudaEventRecord(e1);
                cudaError_t err = cudaDeviceSynchronize();
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                const double tb = (double)sms * iters * 16384 / (ms * 1e-3) / 1e12;
                printf("%-7s stages=%2d group=%2d  %6.2f TB/s  (%.1f B/clk/SM @1.965GHz)  %s\n",
                       names[mode], stages, group, tb, tb * 1e12 / sms / 1.965e9,
                       cudaGetErrorString(err));
            }
    return 0;
}
