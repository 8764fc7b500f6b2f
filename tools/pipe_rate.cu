// pipe_rate.cu -- microbenchmark: MMA -> epilogue handshake over a
// double-buffered TMEM accumulator (no TMA: operands static in smem).
//
// One thread issues 5 x (M=128, N=256, K=32) i8 MMAs per tile into
// accumulator acc = tile % 2 and commits acc_full[acc]; 16 epilogue warps
// wait acc_full, tcgen05.ld their 64 columns, and arrive acc_empty[acc];
// the MMA thread waits acc_empty before reusing a buffer.  Variants:
//   wait mode 0: try_wait with suspend hint, 1: try_wait spin
//   ld: 0 = no TMEM load, 1 = 2 x .x32 loads
// Reports cycles per tile (ideal = 5 x 128 = 640).  Diagnostics only.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rate pipe_rate.cu -lcuda
//
// With stages > 0 the A operand streams through a TMA ring (box 128 rows x
// 128 B, SWIZZLE_128B, from an L2-resident buffer) as in the filter kernel.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t make_desc128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_hint(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 20000;\n\t@!p bra W_%=;\n\t}" ::"r"(
            smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__global__ void __launch_bounds__(576, 1) pipe_rate_kernel(const __grid_constant__ CUtensorMap tm,
                                                            int n_src_tiles, int stages,
                                                            int tiles, int wait_mode, int do_ld,
                                                            long long *cycles, int *sink) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uintptr_t base = ((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023;
    unsigned char *sA = (unsigned char *)base;
    unsigned char *sB = sA + 128 * 128;
    unsigned char *sR = sB + 256 * 128;  // A ring
    __shared__ uint64_t acc_full[2], acc_empty[2], a_full[16], a_empty[16];
    __shared__ uint32_t tmem_base_s;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x)
        reinterpret_cast<int32_t *>(sA)[i] = 0x01010101;
    if (threadIdx.x == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&acc_full[s], 1);
            mbar_init(&acc_empty[s], 16);
        }
        for (int s = 0; s < 16; ++s) {
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_u32(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_s;
    if (warp == 16) {
        if (lane == 0) {
            const uint32_t idesc =
                (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | (8u << 24);
            const uint64_t ad0 = make_desc128(smem_u32(sA)), bd = make_desc128(smem_u32(sB));
            const uint64_t rd0 = make_desc128(smem_u32(sR));
            long long t0 = clock64();
            int stage = 0;
            uint32_t aph = 0;
            for (int t = 0; t < tiles; ++t) {
                const int acc = t & 1;
                const uint32_t ph = ((t >> 1) & 1) ^ 1;
                while (!mbar_try(&acc_empty[acc], ph)) {
                }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                uint64_t ad = ad0;
                if (stages > 0) {
                    while (!mbar_try(&a_full[stage], aph)) {
                    }
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    ad = rd0 + (uint64_t)((stage * 16384) >> 4);
                }
                const uint32_t d = tmem + (uint32_t)(acc * 256);
#pragma unroll
                for (int kk = 0; kk < 5; ++kk)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(ad + (uint64_t)(2 * (kk & 3))), "l"(bd + (uint64_t)(2 * (kk & 3))),
                        "r"(idesc), "r"(kk)
                        : "memory");
                if (stages > 0) {
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                            smem_u32(&a_empty[stage]))
                        : "memory");
                    if (++stage == stages) {
                        stage = 0;
                        aph ^= 1;
                    }
                }
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        smem_u32(&acc_full[acc]))
                    : "memory");
            }
            long long t1 = clock64();
            cycles[blockIdx.x] = t1 - t0;
        }
    } else if (warp == 17) {
        if (lane == 0 && stages > 0) {
            int stage = 0;
            uint32_t aph = 0;
            for (int t = 0; t < tiles; ++t) {
                while (!mbar_try(&a_empty[stage], aph ^ 1)) {
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16384;" ::"r"(
                                 smem_u32(&a_full[stage]))
                             : "memory");
                const int row0 = (int)(((long long)blockIdx.x * 977 + t) % n_src_tiles) * 128;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(sR + stage * 16384)),
                    "l"((uint64_t)&tm), "r"(smem_u32(&a_full[stage])), "r"(0), "r"(row0)
                    : "memory");
                if (++stage == stages) {
                    stage = 0;
                    aph ^= 1;
                }
            }
        }
    } else {
        const int quarter = warp & 3;
        const int col0 = (warp >> 2) * 64;
        int x = 0;
        for (int t = 0; t < tiles; ++t) {
            const int acc = t & 1;
            const uint32_t ph = (t >> 1) & 1;
            if (wait_mode == 0)
                mbar_wait_hint(&acc_full[acc], ph);
            else
                while (!mbar_try(&acc_full[acc], ph)) {
                }
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (do_ld) {
                const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * 256 + col0);
                uint32_t v[2][32];
#pragma unroll
                for (int l = 0; l < 2; ++l)
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32"
                        " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15,"
                        " %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31},"
                        " [%32];"
                        : "=r"(v[l][0]), "=r"(v[l][1]), "=r"(v[l][2]), "=r"(v[l][3]), "=r"(v[l][4]),
                          "=r"(v[l][5]), "=r"(v[l][6]), "=r"(v[l][7]), "=r"(v[l][8]), "=r"(v[l][9]),
                          "=r"(v[l][10]), "=r"(v[l][11]), "=r"(v[l][12]), "=r"(v[l][13]),
                          "=r"(v[l][14]), "=r"(v[l][15]), "=r"(v[l][16]), "=r"(v[l][17]),
                          "=r"(v[l][18]), "=r"(v[l][19]), "=r"(v[l][20]), "=r"(v[l][21]),
                          "=r"(v[l][22]), "=r"(v[l][23]), "=r"(v[l][24]), "=r"(v[l][25]),
                          "=r"(v[l][26]), "=r"(v[l][27]), "=r"(v[l][28]), "=r"(v[l][29]),
                          "=r"(v[l][30]), "=r"(v[l][31])
                        : "r"(ta + (uint32_t)(32 * l))
                        : "memory");
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int l = 0; l < 2; ++l)
#pragma unroll
                    for (int j = 0; j < 32; ++j) x &= (int)v[l][j];
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&acc_empty[acc]))
                             : "memory");
        }
        if (x == 0x1234567) sink[0] = x;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long *d;
    int *sink;
    cudaMalloc(&d, sms * sizeof(long long));
    cudaMalloc(&sink, 4);
    const size_t smem = 1024 + (128 + 256) * 128 + 8 * 16384;
    cudaFuncSetAttribute(pipe_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const long long bytes = 64ll << 20;
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
    const int n_src_tiles = (int)(bytes / 16384);
    for (int stages : {0, 4, 8})
    for (int do_ld = 0; do_ld < 2; ++do_ld)
        for (int wm = 0; wm < 2; ++wm) {
            const int tiles = 4000;
            pipe_rate_kernel<<<sms, 576, smem>>>(tm, n_src_tiles, stages, 16, wm, do_ld, d, sink);
            pipe_rate_kernel<<<sms, 576, smem>>>(tm, n_src_tiles, stages, tiles, wm, do_ld, d, sink);
            cudaError_t err = cudaDeviceSynchronize();
            long long h[1024];
            cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < sms; ++i) avg += (double)h[i];
            avg /= sms;
            printf("stages=%d ld=%d wait=%s: %.1f cycles/tile (ideal 640)  (%s)\n", stages, do_ld,
                   wm == 0 ? "hint" : "spin", avg / tiles, cudaGetErrorString(err));
        }
    return 0;
}
