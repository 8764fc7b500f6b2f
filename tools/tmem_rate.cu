// tmem_rate.cu -- microbenchmark: tcgen05.ld (TMEM -> registers) throughput.
//
// W warps per CTA (one CTA per SM), each repeatedly loading C columns of its
// 32-lane TMEM quarter with 32x32b.x32 loads; optionally while one thread
// keeps the tensor core busy with M=128 N=256 K=32 i8 MMAs into the other
// half of TMEM.  Reports bytes/clk/SM.  Diagnostics only.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_rate tmem_rate.cu
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

template <int NLD>  // x32 loads per iteration per warp
__global__ void __launch_bounds__(544, 1) tmem_rate_kernel(int iters, int with_mma,
                                                            long long *cycles, int *sink) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uintptr_t base = ((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023;
    unsigned char *sA = (unsigned char *)base;
    unsigned char *sB = sA + 128 * 128;
    __shared__ uint32_t tmem_base_s;
    __shared__ int done_warps;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x)
        reinterpret_cast<int32_t *>(sA)[i] = 0x01010101;
    if (threadIdx.x == 0) done_warps = 0;
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
        // MMA issuer into columns [256, 512)
        if (lane == 0 && with_mma) {
            const uint32_t idesc =
                (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | (8u << 24);
            const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
            long long m0 = clock64(), nm = 0;
            while (*(volatile int *)&done_warps < 16) {
                nm += 256;
                for (int r = 0; r < 64; ++r)
                    for (int kk = 0; kk < 4; ++kk)
                        asm volatile(
                            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(
                                tmem + 256u),
                            "l"(make_desc128(a0 + kk * 32)), "l"(make_desc128(b0 + kk * 32)),
                            "r"(idesc), "r"(kk)
                            : "memory");
            }
            if (blockIdx.x == 0) printf("  MMA stream during loads: %.1f cycles per M128N256K32 MMA\n", (double)(clock64() - m0) / nm);
        }
    } else {
        const int quarter = warp & 3;
        const int col0 = (warp >> 2) * 64;  // 4 column groups of 64 in [0, 256)
        const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)col0;
        int acc = 0;
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            uint32_t v[NLD][32];
#pragma unroll
            for (int l = 0; l < NLD; ++l)
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
                    : "r"(ta + (uint32_t)(32 * (l & 1)))
                    : "memory");
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int l = 0; l < NLD; ++l)
#pragma unroll
                for (int j = 0; j < 32; ++j) acc ^= (int)v[l][j];
        }
        long long t1 = clock64();
        if (lane == 0) {
            cycles[blockIdx.x * 16 + warp] = t1 - t0;
            atomicAdd(&done_warps, 1);
        }
        if (acc == 0x1234567) sink[0] = acc;
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
    cudaMalloc(&d, sms * 16 * sizeof(long long));
    cudaMalloc(&sink, 4);
    const size_t smem = 1024 + (128 + 256) * 128;
    cudaFuncSetAttribute(tmem_rate_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    for (int with_mma = 0; with_mma < 2; ++with_mma) {
        const int iters = 2000;
        tmem_rate_kernel<2><<<sms, 544, smem>>>(10, with_mma, d, sink);
        tmem_rate_kernel<2><<<sms, 544, smem>>>(iters, with_mma, d, sink);
        cudaError_t err = cudaDeviceSynchronize();
        long long h[148 * 16];
        cudaMemcpy(h, d, sms * 16 * sizeof(long long), cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < sms * 16; ++i) mx = h[i] > mx ? (double)h[i] : mx;
        // bytes per iteration per SM: 16 warps x 32 lanes x 64 cols x 4 B
        const double bytes = 16.0 * 32 * 64 * 4;
        printf("tcgen05.ld 16 warps x 64 cols%s: %.1f cycles/iter (full 128x256 tile), %.1f B/clk/SM  (%s)\n",
               with_mma ? " + MMA stream" : "", mx / iters, bytes * iters / mx,
               cudaGetErrorString(err));
    }
    return 0;
}
