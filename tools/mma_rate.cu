// mma_rate.cu -- microbenchmark: raw tcgen05.mma issue rate on one B200 SM.
//
// Every CTA (one per SM) issues R back-to-back MMAs from a fixed shared-memory
// tile into TMEM (no TMA, no epilogue) and reports cycles per MMA, for the
// shapes the filter kernel uses: kind::i8 M=128 x N x K=32 and, for
// comparison, kind::f16 (bf16) M=128 x N x K=16.  Diagnostics only.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t make_desc32(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)1 << 16) | ((uint64_t)16 << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
__device__ __forceinline__ uint64_t make_desc128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <int KIND, int N, int VAR = 0>  // KIND 0 = i8, 1 = f16(bf16)
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int reps, long long *cycles,
                                                          const int8_t *stream_src, int stream_tiles) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uintptr_t base = ((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023;
    unsigned char *sA = (unsigned char *)base;        // 128 x 128 B
    unsigned char *sB = sA + 128 * 128;               // N x 128 B
    unsigned char *sS = sB + N * 128;                 // 4 x 16 KiB streaming ring
    __shared__ uint64_t bar;
    __shared__ uint64_t cbar[2];
    __shared__ uint64_t sfull[4];
    __shared__ volatile int stop;
    __shared__ uint32_t tmem_base_s;
    for (int i = threadIdx.x; i < (128 + N) * 128 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(sA)[i] =
            VAR == 9 ? (uint32_t)(i * 2654435761u) ^ 0x5bd1e995u : 0x01010101u;  // 9: random bytes
    if (threadIdx.x == 0) {
        stop = 0;
        for (int i = 0; i < 4; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sfull[i])));
        for (int i = 0; i < 2; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cbar[i])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            smem_u32(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base_s;
    uint32_t idesc;
    if (KIND == 0)
        idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    else if (KIND == 2)  // unsigned x unsigned bytes
        idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    else  // bf16 x bf16 -> f32: D fmt f32 (1 at bit 4), A/B fmt bf16 (1 at 7, 1 at 10)
        idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        t0 = clock64();
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        for (int r = 0; r < reps; ++r) {
            const uint32_t d = tmem + (uint32_t)((r & 1) * N);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                // VAR 10: a different A tile every rep (4 tiles of the ring)
                const uint32_t abase = VAR == 10 ? smem_u32(sS) + (uint32_t)((r & 3) * 16384) : a0;
                const uint64_t ad = make_desc128(abase + kk * 32), bd = make_desc128(b0 + kk * 32);
                if (KIND != 1)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(ad), "l"(bd), "r"(idesc), "r"(kk)
                        : "memory");
                else
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(ad), "l"(bd), "r"(idesc), "r"(kk)
                        : "memory");
            }
            if (VAR >= 1 && VAR < 9)
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        smem_u32(&cbar[0]))
                    : "memory");
            if (VAR >= 2 && VAR < 9) {
                const uint64_t ad = (VAR == 2) ? make_desc32(a0) : make_desc128(a0);
                const uint64_t bd = (VAR == 2) ? make_desc32(b0) : make_desc128(b0);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(1)
                    : "memory");
                asm volatile(
                    "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        smem_u32(&cbar[1]))
                    : "memory");
            }
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&bar))
            : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\n\tW:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
                smem_u32(&bar))
            : "memory");
        t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
        stop = 1;
    } else if (threadIdx.x == 64 && stream_tiles > 0) {
        // L2 -> smem stream of 16 KiB bulk copies, 4 in flight, concurrent
        // with the MMAs (the filter kernel's database-tile traffic)
        uint32_t ph[4] = {0, 0, 0, 0};
        long long i = 0;
        for (int s = 0; s < 4; ++s, ++i) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16384;" ::"r"(smem_u32(&sfull[s])) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                         ::"r"(smem_u32(sS + s * 16384)), "l"(stream_src + ((blockIdx.x * 131 + i) % stream_tiles) * 16384), "r"(smem_u32(&sfull[s])) : "memory");
        }
        while (!stop) {
            for (int s = 0; s < 4 && !stop; ++s, ++i) {
                asm volatile("{\n\t.reg .pred p;\n\tW2_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2_%=;\n\t}" ::"r"(smem_u32(&sfull[s])), "r"(ph[s]) : "memory");
                ph[s] ^= 1;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16384;" ::"r"(smem_u32(&sfull[s])) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                             ::"r"(smem_u32(sS + s * 16384)), "l"(stream_src + ((blockIdx.x * 131 + i) % stream_tiles) * 16384), "r"(smem_u32(&sfull[s])) : "memory");
            }
        }
        for (int s = 0; s < 4; ++s)
            asm volatile("{\n\t.reg .pred p;\n\tW3_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W3_%=;\n\t}" ::"r"(smem_u32(&sfull[s])), "r"(ph[s]) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int KIND, int N, int VAR = 0>
void run(const char *name, int sms, const int8_t *src = nullptr, int tiles = 0) {
    const int reps = 4096;
    long long *d;
    cudaMalloc(&d, sms * sizeof(long long));
    size_t smem = 1024 + (128 + N) * 128 + 4 * 16384;
    cudaFuncSetAttribute(mma_rate_kernel<KIND, N, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mma_rate_kernel<KIND, N, VAR><<<sms, 128, smem>>>(16, d, src, tiles);  // warm
    cudaEventRecord(e0);
    mma_rate_kernel<KIND, N, VAR><<<sms, 128, smem>>>(reps, d, src, tiles);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[1024];
    cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += (double)h[i];
    avg /= sms;
    const double mmas = ((VAR >= 2 && VAR < 9) ? 5.0 : 4.0) * reps;
    const double kmul = KIND != 1 ? 32 : 16;
    const double ops = 2.0 * 128 * N * kmul * mmas * sms;
    printf("%-6s%s N=%3d  %7.1f cycles/MMA  %8.1f T(FL)OP/s over %.3f ms  (%s)\n", name,
           tiles ? "+stream" : (VAR == 1 ? "+commit" : (VAR == 2 ? "+bias32" : (VAR == 3 ? "+bias128" : "       "))), N,
           avg / mmas, ops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(err));
    (void)0;
    cudaFree(d);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int8_t *src;
    const int tiles = 4096;  // 64 MiB, L2 resident
    cudaMalloc(&src, (size_t)tiles * 16384);
    cudaMemset(src, 1, (size_t)tiles * 16384);
    run<0, 256>("i8", sms);
    run<2, 256>("u8", sms);
    run<0, 224>("i8", sms);
    run<2, 224>("u8", sms);
    run<0, 192>("i8", sms);
    run<0, 160>("i8", sms);
    run<2, 224>("u8", sms, src, tiles);
    run<0, 256, 9>("i8rnd", sms);
    run<0, 256, 10>("i8 A-rot", sms);
    run<2, 224, 10>("u8 A-rot", sms);
    run<0, 128, 10>("i8 A-rot", sms);
    run<2, 224, 9>("u8rnd", sms);
    run<0, 128, 9>("i8rnd", sms);
    run<0, 256, 1>("i8", sms);
    run<0, 256, 2>("i8", sms);
    run<0, 256, 3>("i8", sms);
    run<0, 256>("i8", sms, src, tiles);
    run<0, 128>("i8", sms, src, tiles);
    run<0, 128>("i8", sms);
    run<0, 64>("i8", sms);
    run<0, 64, 1>("i8", sms);
    run<0, 64, 2>("i8", sms);
    run<0, 64>("i8", sms, src, tiles);
    // streaming from HBM (1 GiB region, beyond L2) concurrently with the MMAs
    int8_t *big;
    const int btiles = 65536;
    cudaMalloc(&big, (size_t)btiles * 16384);
    cudaMemset(big, 1, (size_t)btiles * 16384);
    printf("HBM stream:\n");
    run<0, 64>("i8", sms, big, btiles);
    run<0, 128>("i8", sms, big, btiles);
    run<0, 256>("i8", sms, big, btiles);
    run<1, 256>("bf16", sms);
    run<1, 128>("bf16", sms);
    return 0;
}
