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
__device__ __forceinline__ uint64_t make_desc128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <int KIND, int N>  // KIND 0 = i8, 1 = f16(bf16)
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int reps, long long *cycles) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    uintptr_t base = ((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023;
    unsigned char *sA = (unsigned char *)base;        // 128 x 128 B
    unsigned char *sB = sA + 128 * 128;               // N x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base_s;
    for (int i = threadIdx.x; i < (128 + N) * 128 / 4; i += blockDim.x)
        reinterpret_cast<int32_t *>(sA)[i] = 0x01010101;
    if (threadIdx.x == 0) {
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
                const uint64_t ad = make_desc128(a0 + kk * 32), bd = make_desc128(b0 + kk * 32);
                if (KIND == 0)
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
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int KIND, int N>
void run(const char *name, int sms) {
    const int reps = 4096;
    long long *d;
    cudaMalloc(&d, sms * sizeof(long long));
    size_t smem = 1024 + (128 + N) * 128;
    cudaFuncSetAttribute(mma_rate_kernel<KIND, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mma_rate_kernel<KIND, N><<<sms, 128, smem>>>(16, d);  // warm
    cudaEventRecord(e0);
    mma_rate_kernel<KIND, N><<<sms, 128, smem>>>(reps, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[1024];
    cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += (double)h[i];
    avg /= sms;
    const double mmas = 4.0 * reps;
    const double kmul = KIND == 0 ? 32 : 16;
    const double ops = 2.0 * 128 * N * kmul * mmas * sms;
    printf("%-10s N=%3d  %7.1f cycles/MMA  %8.1f T(FL)OP/s over %.3f ms  (%s)\n", name, N,
           avg / mmas, ops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(err));
    cudaFree(d);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 256>("i8", sms);
    run<0, 128>("i8", sms);
    run<0, 64>("i8", sms);
    run<1, 256>("bf16", sms);
    run<1, 128>("bf16", sms);
    return 0;
}
