// qa_tc_ptx.cuh -- inline-PTX building blocks of the tcgen05 filter kernels
// (mbarriers, TMA, tcgen05.mma / commit / ld, UMMA descriptors, shared-memory
// accesses by 32-bit address).  sm_100a only.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

namespace qa {

// 2-D uint8 tensor map over [rows, cols] (row stride ld bytes), box of
// sw x box_rows bytes in the matching 32/64/128-byte swizzle
// (qa_filter_tc.cu).
bool make_map(CUtensorMap *m, const int8_t *ptr, int64_t rows, int64_t cols, int64_t ld,
              int box_rows, int sw);

namespace {

// try_wait suspend-time hint for the epilogue warps' waits (ns)
#ifndef QA_WAIT_HINT_NS
#define QA_WAIT_HINT_NS 20000
#endif
constexpr int kWaitHintNs = QA_WAIT_HINT_NS;

// ------------------------------------------------------------------ PTX --

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t"
        "}" ::"r"(addr),
        "r"(parity), "n"(kWaitHintNs)
        : "memory");
}

__device__ __forceinline__ bool mbar_try(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t"
        "}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Wait with nanosleep backoff, for the single-thread roles (producer, MMA,
// bias), which would otherwise spin and steal issue slots from the epilogue
// warps sharing their SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    if (mbar_try(bar, parity)) return;
    uint32_t ns = 16;
    while (!mbar_try(bar, parity)) {
        __nanosleep(ns);
        ns = ns < 64 ? ns * 2 : 64;
    }
}

template <uint32_t kMaxNs>
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, uint32_t parity) {
    uint32_t ns = 32;
    while (!mbar_try(bar, parity)) {
        __nanosleep(ns);
        ns = ns < kMaxNs ? ns * 2 : kMaxNs;
    }
}

// Pure polling wait for the latency-critical MMA issuer.
__device__ __forceinline__ void mbar_wait_spin(uint64_t *bar, uint32_t parity) {
    while (!mbar_try(bar, parity)) {
    }
}

// Wait accounting (diagnostics build, -DQA_WAIT_STATS): cycles each role
// spends in each wait, summed per CTA and printed by CTAs 0..1.
#ifdef QA_WAIT_STATS
#define WSTAT(i, stmt)                      \
    do {                                    \
        const long long _t0 = clock64();    \
        stmt;                               \
        wst[i] += clock64() - _t0;          \
    } while (0)
#else
#define WSTAT(i, stmt) stmt
#endif
#ifdef QA_WAIT_STATS
constexpr int kWst = 16;
#endif

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}


__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)map) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}


// One K chunk of a tile, issued by one elected lane of a converged warp:
// KSTEPS MMAs of K=32 bytes (descriptor start addresses step by 32 B = 2 in
// the >>4 encoding), then a commit to `bar`.  Inline PTX with elect.sync
// keeps the issue free of per-lane branching.
template <int KSTEPS>
__device__ __forceinline__ void mma_chunk_elect(uint32_t tmem_d, uint64_t ad, uint64_t bd,
                                                uint32_t idesc, uint32_t first, uint32_t bar) {
    static_assert(KSTEPS == 1 || KSTEPS == 2 || KSTEPS == 4, "1, 2 or 4 K steps");
    if constexpr (KSTEPS == 4) {
        asm volatile(
            "{\n\t.reg .pred e, p;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.eq.u32 p, %4, 0;\n\t"
            "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
            "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a2, b2, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a3, b3, %3, 1;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t"
            "}" ::"r"(tmem_d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(first), "r"(bar)
            : "memory");
    } else if constexpr (KSTEPS == 2) {
        asm volatile(
            "{\n\t.reg .pred e, p;\n\t.reg .b64 a1, b1;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.eq.u32 p, %4, 0;\n\t"
            "add.s64 a1, %1, 2;\n\tadd.s64 b1, %2, 2;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, %3, 1;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t"
            "}" ::"r"(tmem_d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(first), "r"(bar)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred e, p;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.eq.u32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t"
            "}" ::"r"(tmem_d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(first), "r"(bar)
            : "memory");
    }
}

// The bias MMA of a tile (accumulate) and the commit that hands the tile to
// the epilogue, by one elected lane of a converged warp.
__device__ __forceinline__ void mma_bias_commit_elect(uint32_t tmem_d, uint64_t ad, uint64_t bd,
                                                      uint32_t idesc, uint32_t do_mma,
                                                      uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e, m;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.and.u32 m, %4, 0, e;\n\t"
        "@m tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t"
        "}" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(do_mma), "r"(bar)
        : "memory");
}

// an extra bias MMA (same constant A tile and digits; no commit)
__device__ __forceinline__ void mma_bias_elect(uint32_t tmem_d, uint64_t ad, uint64_t bd,
                                               uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;\n\t"
        "}" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc)
        : "memory");
}

__device__ __forceinline__ void tmem_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// tcgen05.wait::ld that names the 16 destination registers of an earlier
// tcgen05.ld as in-out operands: their consumers then depend on the wait
// (with other loads in flight the compiler must not move a use above it).
__device__ __forceinline__ void tmem_wait_regs(int32_t (&v)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                   "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                   "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
                 :
                 : "memory");
}

// tcgen05.ld of C (16 or 32) consecutive accumulator columns of this warp's
// 32 TMEM lanes; the registers are valid after tmem_wait().
template <int C>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, int32_t (&v)[C]) {
    if constexpr (C == 32) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32"
            " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15,"
            " %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31},"
            " [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
              "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
              "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]),
              "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr)
            : "memory");
    } else if constexpr (C == 8) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32"
            " {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7])
            : "r"(taddr)
            : "memory");
    } else {
        static_assert(C == 16, "8, 16 or 32 columns");
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32"
            " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15},"
            " [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr)
            : "memory");
    }
}

// Shared-memory atomics / stores by 32-bit shared address.  (Through a
// generic pointer the compiler emits generic ATOM / ST, an order of
// magnitude slower on the survivor path.)
__device__ __forceinline__ int32_t atom_add_smem(uint32_t addr, int32_t v) {
    int32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void sts64(uint32_t addr, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}

__device__ __forceinline__ int32_t lds32(uint32_t addr) {
    int32_t r;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(r) : "r"(addr));
    return r;
}


// UMMA shared-memory descriptor, K-major, swizzle SW bytes (32/64/128):
// start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major: 1),
// SBO>>4 [32,46) = 8 rows * SW bytes, version 1 at bit 46, layout type
// [61,64): 128B=2, 64B=4, 32B=6.
template <int SW>
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    constexpr uint64_t layout = SW == 128 ? 2 : (SW == 64 ? 4 : 6);
    constexpr uint64_t sbo = (8 * SW) >> 4;
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)1 << 16) | (sbo << 32) |
           ((uint64_t)1 << 46) | (layout << 61);
}

}  // namespace
}  // namespace qa
