// qa_filter_tc.cu -- the fused tensor-core filter pass (sm_100a).
//
// One pass scores database rows [r_lo, r_hi) against a chunk of queries and
// keeps only the (query, row) pairs that can still enter the query's top-k:
//
//   * int8 x int8 -> int32 contraction on the 5th-gen tensor cores:
//     tcgen05.mma.cta_group::1.kind::i8, M = 128 database rows, N = up to 256
//     queries, K = 32 bytes per instruction, accumulator in TMEM (double
//     buffered: 2 x N of the 512 columns);
//   * operands staged by TMA (cp.async.bulk.tensor.2d) in the 32/64/128-byte
//     swizzle the UMMA shared-memory descriptors expect; the query tile (B)
//     is loaded once per work unit, database tiles (A) stream through a
//     multi-stage mbarrier ring;
//   * the per-query filter bound is folded INTO the accumulator: one extra
//     K=32 MMA per tile multiplies a constant A tile (all 127) by a per-unit
//     B tile of int8 "bias digits", adding bias_q = 127 * sum(digits) >= -B_q
//     to every dot of query q.  A row can pass the bound only if its biased
//     value is >= 0, so the epilogue's fast path is a sign test: a 3-input
//     LOP3 AND-reduction of 32 accumulators (~0.5 instruction per element);
//   * the rare lanes with a non-negative value run the exact per-row test
//     and stage survivors in shared memory; each work unit flushes them to
//     the per-query global candidate lists with one atomic per query.  The
//     int32 score matrix never reaches HBM.
//
// Bounds (necessary conditions on the dot product, per query and per work
// unit of <= 32 consecutive tiles; units lie inside one norm-sorted block of
// the index, so the unit's norm range is narrow):
//   IP       dot >= D                      (D = k-th dot so far)
//   L2       xx - 2 dot <= T          =>   dot >= ceil((min xx - T) / 2)
//   angular  dot / xn >= P            =>   dot >= ceil(P * (P >= 0 ? min xn : max xn))
// A bound beyond the bias range is clamped conservatively, or -- if it would
// need a bias above the maximum -- its 32-column chunk is flagged
// "exceptional" and every element of the chunk takes the exact test.
//
// Warp roles (640 threads, 1 CTA per SM, persistent over an atomic counter):
//   warp 0  TMA producer          warp 1  MMA issuer (one lane)
//   warp 2  TMEM allocator        warp 3  bias builder (per work unit)
//   warps 4-19  epilogue (warp w: TMEM lanes 32*(w%4).., N/4 query columns)
//
// Reference semantics being accelerated: _core.pyx:301-330 (_scan_i8), pair
// kernel _core.pyx:49-96.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "qa_common.cuh"
#include "qa_internal.h"
#include "qa_tc_ptx.cuh"

namespace qa {

namespace {

constexpr int kBlockM = 128;
// Exact threshold test of bias-bound survivors in the epilogue, per metric.
// Angular and IP: off -- the bias bound alone decides (angular admits ~5 %
// more candidates on cfg1), the select scores every candidate exactly
// anyway, and the shorter survivor path wins (exact test: -3 % on cfg1, -2 %
// on cfg3).  L2: on -- its bound carries the bias granularity (127 x reps,
// reps ~3 for SIFT-like codes) and the unit's smallest norm; on cfg2 it
// admitted 57 % more than the exact test (627k vs 398k per 1024-query pass)
// and the exact test is +24 % q/s.  -DQA_EXACT_IN_EPILOGUE=0/1 forces it.
template <int M>
__host__ __device__ constexpr bool exact_epi() {
#if defined(QA_EXACT_IN_EPILOGUE)
    return QA_EXACT_IN_EPILOGUE != 0;
#else
    return M == kL2;
#endif
}
// MMA issuers: warp 1 plus warps 20.. (kMmaWarpsMax in all).  One warp issuing
// every tile's MMAs was the critical path of short-K passes: its ~150
// dependent SASS instructions per tile (waits, descriptor moves into uniform
// registers, elect, 5 MMAs, 2 commits) take ~1000 cycles, four times the
// tile's tensor time at K = 128 (ncu: no hot spot in that warp, every
// instruction waiting on the one before it).  Tile T of a CTA is issued by
// MMA warp T mod W, W dividing the accumulator count, so every accumulator
// has one issuer and every barrier wait still sees consecutive phases.
#ifndef QA_UNIT_LOOKAHEAD
#define QA_UNIT_LOOKAHEAD 1
#endif
#ifndef QA_MMA_WARPS
#define QA_MMA_WARPS 4
#endif
constexpr int kMmaWarpsMax = QA_MMA_WARPS;
constexpr int kMmaWarpX = 20;    // first extra MMA warp
// A second bias builder (the last warp) takes the odd work units: runs of
// single-tile units (the unit table's wide-norm blocks) are shorter than one
// builder's latency per unit (global loads, the norm copy, the digits).
constexpr int kThreads = 640 + 32 * (kMmaWarpsMax - 1) + 32;
constexpr int kBiasWarp = 3;
constexpr int kBiasWarp2 = kThreads / 32 - 1;
constexpr int kEpiWarp0 = 4;
constexpr int kEpiThreads = 512;
constexpr int kStageCapDefault = 2048;  // survivors staged in smem per work unit
constexpr int kBiasK = 32;       // K of the bias MMA (int8 columns)
constexpr int kBiasA = 127;      // constant of the bias A tile
constexpr int kSMin = -128 * kBiasK;  // digit-sum range
constexpr int kSMax = 127 * kBiasK;
constexpr int kMaxBiasReps = 8;
// TMEM accumulators in flight: all 512 columns (N=256: 2, N=128: 4, N=64: 8).
// With small query tiles the MMA of a tile is short, and two buffers left
// the pipeline bound by the MMA -> epilogue -> MMA hand-off latency.
template <int N>
__host__ __device__ constexpr int nacc() { return 512 / N < 8 ? 512 / N : 8; }
// Small query tiles (N = 64, the HBM-bound small-batch regime) skip the bias
// MMAs: each epilogue thread holds its 16 columns' bounds in registers and
// compares directly.  The tensor pipe then runs 4 MMAs per tile instead of
// 4 + reps (measured -20 % per tile with the bias MMAs removed).
#ifndef QA_DIRECT_N
#define QA_DIRECT_N 64
#endif
template <int N>
__host__ __device__ constexpr bool direct_bounds() { return N <= QA_DIRECT_N; }  // bias MMAs per tile at most (|bias| <= 4.1M)

// Epilogue organisation of the filter pass proper (kKind 0) for N >= 128:
// the 16 epilogue warps form G = min(accumulators, 4) groups; group g takes
// the CTA's tiles T = g, g + G, ... (the accumulators a = g mod G), each of
// its warps one TMEM lane quarter x N / (warps per quarter) columns, read as
// pairs of 16-column loads under one wait.  With every warp on every tile (the other kinds, and N = 64)
// each warp paid the tile's fixed costs (barrier wait, release, loop) per 32
// columns and the TMEM load latency was exposed once per tile; the groups
// pay them once per 64 or 128 columns and work on G tiles at a time.
#ifndef QA_EPI_GROUPS
#define QA_EPI_GROUPS 1
#endif
template <int N, int kKind>
__host__ __device__ constexpr bool grouped_epi() {
    return QA_EPI_GROUPS != 0 && kKind == 0 && !direct_bounds<N>();
}
#ifndef QA_EPI_ACC_PER_GROUP
#define QA_EPI_ACC_PER_GROUP 2
#endif
// A lane whose 8-column group holds a non-negative value parks the group
// (8 values + a key) in its warp's buffer; the warp tests the parked values
// one per lane once kHitDrain groups are waiting (and at the end of the work
// unit).  Testing them in place ran the exact test one candidate at a time
// with the other lanes idle -- a third of the epilogue's time for ~10
// candidates per 16k-value tile.
constexpr int kHitDrain = 8;
constexpr int kHitCap = kHitDrain + 32;  // one more group from every lane
template <int N>
__host__ __device__ constexpr int hit_words() {
    return direct_bounds<N>() ? 0 : 16 * kHitCap * 9;
}
template <int N>
__host__ __device__ constexpr int epi_groups() {
    // two accumulators per group: the MMAs of a group's next tile run while
    // it tests the current one
    constexpr int g = nacc<N>() / QA_EPI_ACC_PER_GROUP;
    return g < 1 ? 1 : (g > 4 ? 4 : g);
}

// Instruction descriptor for kind::i8: D=S32 (bits 4-5 = 2), A/B signed
// int8 (bits 7-9, 10-12 = 1), both K-major, N>>3 at 17, M>>4 at 24.
__host__ __device__ constexpr uint32_t make_idesc(int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(kBlockM >> 4) << 24);
}

// 1 when any of v[0..C) is >= 0: sign bit of the AND of all values
template <int C>
__device__ __forceinline__ bool any_nonneg(const int32_t (&v)[C]) {
    int32_t r[C / 2];
#pragma unroll
    for (int i = 0; i < C / 2; ++i) r[i] = v[2 * i] & v[2 * i + 1];
#pragma unroll
    for (int w = C / 2; w > 1; w >>= 1)
#pragma unroll
        for (int i = 0; i < w / 2; ++i) r[i] = r[2 * i] & r[2 * i + 1];
    return r[0] >= 0;
}

// A survivor staged in shared memory: query column (8 bits), its slot among
// the unit's survivors of that query (12 bits), row within the unit (12
// bits), and the dot product.
struct Staged {
    uint32_t key;  // qloc | sq << 8 | rowrel << 20
    int32_t dot;
};
constexpr int kUnitRowsMax = 32 * kBlockM;  // rows of a work unit (<= 32 tiles)
constexpr int kURing = 4;                   // unit-id ring (dynamic scheduling)

struct Params {
    FilterArgs a;
    int64_t n_tiles;        // 128-row tiles in [r_lo, r_hi)
    int64_t tiles_per_unit;
    int64_t n_qtiles;
    int64_t n_units;
    int kchunks;            // kdim / SW
    int stages;
    int b_slots;            // 1 or 2 query-tile buffers
    int stage_cap;          // survivor staging entries per slot
    int norm_bulk;          // norm arrays 16-byte aligned (bulk-copyable)
    int mma_warps;          // MMA issuer warps (divides the accumulator count)
    uint32_t idesc;         // MMA instruction descriptor (signed or unsigned bytes)
};

// Work unit u -> (query tile t = u mod n_qtiles, row unit b = u / n_qtiles).
// Query tiles vary fastest, so the CTAs working at the same time share row
// blocks (L2 reuse of the streamed database tiles).  Row unit b covers fixed
// runs of tiles_per_unit tiles, or the entry b of the pass's unit table
// (launch_unit_table: wide-norm blocks split into single tiles, listed
// first).  Units are handed out dynamically (a global counter read by the
// producer, resolved and published through the unit ring): the cost of a unit
// is dominated by its survivors, which concentrate in the norm bands near the
// queries' -- a static round-robin left the slowest CTA at 3.7x the fastest
// on cfg2.

// kKind 0: the filter pass proper (mode 0); 1: the dense, masked-dense and
// diagnostic passes (modes 1-3); 2: the sampled estimate (mode 4).  Separate
// instances keep each hot loop's register allocation free of the other paths.
template <int SW, int N, int M, int kKind>
__global__ void __launch_bounds__(kThreads, 1)
    filter_tc_kernel(const __grid_constant__ CUtensorMap tm_db,
                     const __grid_constant__ CUtensorMap tm_q, const Params p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const FilterArgs &a = p.a;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    constexpr int kNacc = nacc<N>();
#ifdef QA_WAIT_STATS
    long long wst[kWst] = {};
    __shared__ unsigned long long wst_s[kWst];
    if (threadIdx.x < kWst) wst_s[threadIdx.x] = 0;
    const long long t_start = clock64();
#endif

    // ---- shared memory carve-up (1024-aligned operand buffers) ----
    // (pointer arithmetic on the __shared__ array, not integer casts: the
    // compiler then knows every derived pointer is shared memory and emits
    // LDS / STS / ATOMS instead of generic accesses)
    unsigned char *sA = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t a_stage_bytes = kBlockM * SW;
    const uint32_t b_bytes = (uint32_t)N * (uint32_t)a.kdim;
    unsigned char *sB = sA + (size_t)p.stages * a_stage_bytes;
    // the query tile is double-buffered across work units when two copies fit
    // in 64 KiB, else single-buffered (one MMA bubble per unit switch)
    const int bslots = p.b_slots;
    unsigned char *sAbias = sB + (size_t)bslots * b_bytes;          // [128][32] = 127
    unsigned char *sBbias = sAbias + kBlockM * kBiasK;              // [2][N][32] digits
    const int stage_cap = p.stage_cap;
    Staged *stage_all = (Staged *)(sBbias + 2 * N * kBiasK);        // [2][stage_cap]
    // row norms of the unit (L2: sqnorm, angular: float bits), staged by the
    // bias warp for the exact test
    constexpr bool kExactInEpilogue = exact_epi<M>();
    constexpr int kNormSlots = (M == kIP || !kExactInEpilogue) ? 0 : 2;
    int32_t *norm_all = (int32_t *)(stage_all + 2 * stage_cap);     // [2][kUnitRowsMax]
    int32_t *thr_all = norm_all + kNormSlots * kUnitRowsMax;        // [2][N] thresholds
    int32_t *bias_s = thr_all + 2 * N;                              // [2][N] bias_q
    int32_t *exc_s = bias_s + 2 * N;                                // [2][N/32] flags
    int32_t *qcnt_all = exc_s + 2 * (N / 32);                       // [2][N] staged per query
    int32_t *qbase = qcnt_all + 2 * N;                              // [N] (flush warp)
    int32_t *bnd_all = qbase + N;                                   // [2][N] direct bounds
    // grouped epilogue: per-warp buffers of candidate 8-column groups
    int32_t *hit_all = bnd_all + 2 * N;                             // [16][kHitCap][8 + 1]
    uint64_t *bars = (uint64_t *)(hit_all + hit_words<N>());
    uint64_t *a_full = bars;
    uint64_t *a_empty = a_full + p.stages;
    uint64_t *b_full = a_empty + p.stages;
    uint64_t *b_empty = b_full + 2;
    uint64_t *acc_full = b_empty + 2;
    uint64_t *acc_empty = acc_full + kNacc;
    uint64_t *bias_full = acc_empty + kNacc;
    uint64_t *bias_empty = bias_full + 2;
    uint64_t *stage_full = bias_empty + 2;
    uint64_t *stage_free = stage_full + 2;
    uint64_t *norm_full = stage_free + 2;
    uint64_t *unit_full = norm_full + 2;        // [kURing] unit id published
    uint64_t *unit_empty = unit_full + kURing;  // [kURing] every role has read it
    uint32_t *tmem_base_s = (uint32_t *)(unit_empty + kURing);
    int32_t *stage_n_all = (int32_t *)(tmem_base_s + 1);  // [2]
    int32_t *reps_s = stage_n_all + 2;  // [2] bias MMAs per tile of the unit
    // [kURing] published work units {query tile, row unit, first tile, tiles}
    // (x = -1: no more work), 16-byte aligned
    unsigned char *uring_b = (unsigned char *)(reps_s + 2);
    uring_b += (16u - (smem_u32(uring_b) & 15u)) & 15u;
    int4 *uring = (int4 *)uring_b;
    constexpr int kEpiWarps = kEpiThreads / 32;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(a_full + s, 1);
            mbar_init(a_empty + s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(b_full + s, 1);
            mbar_init(b_empty + s, p.mma_warps);        // every MMA warp's commit
            mbar_init(bias_full + s, 1);
            mbar_init(bias_empty + s, p.mma_warps + kEpiWarps);  // MMA commits + epilogue warps
            mbar_init(stage_full + s, kEpiWarps);
            mbar_init(stage_free + s, 1);               // flush warp
            mbar_init(norm_full + s, 1);
            stage_n_all[s] = 0;
        }
        for (int s = 0; s < kNacc; ++s) {
            mbar_init(acc_full + s, 1);
            mbar_init(acc_empty + s, grouped_epi<N, kKind>() ? kEpiWarps / epi_groups<N>() : kEpiWarps);
        }
        for (int s = 0; s < kURing; ++s) {
            mbar_init(unit_full + s, 1);
            mbar_init(unit_empty + s, kEpiWarps + 3 + p.mma_warps);  // MMA, 2 bias, flush, epilogue warps
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tm_db);
        prefetch_tmap(&tm_q);
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_base_s)),
                     "n"(kNacc * N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // constant bias A tile (every byte 127: any K-major layout reads the same)
    for (int i = threadIdx.x; i < kBlockM * kBiasK / 4; i += kThreads)
        reinterpret_cast<int32_t *>(sAbias)[i] = 0x7f7f7f7f;
    for (int i = threadIdx.x; i < 2 * N; i += kThreads) qcnt_all[i] = 0;
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_base_s;

    // the it-th unit of this CTA (every consumer role walks the same
    // sequence); the slot is handed back as soon as the id is read
    auto unit_take = [&](int it) -> int4 {
        const int s = it & (kURing - 1);
        mbar_wait(unit_full + s, (uint32_t)(it / kURing) & 1);
        int4 e;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(e.x), "=r"(e.y), "=r"(e.z), "=r"(e.w)
                     : "r"(smem_u32(uring + s))
                     : "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(unit_empty + s);
        return e;
    };

    if (warp == 0) {
        // =============================== TMA producer ===================
        if (lane == 0) {
            int stage = 0;
            uint32_t aph = 0;
            // Units are handed out by a global counter (dynamic scheduling:
            // survivors concentrate in a few norm bands, so units differ in
            // cost by several x).  The producer resolves each unit (query
            // tile, row unit, its tiles -- a table lookup for table passes)
            // and publishes it to the other roles through a 4-slot ring, two
            // units ahead.  The counter's atomic, the table load and the
            // publication of consecutive units are pipelined (each waits one
            // iteration for its predecessor): a run of single-tile units
            // does not pay two global round trips per unit, and no consumer
            // role touches global memory or 64-bit division for a unit.
            const unsigned n_units = (unsigned)(
                a.unit_table ? (int64_t)__ldg(a.unit_count) * p.n_qtiles : p.n_units);
            const unsigned nqt = (unsigned)p.n_qtiles;
            auto resolve = [&](unsigned v) -> int2 {
                if (v >= n_units) return make_int2(0, 0);
                const unsigned rb = v / nqt;
                if (a.unit_table) return __ldg(reinterpret_cast<const int2 *>(a.unit_table) + rb);
                const int64_t t0 = (int64_t)rb * p.tiles_per_unit;
                return make_int2((int)t0, (int)(min(p.n_tiles, t0 + p.tiles_per_unit) - t0));
            };
            auto publish = [&](int k, unsigned v, int2 e) {
                const int s = k & (kURing - 1);
                WSTAT(14, mbar_wait_sleep(unit_empty + s, ((uint32_t)(k / kURing) & 1) ^ 1));
                const bool live = v < n_units;
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(uring + s)),
                             "r"(live ? (int)(v % nqt) : -1), "r"((int)(v / nqt)), "r"(e.x), "r"(e.y)
                             : "memory");
                mbar_arrive(unit_full + s);
            };
            // Claims run two units ahead of the unit being loaded (a claimed
            // unit is work no other CTA can take: deeper claims cost balance
            // at the end of the pass) -- except through a run of single-tile
            // units, where the claim and the table load of the next units
            // stay in flight across iterations (vb: claimed, va/ea: claimed
            // and being resolved).  Units are published in claim order.
            static_assert(QA_UNIT_LOOKAHEAD == 1 || QA_UNIT_LOOKAHEAD == 2, "1 or 2 units ahead");
            unsigned va = atomicAdd(a.sched, 1u), vb = 0;
            int2 ea = resolve(va);
            publish(0, va, ea);
            if (QA_UNIT_LOOKAHEAD == 2) {
                vb = atomicAdd(a.sched, 1u);
                ea = resolve(vb);
                publish(1, vb, ea);
            }
            bool have_a = false, have_b = false, deep = true;
            for (int it = 0;; ++it) {
                int4 un;  // own publication (the slot is rewritten at it + 2 at the earliest)
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(un.x), "=r"(un.y), "=r"(un.z), "=r"(un.w)
                             : "r"(smem_u32(uring + (it & (kURing - 1))))
                             : "memory");
                if (un.x < 0) break;
                if (!have_a) {
                    va = have_b ? vb : atomicAdd(a.sched, 1u);
                    have_b = false;
                    ea = resolve(va);
                }
                publish(it + QA_UNIT_LOOKAHEAD, va, ea);
                deep = deep && va < n_units && ea.y <= 1;
                have_a = have_b;
                if (have_b) {
                    va = vb;
                    ea = resolve(vb);  // in flight until the next iteration's publish
                }
                have_b = deep;
                if (deep) vb = atomicAdd(a.sched, 1u);  // in flight until the next iteration
                const int64_t t = un.x;
                // resident query tile for this unit
                const int bslot = it % bslots;
                const uint32_t bph = (uint32_t)(it / bslots) & 1;
                WSTAT(0, mbar_wait_sleep(b_empty + bslot, bph ^ 1));
                mbar_arrive_expect_tx(b_full + bslot, b_bytes);
                unsigned char *dstB = sB + (size_t)bslot * b_bytes;
                for (int c = 0; c < p.kchunks; ++c)
                    tma_load_2d(dstB + (size_t)c * N * SW, &tm_q, b_full + bslot, c * SW,
                                (int32_t)(t * N));
                // streamed database tiles
                const int64_t tile0 = un.z, tile1 = (int64_t)un.z + un.w;
                const int64_t tstep = a.mode == 4 ? a.sample_stride : 1;  // sampled tiles
                for (int64_t tile = tile0; tile < tile1; ++tile) {
                    const int32_t row0 = (int32_t)(a.r_lo + tile * tstep * kBlockM);
                    for (int c = 0; c < p.kchunks; ++c) {
                        WSTAT(1, mbar_wait_sleep(a_empty + stage, aph ^ 1));
                        mbar_arrive_expect_tx(a_full + stage, a_stage_bytes);
                        tma_load_2d(sA + (size_t)stage * a_stage_bytes, &tm_db, a_full + stage,
                                    c * SW, row0);
                        if (++stage == p.stages) {
                            stage = 0;
                            aph ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1 || (warp >= kMmaWarpX && warp != kBiasWarp2)) {
        // =============================== MMA issuers ====================
        // MMA warp mw issues the CTA's tiles T = mw, mw + W, ... (T counts
        // tiles across work units).  The whole warp walks the pipeline
        // (uniform control flow, no lanes parked at a warp barrier); one
        // elected lane issues.  Descriptors are formed once: the
        // start-address field is the low 14 bits (addr >> 4) and smem
        // addresses stay below 256 KiB, so stepping a descriptor is a 64-bit
        // add of (bytes >> 4).
        const int nw = p.mma_warps;
        const int mw = warp == 1 ? 0 : warp - kMmaWarpX + 1;
        if (mw < nw) {
        const uint32_t idesc = p.idesc;
        const uint64_t adesc0 = make_desc<SW>(smem_u32(sA));
        const uint64_t bdesc0 = make_desc<SW>(smem_u32(sB));
        const uint64_t abias_desc = make_desc<32>(smem_u32(sAbias));
        const uint64_t bbias_desc0 = make_desc<32>(smem_u32(sBbias));
        // this warp's next tile: its A stage / phase and accumulator / phase
        int stage = (mw * p.kchunks) % p.stages;
        uint32_t aph = (uint32_t)((mw * p.kchunks) / p.stages) & 1;
        int acc = mw % kNacc;
        uint32_t accph = (uint32_t)(mw / kNacc) & 1;
        const int skip = (nw - 1) * p.kchunks;  // stages of the other warps' tiles
        int first = mw;  // this warp's first tile of the unit
        for (int it = 0;; ++it) {
            const int4 un = unit_take(it);
            if (un.x < 0) break;
            const int slot = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            const int64_t t = un.x, b = un.y, tile0 = un.z, tile1 = (int64_t)un.z + un.w;
            (void)b, (void)t, (void)tile0, (void)tile1;
            const int ntl = (int)(tile1 - tile0);
            const int bslot = it % bslots;
            WSTAT(2, mbar_wait_spin(b_full + bslot, (uint32_t)(it / bslots) & 1));
            WSTAT(3, mbar_wait_spin(bias_full + slot, ph));
            const uint64_t bdesc = bdesc0 + (uint64_t)(((uint32_t)bslot * b_bytes) >> 4);
            const uint64_t bbias_desc = bbias_desc0 + (uint64_t)((slot * N * kBiasK) >> 4);
            const int reps = reps_s[slot];  // written before bias_full
            int ti = first;
            for (; ti < ntl; ti += nw) {
                WSTAT(4, mbar_wait_spin(acc_empty + acc, accph ^ 1));
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + (uint32_t)(acc * N);
                for (int c = 0; c < p.kchunks; ++c) {
                    WSTAT(5, mbar_wait_spin(a_full + stage, aph));
                    tc_fence_after();
                    // "mma-with-elect": the whole warp reaches the issue,
                    // one lane issues (no divergent branch around it)
                    const uint64_t ad = adesc0 + (uint64_t)((stage * a_stage_bytes) >> 4);
                    const uint64_t bd = bdesc + (uint64_t)((c * N * SW) >> 4);
                    mma_chunk_elect<SW / 32>(tmem_d, ad, bd, idesc, c == 0 ? 1u : 0u,
                                             smem_u32(a_empty + stage));
                    if (++stage == p.stages) {
                        stage = 0;
                        aph ^= 1;
                    }
                }
                // + bias_q on every row: constant A (127) x per-query digits,
                // issued `reps` times (bounds beyond one MMA's range)
                for (int r = 1; r < reps; ++r)
                    mma_bias_elect(tmem_d, abias_desc, bbias_desc, idesc);
                mma_bias_commit_elect(tmem_d, abias_desc, bbias_desc, idesc,
                                      reps == 0 ? 0u : 1u, smem_u32(acc_full + acc));
                // on to this warp's next tile (nw tiles further)
                stage += skip;
                while (stage >= p.stages) {
                    stage -= p.stages;
                    aph ^= 1;
                }
                acc += nw;
                if (acc >= kNacc) {
                    acc -= kNacc;
                    accph ^= 1;
                }
            }
            first = ti - ntl;
            // this warp's MMAs of the unit are done with the query tile and
            // the bias tile (a warp without a tile in the unit arrives at once)
            if (lane == 0) {
                tc_commit(b_empty + bslot);
                tc_commit(bias_empty + slot);
            }
            __syncwarp();
        }
        }
    } else if (warp == kBiasWarp || warp == kBiasWarp2) {
        // =============================== bias builder ===================
        // Per work unit and query column: the bound B_q (see header), the
        // digit sum S_q = ceil(-B_q / 127) clamped to [kSMin, kSMax] (a bias
        // that would need more than kSMax flags its 32-column chunk), the
        // digits (S_q spread over 32 int8) into the bias B tile, and
        // bias_q = 127 * S_q for the epilogue's exact re-test.  Runs up to
        // two units ahead of the MMA.
        constexpr int kQPL = N / 32;  // query columns per lane
        const bool filtered = (a.mode == 0 || a.mode == 3);
        const int my_slot = warp == kBiasWarp ? 0 : 1;
        for (int it = 0;; ++it) {
            const int4 un = unit_take(it);
            if (un.x < 0) break;
            const int slot = it & 1;
            if (slot != my_slot) continue;  // the other builder's unit
            const uint32_t ph = (it >> 1) & 1;
            const int64_t t = un.x, b = un.y, tile0 = un.z, tile1 = (int64_t)un.z + un.w;
            (void)b, (void)t, (void)tile0, (void)tile1;
            const int64_t q0 = t * N;
            const int nqt = (int)min((int64_t)N, a.nq - q0);
            // all global reads of the unit issued together: thresholds of
            // this lane's columns and the norm ranges of the unit's tiles
            int32_t Tq[kQPL];
#pragma unroll
            for (int i = 0; i < kQPL; ++i) {
                const int q = i * 32 + lane;
                Tq[i] = (filtered && q < nqt) ? __ldg(a.thr + q0 + q) : 0;
            }
            float nlo = INFINITY, nhi = -INFINITY;
            int32_t xlo = INT32_MAX;
            if (filtered && M != kIP) {
                const int64_t gt0 = (a.r_lo >> 7) + tile0;
                const int64_t gt1 = (a.r_lo >> 7) + tile1;
                for (int64_t g = gt0 + lane; g < gt1; g += 32) {
                    if constexpr (M == kL2) {
                        xlo = min(xlo, __ldg(a.grp_lo + g));
                    } else {
                        nlo = fminf(nlo, __int_as_float(__ldg(a.grp_lo + g)));
                        nhi = fmaxf(nhi, __int_as_float(__ldg(a.grp_hi + g)));
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    xlo = min(xlo, __shfl_xor_sync(0xffffffffu, xlo, o));
                    nlo = fminf(nlo, __shfl_xor_sync(0xffffffffu, nlo, o));
                    nhi = fmaxf(nhi, __shfl_xor_sync(0xffffffffu, nhi, o));
                }
            }
            WSTAT(6, mbar_wait_sleep(bias_empty + slot, ph ^ 1));
            // the unit's row norms -> smem (bulk copy; the < 4 tail rows and
            // unaligned arrays by plain loads)
            const bool stage_norms = kExactInEpilogue && (M != kIP) && a.mode == 0;
            if (stage_norms) {
                const int32_t row0 = (int32_t)(a.r_lo + tile0 * kBlockM);
                const int32_t nrows = (int32_t)min((tile1 - tile0) * kBlockM, a.r_hi - (int64_t)row0);
                const int32_t *src = (M == kL2) ? a.db_sqnorm + row0
                                                : reinterpret_cast<const int32_t *>(a.db_norm) + row0;
                int32_t *dst = norm_all + slot * kUnitRowsMax;
                const int32_t nbulk = p.norm_bulk ? (nrows & ~3) : 0;
                if (lane == 0) {
                    mbar_arrive_expect_tx(norm_full + slot, (uint32_t)nbulk * 4u);
                    if (nbulk > 0)
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                            " [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                            "l"(src), "r"(nbulk * 4), "r"(smem_u32(norm_full + slot))
                            : "memory");
                }
                for (int32_t i = nbulk + lane; i < nrows; i += 32) dst[i] = __ldg(src + i);
            }
            int32_t *bias_out = bias_s + slot * N;
            int32_t *thr_out = thr_all + slot * N;
            int32_t *digits_out = reinterpret_cast<int32_t *>(sBbias + slot * N * kBiasK);
            // the bounds first: the unit's bias MMA count `reps` is the
            // smallest that represents every representable bound (one MMA
            // adds up to 127 * 127 * 32 = 516k; codes far from zero, e.g.
            // SIFT-like data under min/max calibration, give dots of ~1e6)
            long long Bq[kQPL];
            int need = 1;
#pragma unroll
            for (int i = 0; i < kQPL; ++i) {
                const int q = i * 32 + lane;
                Bq[i] = 0;
                if (filtered && q < nqt) {
                    const int32_t T = Tq[i];
                    long long B;  // necessary condition dot >= B
                    if constexpr (M == kIP) {
                        B = T;
                    } else if constexpr (M == kL2) {
                        B = ((long long)xlo - (long long)T + 1) >> 1;
                    } else {
                        const float P = __int_as_float(T);
                        const float w = P >= 0.f ? nlo : nhi;
                        const float bf = __fmul_rd(P, w);  // toward -inf: conservative
                        B = bf >= 4.0e9f ? (long long)4000000000LL
                                         : (bf <= -4.0e9f ? (long long)-4000000000LL
                                                          : (long long)ceilf(bf));
                    }
                    Bq[i] = B;
                    const uint32_t mag = (uint32_t)(B >= 0 ? B : -B);  // <= 2^32 - 2^28
                    constexpr uint32_t per = (uint32_t)kBiasA * kSMax;  // 516k
                    if (mag <= per * kMaxBiasReps) need = max(need, (int)((mag + per - 1u) / per));
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) need = max(need, __shfl_xor_sync(0xffffffffu, need, o));
            constexpr bool kDirect = direct_bounds<N>();
            // dense / diagnostic passes: no bias MMA at all
            const int reps = kDirect ? 0 : (filtered ? max(1, need) : 0);
            const long long unit_a = (long long)kBiasA * (reps > 0 ? reps : 1);
            int32_t *bnd_out = bnd_all + slot * N;
#pragma unroll
            for (int i = 0; i < kQPL; ++i) {
                const int q = i * 32 + lane;
                int S = kSMin;  // padded columns: most negative bias
                bool exc = false;
                // thresholds for the exact test; padded columns never pass
                thr_out[q] = (filtered && q < nqt)
                                 ? Tq[i]
                                 : ((M == kIP) ? INT32_MAX : (M == kL2 ? INT32_MIN : 0x7fc00000));
                if constexpr (kDirect) {
                    // dot >= bnd; |dot| < 2^30, so dot - bnd never wraps
                    const long long B = !filtered ? -(1ll << 30)
                                                  : (q < nqt ? Bq[i] : (1ll << 30));
                    bnd_out[q] = (int32_t)(B < -(1ll << 30) ? -(1ll << 30)
                                                            : (B > (1ll << 30) ? (1ll << 30) : B));
                    S = 0;
                } else if (!filtered) {
                    S = 0;  // dense / diagnostic passes: plain dots
                } else if (q < nqt) {
                    // smallest S with reps*127*S >= -B
                    // (|B| <= 2^32 - 2^20: one unsigned 32-bit division; the
                    // builder's latency per unit is what short units wait for)
                    const long long nb = -Bq[i];
                    const uint32_t mag = (uint32_t)(nb >= 0 ? nb : -nb);
                    const uint32_t ua = (uint32_t)unit_a;
                    const uint32_t qd = mag / ua;
                    long long s = nb >= 0 ? (long long)qd + (mag - qd * ua != 0u) : -(long long)qd;
                    if (s > kSMax) {
                        s = kSMax;
                        exc = true;
                    }
                    if (s < kSMin) s = kSMin;
                    S = (int)s;
                }
                // direct mode: the epilogue adds bias_q = -bound in registers
                bias_out[q] = kDirect ? -bnd_out[q] : (int32_t)(unit_a * S);
                // spread S over 32 int8 digits: base + (j < rem)
                const int base = (S >= 0) ? S / kBiasK : -((-S + kBiasK - 1) / kBiasK);
                const int rem = S - base * kBiasK;  // 0 .. 31
                const uint32_t w0 = (uint32_t)(base & 0xff) * 0x01010101u;
                const uint32_t w1 = (uint32_t)((base + 1) & 0xff) * 0x01010101u;
                uint32_t dg[kBiasK / 4];
#pragma unroll
                for (int w = 0; w < kBiasK / 4; ++w) {
                    // bytes 4w + j < rem take base + 1
                    const int mb = rem - 4 * w;
                    const uint32_t sel = mb >= 4 ? 0xffffffffu : (mb <= 0 ? 0u : ((1u << (8 * mb)) - 1u));
                    dg[w] = (w0 & ~sel) | (w1 & sel);
                }
                static_assert(kBiasK == 32, "two 16-byte stores per query");
                uint4 *dq = reinterpret_cast<uint4 *>(digits_out + q * (kBiasK / 4));
                dq[0] = make_uint4(dg[0], dg[1], dg[2], dg[3]);
                dq[1] = make_uint4(dg[4], dg[5], dg[6], dg[7]);
                const unsigned eb = __ballot_sync(0xffffffffu, exc);
                if (lane == 0) exc_s[slot * (N / 32) + i] = eb != 0;
            }
            if (stage_norms) {
                WSTAT(7, mbar_wait_sleep(norm_full + slot, ph));
                if constexpr (M == kAngular) {
                    // the exact test multiplies by 1/xn: stage the reciprocal
                    const int32_t row0 = (int32_t)(a.r_lo + tile0 * kBlockM);
                    const int32_t nrows =
                        (int32_t)min((tile1 - tile0) * kBlockM, a.r_hi - (int64_t)row0);
                    int32_t *dst = norm_all + slot * kUnitRowsMax;
                    for (int32_t i = lane; i < nrows; i += 32)
                        dst[i] = __float_as_int(__frcp_rn(__int_as_float(dst[i])));
                }
            }
            if (lane == 0) reps_s[slot] = reps;
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(bias_full + slot);
        }
    } else if (warp == 2) {
        // =============================== survivor flush =================
        // Drains one work unit's staging slot while the epilogue warps
        // already fill the other: one atomic per (query, unit) reserves space
        // in the query's global candidate list, then the staged survivors
        // are copied.  The epilogue never waits on global atomics.
        constexpr int kQPL = N / 32;
        for (int it = 0;; ++it) {
            const int4 un = unit_take(it);
            if (un.x < 0) break;
            const int slot = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            const int64_t t = un.x, b = un.y, tile0 = un.z, tile1 = (int64_t)un.z + un.w;
            (void)b, (void)t, (void)tile0, (void)tile1;
            const int64_t q0 = t * N;
            const int32_t unit_row0 = (int32_t)(a.r_lo + tile0 * kBlockM);
            WSTAT(8, mbar_wait_sleep(stage_full + slot, ph));
            if (a.mode == 0 && stage_n_all[slot] > 0) {
                int32_t *qc = qcnt_all + slot * N;
                Staged *sb = stage_all + slot * stage_cap;
                const int ns = min(stage_n_all[slot], stage_cap);
#ifdef QA_WAIT_STATS
                if (lane == 0) wst[13] += ns;
#endif
                // each survivor's slot among its query's survivors of the unit
                for (int e = lane; e < ns; e += 32) {
                    const uint32_t key = sb[e].key;
                    const int sq = atomicAdd(qc + (key & 0xffu), 1);
                    sb[e].key = key | ((uint32_t)sq << 8);
                }
                __syncwarp();
                // reservations for all of this lane's queries in flight at once
                int32_t cnt[kQPL], got[kQPL];
#pragma unroll
                for (int i = 0; i < kQPL; ++i) cnt[i] = qc[i * 32 + lane];
#pragma unroll
                for (int i = 0; i < kQPL; ++i)
                    got[i] = cnt[i] > 0 ? atomicAdd(a.ccount + q0 + i * 32 + lane, cnt[i]) : 0;
#pragma unroll
                for (int i = 0; i < kQPL; ++i) {
                    qbase[i * 32 + lane] = got[i];
                    qc[i * 32 + lane] = 0;
                }
                __syncwarp();
                for (int e = lane; e < ns; e += 32) {
                    const Staged s = sb[e];
                    const int qloc = (int)(s.key & 0xffu);
                    const int32_t dst = qbase[qloc] + (int32_t)((s.key >> 8) & 0xfffu);
                    if (dst < a.cap)
                        a.cand[(q0 + qloc) * a.cap + dst] =
                            Cand{unit_row0 + (int32_t)(s.key >> 20), s.dot};
                }
                __syncwarp();
                if (lane == 0) stage_n_all[slot] = 0;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(stage_free + slot);
        }
    } else if (warp >= kEpiWarp0) {
        // =============================== epilogue =======================
        constexpr int kCB = N / 4;                 // columns per warp
        constexpr int kC = kCB < 32 ? kCB : 32;    // columns per TMEM load
        const int ew = warp - kEpiWarp0;           // 0..15
        const int quarter = warp & 3;
        const int col0 = (ew >> 2) * kCB;          // first column of this warp
        constexpr bool lean = kKind == 0;
        const uint32_t tm_warp = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)col0;
        int acc = 0;
        uint32_t accph = 0;
        int efirst = 0;  // grouped epilogue: this group's first tile of the unit
        (void)efirst;
        for (int it = 0;; ++it) {
            const int4 un = unit_take(it);
            if (un.x < 0) break;
            const int slot = it & 1;
            const uint32_t ph = (it >> 1) & 1;
            const int64_t t = un.x, b = un.y, tile0 = un.z, tile1 = (int64_t)un.z + un.w;
            (void)b, (void)t, (void)tile0, (void)tile1;
            const int64_t q0 = t * N;
            const int nqt = (int)min((int64_t)N, a.nq - q0);
            // this unit's bias, thresholds and exception flags; a free
            // staging slot (the flush warp drained its previous use)
            WSTAT(9, mbar_wait(bias_full + slot, ph));
            WSTAT(10, mbar_wait(stage_free + slot, ph ^ 1));
            int32_t *stage_n = stage_n_all + slot;
            const uint32_t stage_n_addr = smem_u32(stage_n);
            const uint32_t stage_addr = smem_u32(stage_all + slot * stage_cap);
            const uint32_t thr_addr = smem_u32(thr_all + slot * N);
            const uint32_t bias_addr = smem_u32(bias_s + slot * N);
            const int nch = max(0, min(kCB / kC, (nqt - col0 + kC - 1) / kC));
            // exceptional 32-column chunks of this warp
            uint32_t excm = 0;
            for (int ci = 0; ci < kCB / kC; ++ci)
                if (exc_s[slot * (N / 32) + (col0 + ci * kC) / 32]) excm |= 1u << ci;
            const int32_t r_hi = (int32_t)a.r_hi;
            const int32_t unit_row0 = (int32_t)(a.r_lo + tile0 * kBlockM);
            const int32_t *unit_norm = norm_all + slot * kUnitRowsMax;
            int32_t wrow0 = unit_row0 + quarter * 32;
            const int ntl = (int)(tile1 - tile0);
            if constexpr (grouped_epi<N, kKind>()) {
                // ---- filter pass, the hot loop (grouped, see epi_groups) ----
                constexpr int kG = epi_groups<N>();
                constexpr int kWPG = kEpiWarps / kG;      // warps per group
                constexpr int kCW = N / (kWPG / 4);       // columns per warp
                constexpr int kCh = 16;                   // columns per TMEM load
                constexpr int kNCh = kCW / kCh;
                static_assert(kNCh % 2 == 0, "chunks are taken in pairs");
                const int rest = ew >> 2;                 // 0..3 within the lane quarter
                const int grp = rest % kG;
                const int gcol0 = (rest / kG) * kCW;      // first column of this warp
                const uint32_t tm_g = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)gcol0;
                if (it == 0) {
                    acc = grp;  // group g owns accumulators g, g + G, ...
                    accph = 0;
                    efirst = grp;
                }
                uint32_t excw = 0;  // exceptional 32-column chunks of this warp
                for (int ci = 0; ci < kCW / 32; ++ci)
                    if (exc_s[slot * (N / 32) + (gcol0 + ci * 32) / 32]) excw |= 1u << ci;
                int32_t *hvals = hit_all + ew * (kHitCap * 9);  // [kHitCap][8]
                int32_t *hkeys = hvals + kHitCap * 8;           // [kHitCap]
                const uint32_t hvals_addr = smem_u32(hvals);
                const uint32_t lt_mask = (1u << lane) - 1u;
                int hcnt = 0;  // parked groups (warp-uniform)
                // the parked values, one per lane: exact test, survivors staged
                auto drain = [&]() {
                    __syncwarp();
                    for (int i = lane; i < hcnt * 8; i += 32) {
                        const uint32_t key = (uint32_t)hkeys[i >> 3];
                        const int32_t vj = hvals[i];
                        if (vj < 0 && !(key >> 31)) continue;
                        const int qloc = (int)(key & 0xffu) + (i & 7);
                        const int rowrel = (int)((key >> 8) & 0xfffu);
                        const int32_t dot = (int32_t)((uint32_t)vj -
                                                      (uint32_t)lds32(bias_addr + 4u * (uint32_t)qloc));
                        if constexpr (kExactInEpilogue) {
                            int32_t xx = 0;
                            float inv_xn = 0.f;
                            if constexpr (M != kIP) {
                                const int32_t nb = unit_norm[rowrel];  // staged by the bias warp
                                if constexpr (M == kL2) xx = nb;
                                if constexpr (M == kAngular) inv_xn = __int_as_float(nb);  // 1/xn
                            }
                            const int32_t T = lds32(thr_addr + 4u * (uint32_t)qloc);
                            if (!passes<M>(dot, T, xx, inv_xn)) continue;
                        }
                        const int e = atom_add_smem(stage_n_addr, 1);
                        if (e < stage_cap) {
                            // slot among the query's survivors: the flush warp's
                            sts64(stage_addr + 8u * (uint32_t)e,
                                  (uint32_t)qloc | ((uint32_t)rowrel << 20), (uint32_t)dot);
                        } else {
                            // staging full: direct append (slow, rare)
                            const int32_t sl = atomicAdd(a.ccount + q0 + qloc, 1);
                            if (sl < a.cap)
                                a.cand[(q0 + qloc) * a.cap + sl] = Cand{unit_row0 + rowrel, dot};
                        }
                    }
                    __syncwarp();
                    hcnt = 0;
                };
                // park the lanes' candidate groups (warp-uniform control flow)
                auto park8 = [&](const int32_t *c8, bool hit, int qc0, bool exc, int32_t row) {
                    const unsigned m = __ballot_sync(0xffffffffu, hit);
                    if (!m) return;
                    if (hit) {
                        const int pos = hcnt + __popc(m & lt_mask);
                        const uint32_t va = hvals_addr + 32u * (uint32_t)pos;
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(va), "r"(c8[0]),
                                     "r"(c8[1]), "r"(c8[2]), "r"(c8[3])
                                     : "memory");
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(va + 16u),
                                     "r"(c8[4]), "r"(c8[5]), "r"(c8[6]), "r"(c8[7])
                                     : "memory");
                        hkeys[pos] = (int32_t)((uint32_t)qc0 | ((uint32_t)(row - unit_row0) << 8) |
                                               (exc ? 0x80000000u : 0u));
                    }
                    hcnt += __popc(m);
                    if (hcnt >= kHitDrain) drain();
                };
                // one 16-column chunk: sign test of each 8-column group; the
                // rare chunk with a candidate parks its groups
                auto test16 = [&](const int32_t (&v)[kCh], int ch, int32_t row) {
                    const int32_t g0 = (v[0] & v[1] & v[2]) & (v[3] & v[4] & v[5]) & (v[6] & v[7]);
                    const int32_t g1 =
                        (v[8] & v[9] & v[10]) & (v[11] & v[12] & v[13]) & (v[14] & v[15]);
                    const bool exc = (excw >> (ch * kCh / 32)) & 1u;
                    if (!__any_sync(0xffffffffu, (g0 & g1) >= 0 || exc)) return;
                    const bool rowok = row < r_hi;
                    const int qc0 = gcol0 + ch * kCh;
                    park8(v, rowok && (g0 >= 0 || exc), qc0, exc, row);
                    park8(v + 8, rowok && (g1 >= 0 || exc), qc0 + 8, exc, row);
                };
                int ti = efirst;
                for (; ti < ntl; ti += kG) {
                    const int32_t row = wrow0 + ti * kBlockM + lane;
                    WSTAT(11, mbar_wait(acc_full + acc, accph));
                    tc_fence_after();
                    const uint32_t ta = tm_g + (uint32_t)(acc * N);
                    int32_t va[kCh], vb[kCh];
                    // the two loads of a pair go out back to back and one wait
                    // covers both (ptxas sinks a load issued between the tests
                    // below them, so a look-ahead load hid nothing)
#pragma unroll
                    for (int ch = 0; ch < kNCh; ch += 2) {
                        tmem_ld_cols<kCh>(ta + (uint32_t)(ch * kCh), va);
                        tmem_ld_cols<kCh>(ta + (uint32_t)((ch + 1) * kCh), vb);
                        tmem_wait_regs(va);
                        tmem_wait_regs(vb);
                        if (ch + 2 >= kNCh) {
                            // every column is in registers: hand the accumulator back
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(acc_empty + acc);
                        }
                        test16(va, ch, row);
                        test16(vb, ch + 1, row);
                    }
                    acc += kG;
                    if (acc >= kNacc) {
                        acc -= kNacc;
                        accph ^= 1;
                    }
                }
                efirst = ti - ntl;
                if (hcnt) drain();  // the unit's bias, norms and staging slot end here
            } else if constexpr (lean) {
                // ---- filter pass, the hot loop ----
                // Fast path per tile: TMEM -> registers, one sign bit per
                // 8-column group (AND-reduction), and the accumulator is
                // released right away when no lane of the warp has a group
                // with a non-negative biased value.  Otherwise the hit
                // groups are re-read from TMEM (8 columns at a time, warp-
                // uniform loop), given the exact test, and staged; the
                // accumulator is released after that.
                uint32_t excg = 0;           // groups of exceptional chunks
                for (int ci = 0; ci < kCB / kC; ++ci)
                    if ((excm >> ci) & 1u) excg |= ((1u << (kC / 8)) - 1u) << (ci * (kC / 8));
                int32_t row = wrow0 + lane;
                constexpr bool kDirect = direct_bounds<N>();
                int32_t bq[kDirect ? kCB : 1];
                if constexpr (kDirect) {
#pragma unroll
                    for (int c = 0; c < kCB; ++c) bq[c] = lds32(bias_addr + 4u * (uint32_t)(col0 + c));
                }
                for (int ti = 0; ti < ntl; ++ti, row += kBlockM) {
                    WSTAT(11, mbar_wait(acc_full + acc, accph));
                    tc_fence_after();
                    const uint32_t ta = tm_warp + (uint32_t)(acc * N);
                    int32_t v[kCB / kC][kC];
#pragma unroll
                    for (int ci = 0; ci < kCB / kC; ++ci)
                        tmem_ld_cols<kC>(ta + (uint32_t)(ci * kC), v[ci]);
                    tmem_wait();
                    // the tile is in registers: hand the accumulator back now
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(acc_empty + acc);
                    if (++acc == kNacc) {
                        acc = 0;
                        accph ^= 1;
                    }
                    if constexpr (kDirect) {  // the bias the MMA did not add
#pragma unroll
                        for (int ci = 0; ci < kCB / kC; ++ci)
#pragma unroll
                            for (int j = 0; j < kC; ++j) v[ci][j] += bq[ci * kC + j];
                    }
                    // one AND over all of this lane's values first: most
                    // lane-tiles hold no candidate, and the per-group mask
                    // below is only built for the others
                    int32_t g8s[kCB / 8];
#pragma unroll
                    for (int ci = 0; ci < kCB / kC; ++ci)
#pragma unroll
                        for (int h = 0; h < kC / 8; ++h) {
                            const int32_t *c8 = v[ci] + 8 * h;
                            g8s[ci * (kC / 8) + h] = (c8[0] & c8[1] & c8[2]) &
                                                     (c8[3] & c8[4] & c8[5]) & (c8[6] & c8[7]);
                        }
                    int32_t gall = g8s[0];
#pragma unroll
                    for (int g = 1; g < kCB / 8; ++g) gall &= g8s[g];
                    if ((gall < 0 && !excg) || row >= r_hi) continue;
                    uint32_t hit = excg;
#pragma unroll
                    for (int g = 0; g < kCB / 8; ++g) hit |= ((uint32_t)~g8s[g] >> 31) << g;
                    // slow path (lanes with a candidate group only): exact
                    // test of every non-negative column of a hit group
                    const int rowrel = row - unit_row0;
                    int32_t xx = 0;
                    float inv_xn = 0.f;
                    if constexpr (M != kIP && kExactInEpilogue) {
                        const int32_t nb = unit_norm[rowrel];  // staged by the bias warp
                        if constexpr (M == kL2) xx = nb;
                        if constexpr (M == kAngular) inv_xn = __int_as_float(nb);  // 1/xn
                    }
#pragma unroll
                    for (int ci = 0; ci < kCB / kC; ++ci)
#pragma unroll
                        for (int h = 0; h < kC / 8; ++h) {
                            const int g = ci * (kC / 8) + h;
                            if (!((hit >> g) & 1u)) continue;
                            const int32_t *c8 = v[ci] + 8 * h;
                            uint32_t m8 = 0;
                            if ((excg >> g) & 1u) {
                                m8 = 0xffu;
                            } else {
#pragma unroll
                                for (int j = 0; j < 8; ++j) m8 |= (uint32_t)(c8[j] >= 0) << j;
                            }
                            while (m8) {
                                const int j = __ffs(m8) - 1;
                                m8 &= m8 - 1;
                                int32_t vj = c8[0];
#pragma unroll
                                for (int jj = 1; jj < 8; ++jj) vj = (j == jj) ? c8[jj] : vj;
                                const int qloc = col0 + 8 * g + j;
                                const int32_t dot = (int32_t)((uint32_t)vj -
                                                              (uint32_t)lds32(bias_addr + 4u * (uint32_t)qloc));
                                if constexpr (kExactInEpilogue) {
                                    const int32_t T = lds32(thr_addr + 4u * (uint32_t)qloc);
                                    if (!passes<M>(dot, T, xx, inv_xn)) continue;
                                }
                                const int e = atom_add_smem(stage_n_addr, 1);
                                if (e < stage_cap) {
                                    // slot among the query's survivors: the flush warp's
                                    sts64(stage_addr + 8u * (uint32_t)e,
                                          (uint32_t)qloc | ((uint32_t)rowrel << 20), (uint32_t)dot);
                                } else {
                                    // staging full: direct append (slow, rare)
                                    const int32_t s = atomicAdd(a.ccount + q0 + qloc, 1);
                                    if (s < a.cap) a.cand[(q0 + qloc) * a.cap + s] = Cand{row, dot};
                                }
                            }
                        }
                }
            } else if constexpr (kKind == 2) {
            if constexpr (N <= 128) {
                // ---- sampled estimate: best goodness per (query, bucket) ----
                // A bucket is 8 lanes of one warp (lane & 3 fixed) over the
                // unit's tiles.  The j-th best bucket bounds the j-th best row
                // from below (every bucket best is a distinct row), and with
                // hundreds of buckets per query the two rarely differ.
                // goodness: IP dot, L2 2*dot - xx (int32), angular float(dot)/xn
                // (tracked as float, mapped to an ordered int32 at the end)
                using G = typename std::conditional<M == kAngular, float, int32_t>::type;
                G gbest[kCB];
#pragma unroll
                for (int c = 0; c < kCB; ++c) gbest[c] = M == kAngular ? (G)(-INFINITY) : (G)INT32_MIN;
                const int32_t rstep = (int32_t)(a.sample_stride * kBlockM);
                wrow0 = (int32_t)(a.r_lo + tile0 * a.sample_stride * kBlockM) + quarter * 32;
                // the row norm two tiles ahead (its global load would stall
                // the tile: the accumulator is usually ready)
                auto norm_of = [&](int32_t row) -> int32_t {
                    if constexpr (M == kIP) return 0;
                    if (row >= r_hi) return 0;
                    return M == kL2 ? __ldg(a.db_sqnorm + row)
                                    : __ldg(reinterpret_cast<const int32_t *>(a.db_norm) + row);
                };
                int32_t nrm0 = ntl > 0 ? norm_of(wrow0 + lane) : 0;
                int32_t nrm1 = ntl > 1 ? norm_of(wrow0 + rstep + lane) : 0;
                for (int ti = 0; ti < ntl; ++ti, wrow0 += rstep) {
                    const int32_t row = wrow0 + lane;
                    const bool valid = row < r_hi;
                    const int32_t nrm = nrm0;
                    nrm0 = nrm1;
                    nrm1 = ti + 2 < ntl ? norm_of(row + 2 * rstep) : 0;
                    mbar_wait(acc_full + acc, accph);
                    tc_fence_after();
                    const uint32_t ta = tm_warp + (uint32_t)(acc * N);
                    int32_t v[kCB / kC][kC];
#pragma unroll
                    for (int ci = 0; ci < kCB / kC; ++ci)
                        tmem_ld_cols<kC>(ta + (uint32_t)(ci * kC), v[ci]);
                    tmem_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(acc_empty + acc);
                    if (++acc == kNacc) {
                        acc = 0;
                        accph ^= 1;
                    }
                    if (!valid) continue;
                    const float inv_xn = M == kAngular ? __frcp_rn(__int_as_float(nrm)) : 0.f;
#pragma unroll
                    for (int ci = 0; ci < kCB / kC; ++ci)
#pragma unroll
                        for (int j = 0; j < kC; ++j) {
                            if constexpr (M == kIP) {
                                gbest[ci * kC + j] = max(gbest[ci * kC + j], v[ci][j]);
                            } else if constexpr (M == kL2) {  // |.| < 2^26 for kdim <= 1024
                                gbest[ci * kC + j] = max(gbest[ci * kC + j], 2 * v[ci][j] - nrm);
                            } else {
                                gbest[ci * kC + j] =
                                    fmaxf(gbest[ci * kC + j], __int2float_rn(v[ci][j]) * inv_xn);
                            }
                        }
                }
                int32_t best[kCB];
#pragma unroll
                for (int c = 0; c < kCB; ++c) {
                    if constexpr (M == kAngular) {
                        const int32_t g = __float_as_int(gbest[c]);
                        best[c] = g < 0 ? (g ^ 0x7fffffff) : g;  // float order as int
                    } else {
                        best[c] = (int32_t)gbest[c];
                    }
                }
                // fold lanes differing in bits 4, 3, 2: each lane ends with
                // kCB / 8 columns of its bucket (lane & 3)
                int colb = 0;
#pragma unroll
                for (int o = 16, C = kCB; o >= 4; o >>= 1, C >>= 1) {
                    const bool up = (lane & o) != 0;
#pragma unroll
                    for (int h = 0; h < C / 2; ++h) {
                        const int32_t keep = up ? best[h + C / 2] : best[h];
                        const int32_t send = up ? best[h] : best[h + C / 2];
                        best[h] = max(keep, __shfl_xor_sync(0xffffffffu, send, o));
                    }
                    if (up) colb += C / 2;
                }
                const int64_t bucket = b * 16 + quarter * 4 + (lane & 3);
#pragma unroll
                for (int h = 0; h < kCB / 8; ++h) {
                    const int c = col0 + colb + h;
                    if (c < nqt) a.est_keys[(q0 + c) * a.est_ld + bucket] = best[h];
                }
            }
            } else {
            if (a.mode == 1 || a.mode == 3) {
                // ---- dense (round 0) and masked-dense (early rounds) ----
                // every element has its candidate slot; masked dense marks
                // rows failing the bound row = -1 (no atomics at all)
                for (int ti = 0; ti < ntl; ++ti, wrow0 += kBlockM) {
                    const int32_t row = wrow0 + lane;
                    mbar_wait(acc_full + acc, accph);
                    tc_fence_after();
                    const uint32_t ta = tm_warp + (uint32_t)(acc * N);
                    int32_t v[kCB / kC][kC];
#pragma unroll
                    for (int ci = 0; ci < kCB / kC; ++ci)
                        tmem_ld_cols<kC>(ta + (uint32_t)(ci * kC), v[ci]);
                    tmem_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(acc_empty + acc);
                    if (++acc == kNacc) {
                        acc = 0;
                        accph ^= 1;
                    }
                    if (row >= r_hi) continue;
                    Cand *dst = a.cand + q0 * a.cap + (row - (int32_t)a.r_lo);
#pragma unroll
                    for (int ci = 0; ci < kCB / kC; ++ci) {
                        const bool exc = (excm >> ci) & 1u;
#pragma unroll
                        for (int j = 0; j < kC; ++j) {
                            const int c = col0 + ci * kC + j;
                            if (c >= nqt) break;
                            Cand out;
                            if (a.mode == 1) {
                                out = Cand{row, v[ci][j]};
                            } else {
                                const int32_t bias_c = lds32(bias_addr + 4u * (uint32_t)c);
                                // direct mode: TMEM holds the plain dot
                                const int32_t biased = direct_bounds<N>() ? v[ci][j] + bias_c : v[ci][j];
                                const int32_t dot = (int32_t)((uint32_t)biased - (uint32_t)bias_c);
                                out = (biased >= 0 || exc) ? Cand{row, dot} : Cand{-1, 0};
                            }
                            dst[(int64_t)c * a.cap] = out;
                        }
                    }
                }
            } else {
                // ---- diagnostics (mode 2): the full dot matrix ----
                for (int ti = 0; ti < ntl; ++ti, wrow0 += kBlockM) {
                    const int32_t row = wrow0 + lane;
                    const bool valid = row < r_hi;
                    mbar_wait(acc_full + acc, accph);
                    tc_fence_after();
                    const uint32_t tbase = tm_warp + (uint32_t)(acc * N);
#pragma unroll 1
                    for (int ci = 0; ci < nch; ++ci) {
                        int32_t cur[kC];
                        tmem_ld_cols<kC>(tbase + (uint32_t)(ci * kC), cur);
                        tmem_wait();
                        if (!valid) continue;
#pragma unroll
                        for (int j = 0; j < kC; ++j) {
                            const int c = col0 + ci * kC + j;
                            if (c < nqt) a.dots_out[(q0 + c) * a.ld_dots + row] = cur[j];
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(acc_empty + acc);
                    if (++acc == kNacc) {
                        acc = 0;
                        accph ^= 1;
                    }
                }
            }
            }
            // this warp is done with the unit's bias / thresholds and staging
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(bias_empty + slot);
                mbar_arrive(stage_full + slot);
            }
        }
    }

#ifdef QA_WAIT_STATS
    if (lane == 0)
        for (int i = 0; i < kWst; ++i)
            if (wst[i]) atomicAdd(&wst_s[i], (unsigned long long)wst[i]);
    __syncthreads();
    if (threadIdx.x == 0)
        printf("wstc cta=%d total=%lld surv=%d\n", (int)blockIdx.x, clock64() - t_start,
               (int)wst_s[13]);
    if (threadIdx.x == 0 && blockIdx.x < 2)
        printf("wst cta=%d total=%lld prod[b_empty=%llu a_empty=%llu] mma[b_full=%llu bias_full=%llu "
               "acc_empty=%llu a_full=%llu] bias[bias_empty=%llu norm=%llu] flush[stage_full=%llu] "
               "epi/16[bias_full=%llu stage_free=%llu acc_full=%llu acc_full_x=%llu]\n",
               (int)blockIdx.x, clock64() - t_start, wst_s[0], wst_s[1], wst_s[2], wst_s[3],
               wst_s[4], wst_s[5], wst_s[6], wst_s[7], wst_s[8], wst_s[9] / 16, wst_s[10] / 16,
               wst_s[11] / 16, wst_s[12] / 16);
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "n"(kNacc * N));
    }
}

// ------------------------------------------------------------- host side --

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
    }
    return fn;
}

bool make_map(CUtensorMap *m, const int8_t *ptr, int64_t rows, int64_t cols, int64_t ld,
              int box_rows, int sw) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {(cuuint32_t)sw, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUtensorMapSwizzle swz = sw == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                       : (sw == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                   : CU_TENSOR_MAP_SWIZZLE_32B);
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void *)ptr, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

namespace {

// Diagnostics knobs, read once from the environment; production runs use
// the defaults.
struct Knobs {
    int stage_cap, max_stages, b_slots;
};
const Knobs &knobs() {
    static const Knobs k = [] {
        auto env_int = [](const char *name, int dflt) {
            const char *v = getenv(name);
            return (v && *v) ? atoi(v) : dflt;
        };
        return Knobs{env_int("QA_B200_STAGECAP", kStageCapDefault),
                     env_int("QA_B200_MAXSTAGES", 12), env_int("QA_B200_BSLOTS", 2)};
    }();
    return k;
}

// Tiles per work unit: a power of two <= 32, so units stay inside one
// 32-tile norm-sorted block of an index laid out by qa_order_rows_by_norm;
// at least ~8 units per CTA so the dynamic assignment can balance.  The
// sampled-estimate pass (mode 4) takes ~2 units per CTA instead: its units
// are uniform in cost, and fewer units mean fewer buckets for the select.
int64_t tiles_per_unit(int64_t n_tiles, int64_t n_qtiles, int mode, int sms) {
    int64_t tpu = 1;
    if (mode == 4) {
        const int64_t want = (n_tiles * n_qtiles + 2 * sms - 1) / (2 * (int64_t)sms);
        while (tpu < want && tpu < 32) tpu *= 2;
        return tpu;
    }
    static const int upc = [] {  // diagnostics: units per CTA aimed at
        const char *v = getenv("QA_B200_UNITS_PER_CTA");
        return v && atoi(v) > 0 ? atoi(v) : 8;
    }();
    const int64_t want = (n_tiles * n_qtiles) / ((int64_t)sms * upc);
    while (tpu * 2 <= want && tpu < 32) tpu *= 2;
    return tpu;
}

// Query-tile width N of a pass: the largest whose B buffer fits 64 KiB, no
// larger than the query chunk needs (0: unsupported).
int pick_tile_n(int64_t nq, int64_t kdim, int mode) {
    const int nmax = (int)(65536 / kdim);
    static const int force_n = [] {  // diagnostics: QA_B200_TILE_N=128 / 64
        const char *v = getenv("QA_B200_TILE_N");
        return v ? atoi(v) : 0;
    }();
    if (force_n == 256 && nmax >= 256 && nq > 128 && mode == 0) return 256;
    if (force_n == 128 && nmax >= 128) return 128;
    if (force_n == 64 && nmax >= 64) return 64;
    // 256-query tiles only when K is long enough for the MMA time per tile to
    // cover the epilogue (cfg3, d = 256: 420 vs 542 us per final pass); with
    // K <= 128 the 128-query tiles and their 4 TMEM accumulators absorb the
    // epilogue's survivor work better (cfg2: 1.76M -> 1.90M q/s; cfg1 and
    // the dense round 0 likewise)
    if (nq > 128 && nmax >= 256 && kdim > 128 && mode == 0) return 256;
    if (nq > 64 && nmax >= 128) return 128;
    if (nmax >= 64) return 64;
    return 0;
}

template <int SW, int N, int M>
cudaError_t launch_t(const FilterArgs &a, cudaStream_t st) {
    if (a.mode == 4 && (!a.est_keys || a.sample_stride < 1 || a.max_tpu < 1))
        return cudaErrorInvalidValue;
    CUtensorMap tm_db, tm_q;
    if (!make_map(&tm_db, a.db, a.r_hi, a.kdim, a.ldd, kBlockM, SW)) return cudaErrorNotSupported;
    if (!make_map(&tm_q, a.q, a.nq, a.kdim, a.ldq, N, SW)) return cudaErrorNotSupported;
    Params p;
    p.a = a;
    p.n_tiles = (a.r_hi - a.r_lo + kBlockM - 1) / kBlockM;
    if (a.mode == 4) p.n_tiles = (p.n_tiles + a.sample_stride - 1) / a.sample_stride;
    p.n_qtiles = (a.nq + N - 1) / N;
    p.kchunks = (int)(a.kdim / SW);
    const int sms = num_sms();
    int64_t tpu = tiles_per_unit(p.n_tiles, p.n_qtiles, a.mode, sms);
    if (a.mode == 4) {
        tpu = a.max_tpu;  // the caller sized its bucket array with it
        if ((p.n_tiles + tpu - 1) / tpu * 16 > a.est_ld) return cudaErrorInvalidValue;
    } else if (a.max_tpu > 0) {
        tpu = std::min<int64_t>(tpu, a.max_tpu);
    }
    p.tiles_per_unit = tpu;
    p.n_units = ((p.n_tiles + tpu - 1) / tpu) * p.n_qtiles;
    if (a.unit_table) {
        // a unit table (mode 0 only) lists at most one unit per tile
        if (a.mode != 0 || !a.unit_count) return cudaErrorInvalidValue;
        p.n_units = p.n_tiles * p.n_qtiles;  // upper bound: the grid size
    }
    const Knobs &kn = knobs();
    p.idesc = make_idesc(N);
    p.stage_cap = kn.stage_cap;
    {
        const void *nrm = (M == kL2) ? (const void *)a.db_sqnorm : (const void *)a.db_norm;
        p.norm_bulk = ((uintptr_t)nrm % 16) == 0;
    }
    p.b_slots = (2 * (size_t)N * a.kdim <= 65536) ? 2 : 1;
    if (kn.b_slots == 1) p.b_slots = 1;
    const size_t fixed = 1024 /*align slack*/ + (size_t)p.b_slots * N * a.kdim +
                         kBlockM * kBiasK + 2 * (size_t)N * kBiasK +
                         2 * (size_t)p.stage_cap * sizeof(Staged) +
                         (M == kIP || !exact_epi<M>() ? 0 : 2 * (size_t)kUnitRowsMax * sizeof(int32_t)) +
                         (9 * N + 2 * (N / 32) + hit_words<N>()) * sizeof(int32_t) + 512;
#ifdef QA_WAIT_STATS
    const size_t budget = 227 * 1024 - 3072;  // the static wait counters (2 KiB with alignment)
#else
    const size_t budget = 227 * 1024;
#endif
    const size_t stage_bytes = (size_t)kBlockM * SW;
    // each stage also costs two 8-byte mbarriers
    if (fixed + 2 * (stage_bytes + 16) > budget) return cudaErrorNotSupported;
    int stages = (int)((budget - fixed) / (stage_bytes + 16));
    if (stages > kn.max_stages) stages = kn.max_stages;
    p.stages = stages;
    {
        // every accumulator gets one issuer (W divides the accumulator
        // count), and a warp may run ahead of the others by a full set of
        // accumulators: the A ring must hold those tiles for the stage
        // barriers to see consecutive phases
        // tensor cycles of one tile's MMAs (M128 x N x K32 takes N / 2): one
        // issuer keeps up once they cover its ~1000-cycle issue sequence
        // (cfg3, N = 256, K = 256: 78 % of peak with one issuer, 74 % with two)
        const int tile_cycles = p.kchunks * (SW / 32) * (N / 2);
        int w = tile_cycles >= 1024 ? 1 : std::min(kMmaWarpsMax, nacc<N>());
        while (w > 1 && (nacc<N>() % w != 0)) --w;
        if (stages < nacc<N>() * p.kchunks) w = 1;
        static const int force_w = [] {  // diagnostics: QA_B200_MMA_WARPS=1/2/4
            const char *v = getenv("QA_B200_MMA_WARPS");
            return v ? atoi(v) : 0;
        }();
        if (force_w >= 1 && force_w <= w && nacc<N>() % force_w == 0) w = force_w;
        // a ring of a multiple of W * kchunks stages gives every stage one
        // issuer for the whole pass: its full/empty barriers then never skip
        // a phase for any waiter, whatever order the bulk loads complete in
        // (ring depth beyond 4 tiles measured no gain: cfg2 4 = 7 stages)
        if (w > 1) {
            const int unit = w * p.kchunks;
            if (stages >= unit) {
                stages = stages / unit * unit;
                p.stages = stages;
            } else {
                w = 1;
            }
        }
        p.mma_warps = w;
    }
    const size_t smem = fixed + (size_t)stages * (stage_bytes + 16);
    auto kern = a.mode == 0 ? filter_tc_kernel<SW, N, M, 0>
                            : (a.mode == 4 ? filter_tc_kernel<SW, N, M, 2> : filter_tc_kernel<SW, N, M, 1>);
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int64_t grid = p.n_units < sms ? p.n_units : sms;
    kern<<<(unsigned)grid, kThreads, smem, st>>>(tm_db, tm_q, p);
    return cudaGetLastError();
}

template <int SW, int N>
cudaError_t dispatch_metric(const FilterArgs &a, cudaStream_t st) {
    switch (a.metric) {
        case kIP: return launch_t<SW, N, kIP>(a, st);
        case kL2: return launch_t<SW, N, kL2>(a, st);
        default: return launch_t<SW, N, kAngular>(a, st);
    }
}

template <int SW>
cudaError_t dispatch_n(const FilterArgs &a, cudaStream_t st) {
    switch (pick_tile_n(a.nq, a.kdim, a.mode)) {
        case 256: return dispatch_metric<SW, 256>(a, st);
        case 128: return dispatch_metric<SW, 128>(a, st);
        case 64: return dispatch_metric<SW, 64>(a, st);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace

int filter_tiles_per_unit(int64_t rows, int64_t nq, int64_t kdim) {
    const int n = pick_tile_n(nq, kdim, 0);
    if (n == 0 || rows <= 0) return 0;
    const int64_t n_tiles = (rows + kBlockM - 1) / kBlockM;
    return (int)tiles_per_unit(n_tiles, (nq + n - 1) / n, 0, num_sms());
}

void filter_est_layout(int64_t tiles, int64_t nq, int64_t kdim, int64_t min_buckets, int *tpu,
                       int64_t *buckets) {
    *tpu = 0;
    *buckets = 0;
    const int n = pick_tile_n(nq, kdim, 4);
    if (n == 0 || tiles <= 0) return;
    int64_t t = tiles_per_unit(tiles, (nq + n - 1) / n, 4, num_sms());
    while (t > 1 && (tiles + t - 1) / t * 16 < min_buckets) t /= 2;
    *tpu = (int)t;
    *buckets = (tiles + t - 1) / t * 16;  // 16 buckets per row unit (epilogue)
}

cudaError_t launch_filter_tc(const FilterArgs &a, cudaStream_t st) {
    if (a.r_hi <= a.r_lo || a.nq == 0) return cudaSuccess;
    if (!a.sched) return cudaErrorInvalidValue;
    if (a.kdim % 32 != 0 || a.kdim > 1024) return cudaErrorNotSupported;
    if (a.ldd % 16 != 0 || a.ldq % 16 != 0) return cudaErrorNotSupported;
    if (a.r_hi > INT32_MAX) return cudaErrorNotSupported;
    // the biased accumulator must not wrap: |dot| + |bias| < 2^31
    if (a.kdim > 65536) return cudaErrorNotSupported;
    if (a.kdim % 128 == 0) return dispatch_n<128>(a, st);
    if (a.kdim == 64) return dispatch_n<64>(a, st);
    if (a.kdim == 32) return dispatch_n<32>(a, st);
    return cudaErrorNotSupported;
}

}  // namespace qa
