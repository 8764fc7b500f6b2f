// qa_layout.cu -- index layout: rows ordered by code norm.
//
// The filter derives one integer bound per (work unit of <= 32 tiles,
// query) from the smallest / largest norm among the unit's rows
// (qa_filter_tc.cu).  Storing the index rows in norm-banded blocks makes
// every unit's norm range narrow, so the bound is nearly the exact per-row
// test.  The order starts from a stable radix sort on the int32 squared norm
// (CUB, part of the CUDA toolkit); reported ids stay the caller's row
// positions through the row_ids map passed to the scan.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>

#include "qa_internal.h"

namespace qa {

namespace {

// Stored order (perm[i] = sorted row placed at stored row i):
//
//   [sample region]  kSampleTiles 128-row tiles taken at evenly spaced
//                    positions of the norm-sorted order (tile k at sorted
//                    tile floor(k * Tn / S)), themselves stored interleaved;
//   [main region]    the remaining sorted rows cut into 4096-row blocks
//                    (32 tiles, one narrow norm band each), block-interleaved:
//                    stored block t <- block (t * step + T/2) mod T;
//   [tail]           a partial last block, last.
//
// The search scans row prefixes and its threshold estimate treats the first
// 32768 rows as a sample of the whole index: the sample region makes that
// prefix STRATIFIED over every norm band (L2 neighbours concentrate in the
// bands near the query's norm, so a prefix of a few whole bands misjudges
// their density).  Main-region blocks start at multiples of 4096 rows, so
// every filter work unit (<= 32 tiles, aligned) stays inside one band.
// Indexes too small for the estimate (< 4 sample regions) skip the sample
// region, and so do angular indexes (the caller's choice): their code norms
// span a narrow range, the estimate holds without stratification, and the
// prefix passes keep tight per-unit bounds.
constexpr int64_t kSampleTiles = 256;  // 32768 rows = the plan's estimate prefix

__device__ __forceinline__ int64_t sampled_le(int64_t x, int64_t S, int64_t Tn) {
    // number of k in [0, S) with floor(k * Tn / S) <= x (S == 0: no sample
    // region, and Tn may be 0 then)
    if (x < 0 || S == 0) return 0;
    const int64_t c = ((x + 1) * S + Tn - 1) / Tn;
    return c < S ? c : S;
}

__global__ void layout_kernel(const int32_t *__restrict__ sorted, int64_t n, int64_t Tn, int64_t S,
                              int64_t sstep, int64_t T, int64_t step, int32_t *__restrict__ perm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (i < S * 128) {
        const int64_t slot = i >> 7;
        const int64_t k = (slot * sstep + S / 2) % S;
        perm[i] = sorted[(k * Tn / S) * 128 + (i & 127)];
        return;
    }
    const int64_t j = i - S * 128;  // index in the rest (sorted order minus samples)
    const int64_t bt = j / 4096;
    const int64_t r = bt < T ? ((bt * step + T / 2) % T) * 4096 + (j % 4096) : j;
    // rest tile rt -> sorted tile s: the rt-th tile not sampled
    const int64_t rt = r >> 7;
    int64_t m = sampled_le(rt, S, Tn);
    for (;;) {
        const int64_t m2 = sampled_le(rt + m, S, Tn);
        if (m2 == m) break;
        m = m2;
    }
    perm[i] = sorted[(rt + m) * 128 + (r & 127)];
}

int64_t coprime_step(int64_t full) {
    // a step near T/phi, coprime to T: spreads consecutive stored blocks
    // across the sorted order
    if (full <= 1) return 1;
    int64_t step = (int64_t)((double)full * 0.6180339887) | 1;
    auto gcd = [](int64_t x, int64_t y) {
        while (y) {
            int64_t t = x % y;
            x = y;
            y = t;
        }
        return x;
    };
    while (gcd(step, full) != 1) step += 2;
    return step;
}

__global__ void iota_kernel(int32_t *p, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = (int32_t)i;
}

// one warp per destination row, 16-byte vector copies (ld is a multiple of 32)
__global__ void permute_rows_kernel(const int8_t *__restrict__ src, const int32_t *__restrict__ sq_in,
                                    const float *__restrict__ n_in, int64_t n, int64_t ld,
                                    const int32_t *__restrict__ perm, int8_t *__restrict__ dst,
                                    int32_t *__restrict__ sq_out, float *__restrict__ n_out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < n; r += nwarps) {
        const int64_t s = perm[r];
        const int4 *sp = reinterpret_cast<const int4 *>(src + s * ld);
        int4 *dp = reinterpret_cast<int4 *>(dst + r * ld);
        for (int64_t j = lane; j < ld / 16; j += 32) dp[j] = __ldg(sp + j);
        if (lane == 0) {
            if (sq_out) sq_out[r] = sq_in[s];
            if (n_out) n_out[r] = n_in[s];
        }
    }
}

// one warp per 128-row tile (4 rows per lane)
__global__ void group_ranges_kernel(int metric, const int32_t *__restrict__ sqnorm,
                                    const float *__restrict__ norm, int64_t n,
                                    int32_t *__restrict__ lo, int32_t *__restrict__ hi,
                                    int64_t groups) {
    const int lane = threadIdx.x & 31;
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (g >= groups) return;
    if (metric == 1) {
        int32_t v = INT32_MAX, w = INT32_MIN;
        for (int i = 0; i < 4; ++i) {
            const int64_t r = g * 128 + i * 32 + lane;
            if (r < n) {
                v = min(v, sqnorm[r]);
                w = max(w, sqnorm[r]);
            }
        }
        for (int o = 16; o; o >>= 1) {
            v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
            w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
        }
        if (lane == 0) {
            lo[g] = v;
            hi[g] = w;
        }
    } else {
        float vmin = INFINITY, vmax = -INFINITY;
        for (int i = 0; i < 4; ++i) {
            const int64_t r = g * 128 + i * 32 + lane;
            if (r < n) {
                vmin = fminf(vmin, norm[r]);
                vmax = fmaxf(vmax, norm[r]);
            }
        }
        for (int o = 16; o; o >>= 1) {
            vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
            vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        }
        if (lane == 0) {
            lo[g] = __float_as_int(vmin);
            hi[g] = __float_as_int(vmax);
        }
    }
}

// The work-unit table of a mode-0 filter pass (launch_unit_table): one warp
// per run of tpu tiles writes the run's norm range; the last CTA to finish
// (ticket counter) turns the ranges into the table.
constexpr int kUnitThreads = 1024;

__device__ __forceinline__ double tile_lo_of(int metric, const int32_t *lo, int64_t g) {
    return metric == 1 ? (double)lo[g] : (double)__int_as_float(lo[g]);
}
__device__ __forceinline__ double tile_hi_of(int metric, const int32_t *hi, int64_t g) {
    return metric == 1 ? (double)hi[g] : (double)__int_as_float(hi[g]);
}

__global__ void __launch_bounds__(kUnitThreads) unit_table_kernel(
    int metric, const int32_t *__restrict__ lo, const int32_t *__restrict__ hi, int64_t tile_lo,
    int64_t n_tiles, int tpu, int32_t *__restrict__ table, int32_t *__restrict__ count,
    unsigned *__restrict__ ticket, double *__restrict__ rmin, double *__restrict__ rmax,
    int tail_pct, int tail_split, int wide_tiles) {
    using Reduce = cub::BlockReduce<double, kUnitThreads>;
    using Scan = cub::BlockScan<int, kUnitThreads>;
    __shared__ union {
        typename Reduce::TempStorage r;
        typename Scan::TempStorage s;
    } tmp;
    __shared__ double s_min, s_max;
    __shared__ int s_wide;
    __shared__ bool s_last;
    const int64_t B = (n_tiles + tpu - 1) / tpu;
    const int lane = threadIdx.x & 31;
    // ---- every CTA: the ranges of its runs (one warp per run)
    const int64_t b = (int64_t)blockIdx.x * (kUnitThreads / 32) + (threadIdx.x >> 5);
    if (b < B) {
        double a = INFINITY, z = -INFINITY;
        const int64_t g = b * tpu + lane;
        if (lane < tpu && g < n_tiles) {
            a = tile_lo_of(metric, lo, tile_lo + g);
            z = tile_hi_of(metric, hi, tile_lo + g);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
            z = fmax(z, __shfl_xor_sync(0xffffffffu, z, o));
        }
        if (lane == 0) {
            rmin[b] = a;
            rmax[b] = z;
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // ---- the last CTA: the table
    double vmin = INFINITY, vmax = -INFINITY;
    for (int64_t i = threadIdx.x; i < B; i += kUnitThreads) {
        vmin = fmin(vmin, __ldcg(rmin + i));
        vmax = fmax(vmax, __ldcg(rmax + i));
    }
    vmin = Reduce(tmp.r).Reduce(vmin, [](double x, double y) { return fmin(x, y); });
    __syncthreads();
    vmax = Reduce(tmp.r).Reduce(vmax, [](double x, double y) { return fmax(x, y); });
    if (threadIdx.x == 0) {
        s_min = vmin;
        s_max = vmax;
        s_wide = 0;
        *ticket = 0;  // ready for the next launch
    }
    __syncthreads();
    // a run is wide when its range exceeds 4x the average run's share
    const double limit = 4.0 * (s_max - s_min) / (double)B;
    const int64_t per = (B + kUnitThreads - 1) / kUnitThreads;
    const int64_t b0 = min(B, (int64_t)threadIdx.x * per), b1 = min(B, b0 + per);
    auto tiles_of = [&](int64_t r) { return (int)(min(n_tiles, (r + 1) * tpu) - r * tpu); };
    auto wide = [&](int64_t r) { return tpu > 1 && __ldcg(rmax + r) - __ldcg(rmin + r) > limit; };
    int nw = 0;
    for (int64_t r = b0; r < b1; ++r) nw += wide(r) ? 1 : 0;
    if (nw) atomicAdd(&s_wide, nw);
    __syncthreads();
    // split only when the wide runs are the exception (a layout that is not
    // norm-ordered has no narrow runs; single tiles would only add overhead)
    const bool split = (int64_t)s_wide * 8 <= B;
    // the runs at the end of the table are cut into `tail_split` units each:
    // units are handed out in table order, and a CTA that takes one of the
    // last full runs ends a unit's length after the others (the slowest CTA
    // of a cfg2 pass ended 10 % after the median)
    const int64_t cut = B - (B * tail_pct) / 100;
    auto parts_of = [&](int64_t r) {
        return (r >= cut && tail_split > 1 && tiles_of(r) >= tail_split) ? tail_split : 1;
    };
    int n_split = 0, n_reg = 0;
    for (int64_t r = b0; r < b1; ++r) {
        if (split && wide(r)) n_split += (tiles_of(r) + wide_tiles - 1) / wide_tiles;
        else n_reg += parts_of(r);
    }
    int off_split, off_reg, tot_split;
    Scan(tmp.s).ExclusiveSum(n_split, off_split, tot_split);
    __syncthreads();
    Scan(tmp.s).ExclusiveSum(n_reg, off_reg);
    off_reg += tot_split;
    for (int64_t r = b0; r < b1; ++r) {
        if (split && wide(r)) {
            const int64_t g1 = min(n_tiles, (r + 1) * tpu);
            for (int64_t g = r * tpu; g < g1; g += wide_tiles) {
                table[2 * off_split] = (int32_t)g;
                table[2 * off_split + 1] = (int32_t)min((int64_t)wide_tiles, g1 - g);
                ++off_split;
            }
        } else {
            const int parts = parts_of(r), nt = tiles_of(r);
            int t0 = 0;
            for (int i = 0; i < parts; ++i) {
                const int len = (nt - t0) / (parts - i);
                table[2 * off_reg] = (int32_t)(r * tpu) + t0;
                table[2 * off_reg + 1] = len;
                t0 += len;
                ++off_reg;
            }
        }
    }
    if (threadIdx.x == kUnitThreads - 1) *count = off_reg;
}

}  // namespace

cudaError_t launch_unit_table(int metric, const int32_t *grp_lo, const int32_t *grp_hi,
                              int64_t tile_lo, int64_t n_tiles, int tpu, int32_t *table,
                              int32_t *count, unsigned *ticket, double *scratch, cudaStream_t st) {
    if (metric == 0 || n_tiles <= 0 || tpu < 1 || tpu > 32 || n_tiles > INT32_MAX)
        return cudaErrorInvalidValue;
    const int64_t B = (n_tiles + tpu - 1) / tpu;
    const unsigned grid = (unsigned)((B + kUnitThreads / 32 - 1) / (kUnitThreads / 32));
    static const int tail_pct = [] {  // diagnostics: share of the runs cut into smaller units
        const char *v = getenv("QA_B200_TAIL_PCT");
        return v ? atoi(v) : 10;
    }();
    static const int wide_tiles = [] {  // tiles per unit of a wide-norm run
        const char *v = getenv("QA_B200_WIDE_TILES");
        // cfg2: 8 (= 4) tiles +3.3 % over single tiles, 16 +2.5 %, whole runs
        // -3.5 %: once a candidate costs little in the epilogue, a unit's
        // fixed cost (its bias build) outweighs the tighter single-tile bound
        return v && atoi(v) > 0 ? atoi(v) : 8;
    }();
    static const int tail_split = [] {
        const char *v = getenv("QA_B200_TAIL_SPLIT");
        return v ? atoi(v) : 2;  // cfg2: the last 10 % halved +2.7 %; quarters or 20 % cost more than they save
    }();
    unit_table_kernel<<<grid, kUnitThreads, 0, st>>>(metric, grp_lo, grp_hi, tile_lo, n_tiles, tpu,
                                                     table, count, ticket, scratch, scratch + B,
                                                     tail_pct, tail_split, wide_tiles);
    return cudaGetLastError();
}

cudaError_t launch_group_ranges(int metric, const int32_t *sqnorm, const float *norm, int64_t n,
                                int32_t *lo, int32_t *hi, int64_t groups, cudaStream_t st) {
    if (groups == 0 || metric == 0) return cudaSuccess;
    group_ranges_kernel<<<(unsigned)((groups * 32 + 255) / 256), 256, 0, st>>>(metric, sqnorm, norm,
                                                                              n, lo, hi, groups);
    return cudaGetLastError();
}

cudaError_t launch_order_by_key(const int32_t *key, int64_t n, bool stratify, int32_t *perm,
                                void *scratch,
                                size_t scratch_bytes, size_t *needed, cudaStream_t st) {
    // layout of scratch: [keys_out n*4][vals_in n*4][cub temp]
    size_t temp = 0;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint32_t *)nullptr,
                                                    (uint32_t *)nullptr, (const int32_t *)nullptr,
                                                    (int32_t *)nullptr, (int)n, 0, 32, st);
    if (e != cudaSuccess) return e;
    const size_t off = ((size_t)n * 12 + 255) / 256 * 256;
    *needed = off + temp;
    if (!scratch || scratch_bytes < *needed) return cudaSuccess;  // size query
    uint32_t *keys_out = (uint32_t *)scratch;
    int32_t *vals_in = (int32_t *)((char *)scratch + (size_t)n * 4);
    int32_t *sorted = (int32_t *)((char *)scratch + (size_t)n * 8);
    iota_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(vals_in, n);
    // squared norms are >= 0, so their uint32 order is their int32 order
    e = cub::DeviceRadixSort::SortPairs((char *)scratch + off, temp, (const uint32_t *)key,
                                        keys_out, vals_in, sorted, (int)n, 0, 32, st);
    if (e != cudaSuccess) return e;
    const int64_t Tn = n / 128;
    const int64_t S = (stratify && Tn >= 4 * kSampleTiles) ? kSampleTiles : 0;
    const int64_t T = (n - S * 128) / 4096;
    layout_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sorted, n, Tn, S, coprime_step(S),
                                                               T, coprime_step(T), perm);
    return cudaGetLastError();
}

cudaError_t launch_permute_rows(const int8_t *src, const int32_t *sq_in, const float *n_in,
                                int64_t n, int64_t ld, const int32_t *perm, int8_t *dst,
                                int32_t *sq_out, float *n_out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    int64_t blocks = (n + 7) / 8;
    int64_t cap = (int64_t)num_sms() * 8;
    if (blocks > cap) blocks = cap;
    permute_rows_kernel<<<(unsigned)blocks, 256, 0, st>>>(src, sq_in, n_in, n, ld, perm, dst, sq_out,
                                                          n_out);
    return cudaGetLastError();
}

}  // namespace qa
