// qa_stats.cu -- the reference's calibration statistics on the GPU,
// bit-exact (quantizer.py:176-222 estimate_stats).
//
// What numpy computes (verified against numpy 2.3 in tests/golden):
//   mu[j]    = (sequential float64 sum over rows of x[i, j]) / n
//              (an axis-0 reduction of a C-contiguous block adds row by row;
//              a block one column wide is contiguous along the reduction and
//              numpy sums it pairwise instead -- d % 64 == 1)
//   sigma[j] = sqrt((sequential sum of round(c*c), c = x - mu[j]) / n)
//   min/max  = order-free (NaN propagates)
//   qlo/qhi  = exact order statistics: sorted column at floor((n-1)*0.001)
//              ('lower') and ceil((n-1)*0.999) ('higher'); NaN if the column
//              holds a NaN
//   tam[j]   = max |x - mu[j]| over qlo <= x <= qhi, -inf when none is kept
//   pooled   = float(np.sum(block)) per 64-column block -- numpy's pairwise
//              summation over the flattened block (leaves of <= 128 values
//              summed with 8 interleaved accumulators, split points rounded
//              down to multiples of 8) -- accumulated across blocks in
//              Python float order; pooled sigma likewise over
//              round(round(x - flat_mu)^2).
//
// GPU mapping: the sequential column sums are one thread per column with
// coalesced row reads (order fixed by definition, so no tree); the order
// statistics are a 4-pass 8-bit radix select on float32 order keys with
// per-column shared-memory histograms; tam is an order-free max; the pairwise
// sums split the flattened block into the exact subtrees numpy's recursion
// forms, sum each subtree in one thread on the GPU, and the host recombines
// the top of the tree in the same order.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "qa_common.cuh"
#include "qa_internal.h"

namespace qa {

namespace {

constexpr int kColBlock = 32;     // columns per warp in the sequential sums
constexpr int kStatsChunk = 64;   // the reference's _STATS_CHUNK

// ---- (1) sequential column sums, min, max, NaN flags --------------------
__global__ void colsum_kernel(const float *__restrict__ x, int64_t n, int64_t d, int64_t ldx,
                              double *__restrict__ mu, double *__restrict__ mn,
                              double *__restrict__ mx, int *__restrict__ has_nan) {
    const int64_t j = (int64_t)blockIdx.x * kColBlock + threadIdx.x;
    if (j >= d) return;
    double s = 0.0, lo = INFINITY, hi = -INFINITY;
    bool nan = false;
    const float *p = x + j;
    int64_t i = 0;
    for (; i + 8 <= n; i += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(p + (i + u) * ldx);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double w = (double)v[u];
            s = __dadd_rn(s, w);
            nan |= (w != w);
            lo = fmin(lo, w);
            hi = fmax(hi, w);
        }
    }
    for (; i < n; ++i) {
        const double w = (double)__ldg(p + i * ldx);
        s = __dadd_rn(s, w);
        nan |= (w != w);
        lo = fmin(lo, w);
        hi = fmax(hi, w);
    }
    mu[j] = __ddiv_rn(s, (double)n);
    mn[j] = nan ? NAN : lo;
    mx[j] = nan ? NAN : hi;
    has_nan[j] = nan ? 1 : 0;
}

// ---- (2) sequential sum of squared deviations -> sigma ------------------
__global__ void colvar_kernel(const float *__restrict__ x, int64_t n, int64_t d, int64_t ldx,
                              const double *__restrict__ mu, double *__restrict__ sigma) {
    const int64_t j = (int64_t)blockIdx.x * kColBlock + threadIdx.x;
    if (j >= d) return;
    const double m = mu[j];
    double s = 0.0;
    const float *p = x + j;
    int64_t i = 0;
    for (; i + 8 <= n; i += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(p + (i + u) * ldx);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double c = __dsub_rn((double)v[u], m);
            s = __dadd_rn(s, __dmul_rn(c, c));
        }
    }
    for (; i < n; ++i) {
        const double c = __dsub_rn((double)__ldg(p + i * ldx), m);
        s = __dadd_rn(s, __dmul_rn(c, c));
    }
    sigma[j] = __dsqrt_rn(__ddiv_rn(s, (double)n));
}

// ---- (3) radix select of two order statistics per column ----------------
__device__ __forceinline__ uint32_t fkey(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_to_float(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// state per column c and target t (0 = lo, 1 = hi): prefix (digits found so
// far, in the high bits) and the rank still to skip inside that prefix
struct SelState {
    uint32_t prefix[2];
    int64_t rank[2];
};

constexpr int kSelThreads = 256;
constexpr int kSelRowsPerCta = 4096;

__global__ void __launch_bounds__(kSelThreads)
radix_hist_kernel(const float *__restrict__ x, int64_t n, int64_t lo_col, int ncols, int64_t ldx,
                  const SelState *__restrict__ st, int pass, unsigned int *__restrict__ hist) {
    // hist: [ncols][2][256]
    extern __shared__ unsigned int sh[];
    const int tid = threadIdx.x;
    for (int i = tid; i < ncols * 512; i += kSelThreads) sh[i] = 0;
    __syncthreads();
    const int shift = 24 - 8 * pass;
    const int c = tid % kColBlock;      // column within a 32-wide group
    const int rsub = tid / kColBlock;   // 8 row lanes
    const int64_t r0 = (int64_t)blockIdx.x * kSelRowsPerCta;
    const int64_t r1 = min(n, r0 + kSelRowsPerCta);
    for (int cg = 0; cg < ncols; cg += kColBlock) {
        const int col = cg + c;
        if (col < ncols) {
            const SelState s = st[col];
            for (int64_t r = r0 + rsub; r < r1; r += kSelThreads / kColBlock) {
                const uint32_t k = fkey(__ldg(x + r * ldx + lo_col + col));
                const uint32_t dig = (k >> shift) & 0xffu;
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const bool match = pass == 0 || ((k ^ s.prefix[t]) >> (shift + 8)) == 0;
                    if (match) atomicAdd(&sh[(col * 2 + t) * 256 + dig], 1u);
                }
            }
        }
    }
    __syncthreads();
    for (int i = tid; i < ncols * 512; i += kSelThreads)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// one thread per (column, target): find the digit holding the rank
__global__ void radix_pick_kernel(SelState *__restrict__ st, const unsigned int *__restrict__ hist,
                                  int ncols, int pass) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ncols * 2) return;
    const int col = i >> 1, t = i & 1;
    const unsigned int *h = hist + (size_t)i * 256;
    int64_t rank = st[col].rank[t];
    int dig = 0;
    for (; dig < 255; ++dig) {
        if (rank < (int64_t)h[dig]) break;
        rank -= h[dig];
    }
    const int shift = 24 - 8 * pass;
    st[col].prefix[t] |= (uint32_t)dig << shift;
    st[col].rank[t] = rank;
}

// ---- (4) trimmed abs-max: max |x - mu| over qlo <= x <= qhi -------------
__global__ void __launch_bounds__(kSelThreads)
tam_kernel(const float *__restrict__ x, int64_t n, int64_t d, int64_t ldx,
           const double *__restrict__ mu, const SelState *__restrict__ st,
           const int *__restrict__ has_nan, unsigned long long *__restrict__ tam_bits,
           int *__restrict__ kept_any) {
    const int tid = threadIdx.x;
    const int c = tid % kColBlock, rsub = tid / kColBlock;
    const int64_t r0 = (int64_t)blockIdx.x * kSelRowsPerCta;
    const int64_t r1 = min(n, r0 + kSelRowsPerCta);
    for (int64_t col = (int64_t)blockIdx.y * kColBlock + c; col < d; col += (int64_t)gridDim.y * kColBlock) {
        if (has_nan[col]) continue;      // qlo = NaN: nothing is kept
        const double qlo = (double)key_to_float(st[col].prefix[0]);
        const double qhi = (double)key_to_float(st[col].prefix[1]);
        const double m = mu[col];
        unsigned long long best = 0;
        bool any = false;
        for (int64_t r = r0 + rsub; r < r1; r += kSelThreads / kColBlock) {
            const double w = (double)__ldg(x + r * ldx + col);
            if (w >= qlo && w <= qhi) {
                const double a = fabs(__dsub_rn(w, m));
                const unsigned long long b = (unsigned long long)__double_as_longlong(a);
                best = b > best ? b : best;   // non-negative doubles (and NaN) order as their bits
                any = true;
            }
        }
        if (any) {
            atomicMax(tam_bits + col, best);
            if (!kept_any[col]) atomicExch(kept_any + col, 1);
        }
    }
}

// ---- (5) numpy pairwise sums over the flattened 64-column block ---------
// value of flattened element e of block [*, lo_col, lo_col + c)
struct BlockView {
    const float *x;
    int64_t ldx, lo_col, c;
    double shift;   // pass 2: value = round(round(x - shift)^2)
    int squared;
    __device__ __forceinline__ double at(int64_t e) const {
        const int64_t r = e / c, j = e - r * c;
        const double v = (double)__ldg(x + r * ldx + lo_col + j);
        if (!squared) return v;
        const double t = __dsub_rn(v, shift);
        return __dmul_rn(t, t);
    }
};

// numpy pairwise_sum for a node of length m <= kPwNode starting at e0
__device__ double pw_node(const BlockView &v, int64_t e0, int64_t m) {
    // explicit stack: the recursion splits at n2 = (m/2) - (m/2)%8 until
    // m <= 128; nodes are summed left-to-right and combined as left + right
    struct Frame { int64_t off, len; double left; int state; };
    Frame stk[24];
    int sp = 0;
    stk[0] = {e0, m, 0.0, 0};
    double ret = 0.0;
    for (;;) {
        Frame &f = stk[sp];
        if (f.len <= 128) {
            double res;
            if (f.len < 8) {
                res = 0.0;
                for (int64_t i = 0; i < f.len; ++i) res = __dadd_rn(res, v.at(f.off + i));
            } else {
                double r[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) r[u] = v.at(f.off + u);
                int64_t i = 8;
                const int64_t lim = f.len - (f.len % 8);
                for (; i < lim; i += 8) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) r[u] = __dadd_rn(r[u], v.at(f.off + i + u));
                }
                res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                                __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
                for (; i < f.len; ++i) res = __dadd_rn(res, v.at(f.off + i));
            }
            ret = res;
            // return to the parent frames
            for (;;) {
                if (sp == 0) return ret;
                --sp;
                Frame &p = stk[sp];
                if (p.state == 1) {  // left done -> run right
                    p.left = ret;
                    p.state = 2;
                    int64_t n2 = p.len / 2;
                    n2 -= n2 % 8;
                    stk[++sp] = {p.off + n2, p.len - n2, 0.0, 0};
                    break;
                }
                ret = __dadd_rn(p.left, ret);  // right done
            }
            continue;
        }
        int64_t n2 = f.len / 2;
        n2 -= n2 % 8;
        f.state = 1;
        stk[++sp] = {f.off, n2, 0.0, 0};
    }
}

__global__ void pw_nodes_kernel(BlockView v, const int64_t *__restrict__ off,
                                const int64_t *__restrict__ len, int64_t nodes,
                                double *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nodes) out[i] = pw_node(v, off[i], len[i]);
}

constexpr int64_t kPwNode = 4096;  // subtrees summed by one thread

// host: enumerate the subtrees of numpy's recursion with length <= kPwNode
void pw_split(int64_t off, int64_t m, std::vector<int64_t> &offs, std::vector<int64_t> &lens) {
    if (m <= kPwNode || m <= 128) {
        offs.push_back(off);
        lens.push_back(m);
        return;
    }
    int64_t n2 = m / 2;
    n2 -= n2 % 8;
    pw_split(off, n2, offs, lens);
    pw_split(off + n2, m - n2, offs, lens);
}

// host: recombine in the recursion's order, consuming the node sums
double pw_combine(int64_t m, const double *vals, size_t &idx) {
    if (m <= kPwNode || m <= 128) return vals[idx++];
    int64_t n2 = m / 2;
    n2 -= n2 % 8;
    const double a = pw_combine(n2, vals, idx);
    const double b = pw_combine(m - n2, vals, idx);
    return a + b;
}

// numpy pairwise sum of the m flattened elements of v (synchronous)
cudaError_t pairwise_sum(const BlockView &v, int64_t m, cudaStream_t st, double *out) {
    std::vector<int64_t> offs, lens;
    pw_split(0, m, offs, lens);
    const int64_t nodes = (int64_t)offs.size();
    int64_t *doff = nullptr, *dlen = nullptr;
    double *dnodes = nullptr;
    std::vector<double> vals((size_t)nodes);
    cudaError_t e;
    if ((e = cudaMalloc(&doff, nodes * 8)) == cudaSuccess &&
        (e = cudaMalloc(&dlen, nodes * 8)) == cudaSuccess &&
        (e = cudaMalloc(&dnodes, nodes * 8)) == cudaSuccess &&
        (e = cudaMemcpyAsync(doff, offs.data(), nodes * 8, cudaMemcpyHostToDevice, st)) == cudaSuccess &&
        (e = cudaMemcpyAsync(dlen, lens.data(), nodes * 8, cudaMemcpyHostToDevice, st)) == cudaSuccess) {
        pw_nodes_kernel<<<(unsigned)((nodes + 127) / 128), 128, 0, st>>>(v, doff, dlen, nodes, dnodes);
        if ((e = cudaGetLastError()) == cudaSuccess &&
            (e = cudaMemcpyAsync(vals.data(), dnodes, nodes * 8, cudaMemcpyDeviceToHost, st)) == cudaSuccess &&
            (e = cudaStreamSynchronize(st)) == cudaSuccess) {
            size_t idx = 0;
            *out = pw_combine(m, vals.data(), idx);
        }
    }
    cudaFree(doff);
    cudaFree(dlen);
    cudaFree(dnodes);
    return e;
}

}  // namespace

// Full estimate_stats.  x: device float32 [n, ldx]; outputs: HOST arrays of
// d doubles + two scalars.  Synchronous on `st`.
cudaError_t launch_estimate_stats(const float *x, int64_t n, int64_t d, int64_t ldx, double *mu,
                                  double *sigma, double *mn, double *mx, double *tam,
                                  double *qlo, double *qhi, double *pooled_mu,
                                  double *pooled_sigma, cudaStream_t st) {
    cudaError_t e;
    double *dmu = nullptr, *dsig = nullptr, *dmn = nullptr, *dmx = nullptr;
    int *dnan = nullptr, *dkept = nullptr;
    unsigned long long *dtam = nullptr;
    SelState *dsel = nullptr;
    unsigned int *dhist = nullptr;
    std::vector<SelState> hsel((size_t)d);
    std::vector<int> hnan((size_t)d), hkept((size_t)d);
    std::vector<unsigned long long> htam((size_t)d);
    const int64_t klo = (int64_t)std::floor((double)(n - 1) * 0.001);
    const int64_t khi = (int64_t)std::ceil((double)(n - 1) * 0.999);
    double flat_sum = 0.0, pooled_var = 0.0, last_mu = 0.0, last_sigma = 0.0;
#define QA_CK(x)                         \
    do {                                 \
        if ((e = (x)) != cudaSuccess) goto done; \
    } while (0)
    QA_CK(cudaMalloc(&dmu, d * 8));
    QA_CK(cudaMalloc(&dsig, d * 8));
    QA_CK(cudaMalloc(&dmn, d * 8));
    QA_CK(cudaMalloc(&dmx, d * 8));
    QA_CK(cudaMalloc(&dnan, d * 4));
    QA_CK(cudaMalloc(&dkept, d * 4));
    QA_CK(cudaMalloc(&dtam, d * 8));
    QA_CK(cudaMalloc(&dsel, d * sizeof(SelState)));
    QA_CK(cudaMalloc(&dhist, (size_t)kStatsChunk * 512 * 4));
    {
        const unsigned g = (unsigned)((d + kColBlock - 1) / kColBlock);
        colsum_kernel<<<g, kColBlock, 0, st>>>(x, n, d, ldx, dmu, dmn, dmx, dnan);
        QA_CK(cudaGetLastError());
        if (d % kStatsChunk == 1) {
            // the last 64-column block is one column wide: numpy's axis-0
            // reduction of an [n, 1] block runs along contiguous memory and
            // uses pairwise summation instead of the row-by-row order
            double s1 = 0.0;
            QA_CK(pairwise_sum(BlockView{x, ldx, d - 1, 1, 0.0, 0}, n, st, &s1));
            last_mu = s1 / (double)n;
            QA_CK(cudaMemcpyAsync(dmu + d - 1, &last_mu, 8, cudaMemcpyHostToDevice, st));
        }
        colvar_kernel<<<g, kColBlock, 0, st>>>(x, n, d, ldx, dmu, dsig);
        QA_CK(cudaGetLastError());
        if (d % kStatsChunk == 1) {
            double s2 = 0.0;
            QA_CK(pairwise_sum(BlockView{x, ldx, d - 1, 1, last_mu, 1}, n, st, &s2));
            last_sigma = std::sqrt(s2 / (double)n);
        }
    }
    // order statistics, one 64-column chunk at a time (64 KiB of histograms)
    for (int64_t j = 0; j < d; ++j) hsel[j] = SelState{{0u, 0u}, {klo, khi}};
    QA_CK(cudaMemcpyAsync(dsel, hsel.data(), d * sizeof(SelState), cudaMemcpyHostToDevice, st));
    {
        const unsigned rb = (unsigned)((n + kSelRowsPerCta - 1) / kSelRowsPerCta);
        for (int64_t c0 = 0; c0 < d; c0 += kStatsChunk) {
            const int nc = (int)std::min<int64_t>(kStatsChunk, d - c0);
            const size_t smem = (size_t)nc * 512 * 4;
            QA_CK(cudaFuncSetAttribute(radix_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
            for (int pass = 0; pass < 4; ++pass) {
                QA_CK(cudaMemsetAsync(dhist, 0, smem, st));
                radix_hist_kernel<<<rb, kSelThreads, smem, st>>>(x, n, c0, nc, ldx, dsel + c0, pass,
                                                                 dhist);
                radix_pick_kernel<<<(nc * 2 + 127) / 128, 128, 0, st>>>(dsel + c0, dhist, nc, pass);
                QA_CK(cudaGetLastError());
            }
        }
    }
    QA_CK(cudaMemsetAsync(dtam, 0, d * 8, st));
    QA_CK(cudaMemsetAsync(dkept, 0, d * 4, st));
    {
        dim3 g((unsigned)((n + kSelRowsPerCta - 1) / kSelRowsPerCta),
               (unsigned)std::min<int64_t>((d + kColBlock - 1) / kColBlock, 65535));
        tam_kernel<<<g, kSelThreads, 0, st>>>(x, n, d, ldx, dmu, dsel, dnan, dtam, dkept);
        QA_CK(cudaGetLastError());
    }
    QA_CK(cudaMemcpyAsync(mu, dmu, d * 8, cudaMemcpyDeviceToHost, st));
    QA_CK(cudaMemcpyAsync(sigma, dsig, d * 8, cudaMemcpyDeviceToHost, st));
    QA_CK(cudaMemcpyAsync(mn, dmn, d * 8, cudaMemcpyDeviceToHost, st));
    QA_CK(cudaMemcpyAsync(mx, dmx, d * 8, cudaMemcpyDeviceToHost, st));
    QA_CK(cudaMemcpyAsync(hsel.data(), dsel, d * sizeof(SelState), cudaMemcpyDeviceToHost, st));
    QA_CK(cudaMemcpyAsync(hnan.data(), dnan, d * 4, cudaMemcpyDeviceToHost, st));
    QA_CK(cudaMemcpyAsync(hkept.data(), dkept, d * 4, cudaMemcpyDeviceToHost, st));
    QA_CK(cudaMemcpyAsync(htam.data(), dtam, d * 8, cudaMemcpyDeviceToHost, st));
    QA_CK(cudaStreamSynchronize(st));
    if (d % kStatsChunk == 1) sigma[d - 1] = last_sigma;
    for (int64_t j = 0; j < d; ++j) {
        auto kf = [](uint32_t k) {
            const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
            float f;
            std::memcpy(&f, &u, 4);
            return (double)f;
        };
        qlo[j] = hnan[j] ? NAN : kf(hsel[j].prefix[0]);
        qhi[j] = hnan[j] ? NAN : kf(hsel[j].prefix[1]);
        if (hkept[j]) {
            std::memcpy(&tam[j], &htam[j], 8);
        } else {
            tam[j] = -INFINITY;
        }
    }
    // pooled statistics: numpy pairwise sums per 64-column block
    for (int pass = 0; pass < 2; ++pass) {
        const double shift = pass == 0 ? 0.0 : flat_sum / (double)(n * d);
        for (int64_t c0 = 0; c0 < d; c0 += kStatsChunk) {
            const int64_t c = std::min<int64_t>(kStatsChunk, d - c0);
            double sblk = 0.0;
            QA_CK(pairwise_sum(BlockView{x, ldx, c0, c, shift, pass}, n * c, st, &sblk));
            if (pass == 0)
                flat_sum += sblk;
            else
                pooled_var += sblk;
        }
    }
    *pooled_mu = flat_sum / (double)(n * d);
    *pooled_sigma = std::sqrt(pooled_var / (double)(n * d));
    e = cudaSuccess;
done:
#undef QA_CK
    cudaFree(dmu);
    cudaFree(dsig);
    cudaFree(dmn);
    cudaFree(dmx);
    cudaFree(dnan);
    cudaFree(dkept);
    cudaFree(dtam);
    cudaFree(dsel);
    cudaFree(dhist);
    return e;
}

}  // namespace qa
