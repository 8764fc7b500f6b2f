// qa_select.cu -- exact top-k maintenance between filter passes, final
// score materialisation and the cross-shard merge.
//
// Reference semantics (_core.pyx:301-330): the result for a query is the
// first keff entries of the full (score, id) lexicographic sort.  The filter
// pass only discards rows that provably cannot enter that prefix; this file
// turns the surviving candidates into the exact prefix: exact float64 scores
// (angular: one correctly rounded division + subtraction, _core.pyx:96),
// (score, id) order, truncation to k, and the next pass's threshold.
//
// select: one WARP per query.  The retained list T (sorted, <= k entries)
// lives in shared memory; candidates arrive in chunks of kChunk: they are
// scored exactly, entries already worse than T's k-th are dropped (warp
// ballot compaction), the rest are bitonic-sorted in shared memory and
// merged into T by merge path (each element's output rank = its own index +
// a binary-search count in the other list).
#include <cfloat>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "qa_common.cuh"
#include "qa_internal.h"

namespace qa {

namespace {

constexpr int kChunk = 256;  // candidates sorted per merge step
constexpr int kWarpsMax = 8;
// select_reg_kernel occupancy: 5 blocks of 8 warps per SM (<= 48 registers)
// measured best with the branch-free compare-exchange (6 spills more).
#ifndef QA_SEL_MINB
#define QA_SEL_MINB 5
#endif

__device__ __forceinline__ int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

template <typename T, typename Less>
__device__ void warp_bitonic_sort(T *buf, int P, Less less) {
    const int lane = threadIdx.x & 31;
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = lane; t < (P >> 1); t += 32) {
                const int i = 2 * t - (t & (stride - 1));
                const int j = i + stride;
                const bool up = ((i & size) == 0);
                T a = buf[i], b = buf[j];
                if (up ? less(b, a) : less(a, b)) {
                    buf[i] = b;
                    buf[j] = a;
                }
            }
            __syncwarp();
        }
    }
}

template <typename T, typename Less>
__device__ void block_bitonic_sort(T *buf, int P, Less less) {
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (P >> 1); t += blockDim.x) {
                const int i = 2 * t - (t & (stride - 1));
                const int j = i + stride;
                const bool up = ((i & size) == 0);
                T a = buf[i], b = buf[j];
                if (up ? less(b, a) : less(a, b)) {
                    buf[i] = b;
                    buf[j] = a;
                }
            }
            __syncthreads();
        }
    }
}

struct EntryLess {
    __device__ bool operator()(const Entry &a, const Entry &b) const { return entry_less(a, b); }
};

// number of entries of sorted list L[0, len) strictly less than x
__device__ __forceinline__ int count_less(const Entry *L, int len, const Entry &x) {
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (entry_less(L[mid], x))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

template <int M>
__device__ __forceinline__ Entry make_entry(Cand c, int32_t qq, float qn,
                                            const int32_t *__restrict__ db_sqnorm,
                                            const float *__restrict__ db_norm,
                                            const int32_t *__restrict__ row_ids) {
    Entry e;
    e.row = c.row;
    e.id = row_ids ? __ldg(row_ids + c.row) : c.row;
    if constexpr (M == kIP) {
        e.skey = skey_from_int((int32_t)(0u - (uint32_t)c.dot));
    } else if constexpr (M == kL2) {
        uint32_t s = (uint32_t)qq + (uint32_t)__ldg(db_sqnorm + c.row) - 2u * (uint32_t)c.dot;
        e.skey = skey_from_int((int32_t)s);
    } else {
        e.skey = skey_from_double(angular_score(c.dot, qn, __ldg(db_norm + c.row)));
    }
    return e;
}

// Next-pass threshold from the k-th retained entry (see qa_common.cuh).
template <int M>
__device__ __forceinline__ int32_t threshold_of(const Entry &e, int32_t qq, float qn) {
    if constexpr (M == kIP) {
        return (int32_t)(0u - (uint32_t)int_from_skey(e.skey));  // dot_k; ties may win on id
    } else if constexpr (M == kL2) {
        return (int32_t)((uint32_t)int_from_skey(e.skey) - (uint32_t)qq);  // l2_k - qq
    } else {
        // Rows with score <= score_k have c = dot/xn >= qn*(1 - score_k) - qn*2^-50
        // (two float64 roundings).  The float proxy float(dot)*rcp(xn) is
        // within 3*2^-24 relative of c; a 2^-20 relative band plus qn*2^-40
        // absolute covers both, so no such row is ever filtered out.
        const double c = (1.0 - double_from_skey(e.skey)) * (double)qn;
        const double p = c - fabs(c) * 0x1p-20 - (double)qn * 0x1p-40;
        return __float_as_int(__double2float_rd(p));
    }
}

template <int M>
__global__ void __launch_bounds__(kWarpsMax * 32) select_kernel(SelectArgs a, int kpad) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (q >= a.nq) return;
    const int32_t total = a.ccount[q];
    if (total == 0) return;  // nothing new: state and threshold unchanged
    Entry *T = reinterpret_cast<Entry *>(smem_raw) + (size_t)warp * (2 * kpad + kChunk);
    Entry *O = T + kpad;
    Entry *S = O + kpad;
    const int k = (int)a.k;
    const int m = (int)min((int64_t)total, a.cap);
    if (total > a.cap && lane == 0) {
        a.overflow[q] = 1;
        atomicExch(a.any_overflow, 1);
    }
    const int32_t qq = (M == kL2) ? a.q_sqnorm[q] : 0;
    const float qn = (M == kAngular) ? a.q_norm[q] : 1.0f;
    Entry *st = a.state + q * a.k;
    const Cand *cd = a.cand + q * a.cap;
    int cur = a.state_cnt[q];
    for (int i = lane; i < cur; i += 32) T[i] = st[i];
    __syncwarp();
    int nvalid = 0;
    for (int pos = 0; pos < m; pos += kChunk) {
        const int take = min(kChunk, m - pos);
        // score the chunk; drop entries that cannot beat the current k-th
        const bool full = (cur == k);
        Entry kth;
        if (full) kth = T[k - 1];
        int ns = 0;
        for (int base = 0; base < take; base += 32) {
            const int i = base + lane;
            Entry e;
            bool keep = false, valid = false;
            if (i < take) {
                const Cand c = cd[pos + i];
                if (c.row >= 0) {  // row -1: slot of a masked-dense pass, filtered out
                    valid = true;
                    e = make_entry<M>(c, qq, qn, a.db_sqnorm, a.db_norm, a.row_ids);
                    keep = !full || entry_less(e, kth);
                }
            }
            nvalid += __popc(__ballot_sync(0xffffffffu, valid));
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) S[ns + __popc(bal & ((1u << lane) - 1))] = e;
            ns += __popc(bal);
        }
        if (ns == 0) continue;
        const int P = next_pow2(max(ns, 2));
        for (int i = ns + lane; i < P; i += 32) {
            S[i].skey = ~0ull;
            S[i].id = INT32_MAX;
            S[i].row = -1;
        }
        __syncwarp();
        warp_bitonic_sort(S, P, EntryLess());
        // merge T[0, cur) and S[0, ns) -> O[0, newcur)
        const int newcur = min(k, cur + ns);
        for (int i = lane; i < cur; i += 32) {
            const int r = i + count_less(S, ns, T[i]);
            if (r < newcur) O[r] = T[i];
        }
        for (int i = lane; i < ns; i += 32) {
            const int r = i + count_less(T, cur, S[i]);
            if (r < newcur) O[r] = S[i];
        }
        __syncwarp();
        Entry *tmp = T;
        T = O;
        O = tmp;
        cur = newcur;
    }
    for (int i = lane; i < cur; i += 32) st[i] = T[i];
    if (lane == 0) {
        a.state_cnt[q] = cur;
        if (cur == k) a.thr[q] = threshold_of<M>(T[k - 1], qq, qn);
        if (a.cand_count) atomicAdd(a.cand_count, (unsigned long long)nvalid);
    }
}

// ------------------------------------------------ register select (k<=128) --
//
// The retained list T (<= 128 entries) and a chunk S of 128 candidates live in
// registers, 4 per lane, element index i = e*32 + lane.  S is bitonic-sorted
// (strides < 32 cross lanes by shuffles, 32/64 swap registers), reversed,
// and [T asc | S desc] -- a bitonic sequence of 256 -- is merged: one
// compare at stride 128 leaves the 128 smallest in T's registers, seven more
// stages sort them.  No shared memory, no barriers.
//
// Keys: IP / L2 scores are int32, so (score, id) packs into one u64; angular
// keeps the u64 float64 order key plus the id.
struct RKey64 {
    unsigned long long k;
};
struct RKey96 {
    unsigned long long k;
    int32_t id;
};

__device__ __forceinline__ bool rlt(const RKey64 &a, const RKey64 &b) { return a.k < b.k; }
__device__ __forceinline__ bool rlt(const RKey96 &a, const RKey96 &b) {
    // no short-circuit: predicates combine without branches
    return (a.k < b.k) | ((a.k == b.k) & (a.id < b.id));
}
// c ? a : b, field by field (compiles to SEL, no divergent branch)
__device__ __forceinline__ RKey64 rsel(bool c, const RKey64 &a, const RKey64 &b) {
    return RKey64{c ? a.k : b.k};
}
__device__ __forceinline__ RKey96 rsel(bool c, const RKey96 &a, const RKey96 &b) {
    return RKey96{c ? a.k : b.k, c ? a.id : b.id};
}
__device__ __forceinline__ RKey64 rshfl(const RKey64 &a, int m) {
    return RKey64{__shfl_xor_sync(0xffffffffu, a.k, m)};
}
__device__ __forceinline__ RKey96 rshfl(const RKey96 &a, int m) {
    return RKey96{__shfl_xor_sync(0xffffffffu, a.k, m), __shfl_xor_sync(0xffffffffu, a.id, m)};
}
__device__ __forceinline__ void rsentinel(RKey64 &a) { a.k = ~0ull; }
__device__ __forceinline__ void rsentinel(RKey96 &a) {
    a.k = ~0ull;
    a.id = INT32_MAX;
}

// Entry <-> register key
template <int M>
__device__ __forceinline__ void to_key(const Entry &e, RKey64 &r) {
    r.k = ((unsigned long long)(uint32_t)e.skey << 32) | (uint32_t)e.id;
}
template <int M>
__device__ __forceinline__ void to_key(const Entry &e, RKey96 &r) {
    r.k = e.skey;
    r.id = e.id;
}
__device__ __forceinline__ Entry from_key(const RKey64 &r) {
    Entry e;
    e.skey = r.k >> 32;
    e.id = (int32_t)(uint32_t)r.k;
    e.row = 0;
    return e;
}
__device__ __forceinline__ Entry from_key(const RKey96 &r) {
    Entry e;
    e.skey = r.k;
    e.id = r.id;
    e.row = 0;
    return e;
}

__device__ __forceinline__ RKey64 rbcast(const RKey64 &a, int src) {
    return RKey64{__shfl_sync(0xffffffffu, a.k, src)};
}
__device__ __forceinline__ RKey96 rbcast(const RKey96 &a, int src) {
    return RKey96{__shfl_sync(0xffffffffu, a.k, src), __shfl_sync(0xffffffffu, a.id, src)};
}

// element i of x[R] (i = e*32 + lane), broadcast to the whole warp
template <typename K, int R>
__device__ __forceinline__ K rget(const K (&x)[R], int i) {
    K v = x[0];
#pragma unroll
    for (int e = 1; e < R; ++e) v = rsel((i >> 5) == e, x[e], v);
    return rbcast(v, i & 31);
}

// one compare-exchange stage over x[R] (i = e*32 + lane) for (size, stride)
template <typename K, int R>
__device__ __forceinline__ void rstage(K (&x)[R], int size, int stride) {
    const int lane = threadIdx.x & 31;
    if (stride >= 32) {
        const int es = stride >> 5;
#pragma unroll
        for (int e = 0; e < R; ++e) {
            const int p = e ^ es;
            if (p > e && p < R) {
                const bool up = (((e * 32 + lane) & size) == 0);
                const bool sw = up ? rlt(x[p], x[e]) : rlt(x[e], x[p]);
                const K lo = rsel(sw, x[p], x[e]);
                const K hi = rsel(sw, x[e], x[p]);
                x[e] = lo;
                x[p] = hi;
            }
        }
    } else {
        const bool lower = (lane & stride) == 0;
#pragma unroll
        for (int e = 0; e < R; ++e) {
            const bool up = (((e * 32 + lane) & size) == 0);
            const K o = rshfl(x[e], stride);
            // the lower index of an ascending pair keeps the min
            const bool take = (lower == up) ? rlt(o, x[e]) : rlt(x[e], o);
            x[e] = rsel(take, o, x[e]);
        }
    }
}

template <typename K, int R>
__device__ __forceinline__ void rsort(K (&x)[R]) {
#pragma unroll
    for (int size = 2; size <= 32 * R; size <<= 1)
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) rstage(x, size, stride);
}

// S (sorted ascending, W = 32R) merged into T (sorted ascending, W): T keeps
// the W smallest of both, sorted.
template <typename K, int R>
__device__ __forceinline__ void rmerge(K (&t)[R], const K (&s)[R]) {
    // reverse S (i -> W-1-i): lane -> 31 - lane, e -> R-1-e
    K r[R];
#pragma unroll
    for (int e = 0; e < R; ++e) r[e] = rshfl(s[R - 1 - e], 31);
    // stride-W step of the bitonic merge: T keeps the W smallest
#pragma unroll
    for (int e = 0; e < R; ++e) t[e] = rsel(rlt(r[e], t[e]), r[e], t[e]);
    // t is bitonic now: finish the merge with strides W/2..1 (ascending
    // everywhere: size 2W)
#pragma unroll
    for (int stride = 16 * R; stride > 0; stride >>= 1) rstage(t, 64 * R, stride);
}

// wpq warps per query (1, 2, 4 or 8; a block = 8 warps): with few queries
// the candidates of one query are split over wpq warps (each keeps its own
// top-k -- only the query's first warp starts from the retained list), and
// the group's lists are merged through shared memory at the end.  One warp
// per query is latency-bound on its candidate stream when few warps are
// resident.
template <int M, typename K, int R>
__global__ void __launch_bounds__(256, QA_SEL_MINB) select_reg_kernel(SelectArgs a, int wpq) {
    constexpr int W = 32 * R;  // retained-list / chunk width (k <= W)
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wq = warp % wpq;  // this warp's part of its query
    const int64_t q = (int64_t)blockIdx.x * (8 / wpq) + warp / wpq;
    __shared__ K stage_all[8][160];
    K *stage = stage_all[warp];
    const bool active = q < a.nq && a.ccount[q] > 0;
    const int k = (int)a.k;
    K t[R];
#pragma unroll
    for (int e = 0; e < R; ++e) rsentinel(t[e]);
    int cur = 0;
    int32_t qq = 0;
    float qn = 1.0f;
    Entry *st = nullptr;
    if (active) {
        const int32_t total = a.ccount[q];
        const int m = (int)min((int64_t)total, a.cap);
        if (total > a.cap && lane == 0 && wq == 0) {
            a.overflow[q] = 1;
            atomicExch(a.any_overflow, 1);
        }
        qq = (M == kL2) ? a.q_sqnorm[q] : 0;
        qn = (M == kAngular) ? a.q_norm[q] : 1.0f;
        st = a.state + q * a.k;
        const Cand *cd = a.cand + q * a.cap;
        const int scur = a.state_cnt[q];
        cur = wq == 0 ? scur : 0;
#pragma unroll
        for (int e = 0; e < R; ++e) {
            const int i = e * 32 + lane;
            if (i < cur)
                to_key<M>(st[i], t[e]);
            else
                rsentinel(t[e]);
        }
        // every warp of the query filters against the retained k-th
        K kth;
        rsentinel(kth);
        if (scur == k) {
            Entry e = st[k - 1];
            to_key<M>(e, kth);
        }
        // Candidates are scored 32 at a time (the next 32 are loaded while
        // these are processed); those below the current k-th key are
        // compacted into this warp's smem stage, which is sorted and merged
        // whenever it holds 128 (and once at the end).
        int fill = 0;
        int nvalid = 0;
        const int stride = 32 * wpq;
        int pos = 32 * wq;
        Cand cn = (pos + lane < m) ? cd[pos + lane] : Cand{-1, 0};
        for (; pos < m; pos += stride) {
            const Cand c = cn;
            const int nx = pos + stride + lane;
            cn = (nx < m) ? cd[nx] : Cand{-1, 0};
            bool keep = false, valid = false;
            K key;
            if (c.row >= 0) {  // row -1: slot of a masked-dense pass, filtered out
                valid = true;
                const Entry en = make_entry<M>(c, qq, qn, a.db_sqnorm, a.db_norm, a.row_ids);
                to_key<M>(en, key);
                keep = rlt(key, kth);
            }
            nvalid += __popc(__ballot_sync(0xffffffffu, valid));
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) stage[fill + __popc(bal & ((1u << lane) - 1))] = key;
            fill += __popc(bal);
            const bool last = pos + stride >= m;
            while (fill >= W || (last && fill > 0)) {
                __syncwarp();
                const int ns = min(fill, W);
                K s[R];
#pragma unroll
                for (int e = 0; e < R; ++e) {
                    if (e * 32 + lane < ns)
                        s[e] = stage[e * 32 + lane];
                    else
                        rsentinel(s[e]);
                }
                __syncwarp();
                if (fill > W && lane < fill - W) stage[lane] = stage[W + lane];
                fill -= ns;
                __syncwarp();
                rsort(s);
                rmerge(t, s);
                cur = min(k, cur + ns);
                const K kk = rget(t, k - 1);
                kth = rsel(rlt(kk, kth), kk, kth);
            }
        }
        if (lane == 0 && a.cand_count) atomicAdd(a.cand_count, (unsigned long long)nvalid);
    }
    if (wpq > 1) {
        // merge the group's lists into its first warp: a pairwise tree
        // (log2 wpq levels; at each level warp wq merges warp wq + step's
        // list), not a chain -- the merges are serial shuffle networks
        __syncwarp();
#pragma unroll
        for (int e = 0; e < R; ++e) stage[e * 32 + lane] = t[e];
        if (lane == 0) reinterpret_cast<int *>(stage + W)[0] = cur;
        for (int step = 1; step < wpq; step <<= 1) {
            __syncthreads();  // this level's lists are written
            const bool merger = active && (wq % (2 * step)) == 0;
            if (merger) {
                const K *o = stage_all[warp + step];
                K s[R];
#pragma unroll
                for (int e = 0; e < R; ++e) s[e] = o[e * 32 + lane];
                rmerge(t, s);
                cur = min(k, cur + reinterpret_cast<const int *>(o + W)[0]);
            }
            __syncthreads();  // every read of this level is done
            if (merger && 2 * step < wpq) {
#pragma unroll
                for (int e = 0; e < R; ++e) stage[e * 32 + lane] = t[e];
                if (lane == 0) reinterpret_cast<int *>(stage + W)[0] = cur;
            }
        }
    }
    if (q >= a.nq || wq != 0) return;
    if (a.next_fill >= 0 && lane == 0) a.ccount_reset[q] = a.next_fill;
    if (active) {
#pragma unroll
        for (int e = 0; e < R; ++e) {
            const int i = e * 32 + lane;
            if (i < cur) st[i] = from_key(t[e]);
        }
        // threshold from the k-th entry
        if (cur == k) {
            const K v = rget(t, k - 1);
            if (lane == 0) a.thr[q] = threshold_of<M>(from_key(v), qq, qn);
        }
        if (lane == 0) a.state_cnt[q] = cur;
    }
    if (a.est_j > 0) {
        // fused threshold estimate (formerly estimate_kernel): the est_j-th
        // kept entry bounds the next pass; queries without candidates this
        // round keep their state and take it from memory
        const int j = (int)a.est_j;
        const int cnt = active ? cur : a.state_cnt[q];
        if (cnt < j) {
            if (lane == 0 && !a.est_combine) a.est[q] = ~0ull;
            return;
        }
        Entry e;
        if (active) {
            e = from_key(rget(t, j - 1));
        } else {
            e = a.state[q * a.k + j - 1];
            qq = (M == kL2) ? a.q_sqnorm[q] : 0;
            qn = (M == kAngular) ? a.q_norm[q] : 1.0f;
        }
        if (lane == 0) {
            a.thr[q] = threshold_of<M>(e, qq, qn);
            const unsigned long long prev = a.est[q];
            a.est[q] = (a.est_combine && prev != ~0ull && prev < e.skey) ? prev : e.skey;
        }
    }
}


// ------------------------------------------------- radix select (k<=128) --
//
// Large batches, integer scores (IP / L2): one warp per query.  The retained
// list and the round's surviving candidates are gathered as 64-bit keys
// (score key << 32 | id: the (score, id) order) into a shared-memory buffer
// U; whenever U fills, and once at the end, the k smallest keys are found by
// an MSB-first radix select (8-bit digits, a 256-bin warp histogram per pass,
// early exit once the boundary digit holds exactly the remaining rank) and
// compacted -- no sorting until the end, when the k winners are sorted once
// with the 32*R-wide register network.  The merge-per-chunk select above
// sorts every 128 candidates; with 1024 dense candidates per query (round
// 0) that was ~13k instructions per warp, this is ~3k.
constexpr int kRadixWarps = 4;
constexpr int kRadixCap = 1280;  // keys per warp buffer (k + chunks of candidates)

// the k smallest of U[0, nu) (unique keys) moved to U[0, k); returns the
// largest kept key (the k-th smallest)
__device__ unsigned long long radix_keep_k(unsigned long long *U, int nu, int k, int *hist) {
    const int lane = threadIdx.x & 31;
    // bits above the highest one where the keys differ are common to all:
    // the radix starts at that byte (scores of one query share their top bits)
    unsigned long long kmin = ~0ull, kmax0 = 0;
    for (int i = lane; i < nu; i += 32) {
        const unsigned long long key = U[i];
        kmin = key < kmin ? key : kmin;
        kmax0 = key > kmax0 ? key : kmax0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a0 = __shfl_xor_sync(0xffffffffu, kmin, o);
        const unsigned long long b0 = __shfl_xor_sync(0xffffffffu, kmax0, o);
        kmin = a0 < kmin ? a0 : kmin;
        kmax0 = b0 > kmax0 ? b0 : kmax0;
    }
    const int hi = 63 - __clzll((long long)(kmin ^ kmax0) | 1ll);  // highest differing bit
    int shift0 = (hi / 8) * 8;
    unsigned long long mask = shift0 == 56 ? 0ull : ~0ull << (shift0 + 8);
    unsigned long long prefix = kmin & mask;
    int want = k;  // rank still to place among keys matching prefix
    for (int shift = shift0; shift >= 0; shift -= 8) {
#pragma unroll
        for (int b = 0; b < 8; ++b) hist[lane * 8 + b] = 0;
        __syncwarp();
        for (int base = 0; base < nu; base += 32) {
            const int i = base + lane;
            const unsigned long long key = i < nu ? U[i] : 0ull;
            const bool in = i < nu && (key & mask) == prefix;
            const unsigned act = __ballot_sync(0xffffffffu, in);
            if (in) {
                const int dg = (int)((key >> shift) & 255);
#if defined(QA_RADIX_MATCH) && QA_RADIX_MATCH
                // one shared atomic per distinct digit of the warp
                const unsigned peers = __match_any_sync(act, dg);
                if (lane == __ffs(peers) - 1) atomicAdd(hist + dg, __popc(peers));
#else
                (void)act;
                atomicAdd(hist + dg, 1);
#endif
            }
        }
        __syncwarp();
        int h[8], sum = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            h[b] = hist[lane * 8 + b];
            sum += h[b];
        }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int excl = incl - sum;
        // the lane whose bins hold rank `want`
        const unsigned own = __ballot_sync(0xffffffffu, excl < want && incl >= want);
        const int src = __ffs(own) - 1;
        int d = 0, below = 0, eq = 0;
        if (lane == src) {
            int c = excl;
            bool found = false;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                if (!found && c + h[b] >= want) {
                    found = true;
                    d = lane * 8 + b;
                    below = c;
                    eq = h[b];
                }
                c += h[b];
            }
        }
        d = __shfl_sync(0xffffffffu, d, src);
        below = __shfl_sync(0xffffffffu, below, src);
        eq = __shfl_sync(0xffffffffu, eq, src);
        want -= below;
        prefix |= (unsigned long long)d << shift;
        mask |= 255ull << shift;
        if (eq == want) break;  // every key with this prefix is kept
    }
    const unsigned long long T = prefix | ~mask;  // keep keys <= T: exactly k of them
    // in-place ballot compaction (writes never pass reads); the largest kept
    // key is the k-th smallest
    int w = 0;
    unsigned long long kmax = 0;
    for (int base = 0; base < nu; base += 32) {
        const int i = base + lane;
        const unsigned long long key = i < nu ? U[i] : ~0ull;
        const bool keep = i < nu && key <= T;
        const unsigned bb = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) {
            U[w + __popc(bb & ((1u << lane) - 1))] = key;
            kmax = key > kmax ? key : kmax;
        }
        w += __popc(bb);
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, kmax, o);
        kmax = v > kmax ? v : kmax;
    }
    return kmax;
}

template <int M, int R>
__global__ void __launch_bounds__(kRadixWarps * 32) select_radix_kernel(SelectArgs a) {
    static_assert(M == kIP || M == kL2, "integer scores");
    __shared__ unsigned long long U_all[kRadixWarps][kRadixCap];
    __shared__ int hist_all[kRadixWarps][256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * kRadixWarps + warp;
    if (q >= a.nq) return;  // warp-level work only: no block barriers below
    unsigned long long *U = U_all[warp];
    int *hist = hist_all[warp];
    const int k = (int)a.k;
    const int32_t total = a.ccount[q];
    Entry *st = a.state + q * a.k;
    const int scur = a.state_cnt[q];
    const int32_t qq = (M == kL2) ? a.q_sqnorm[q] : 0;
    int nu = 0, cur = scur;
    if (total > 0) {
        const int m = (int)min((int64_t)total, a.cap);
        if (total > a.cap && lane == 0) {
            a.overflow[q] = 1;
            atomicExch(a.any_overflow, 1);
        }
        for (int i = lane; i < scur; i += 32) {
            RKey64 r;
            to_key<M>(st[i], r);
            U[i] = r.k;
        }
        nu = scur;
        unsigned long long kth = scur == k ? U[k - 1] : ~0ull;  // the state is sorted
        __syncwarp();
        const Cand *cd = a.cand + q * a.cap;
        int nvalid = 0;
        // kIlp candidates per lane per step: their dependent gathers (norm,
        // id of the row) are all in flight before any is used -- the loop is
        // bound by memory latency, not instructions
#ifndef QA_RADIX_ILP
#define QA_RADIX_ILP 4
#endif
        constexpr int kIlp = QA_RADIX_ILP;
        for (int pos = 0; pos < m; pos += 32 * kIlp) {
            Cand c[kIlp];
#pragma unroll
            for (int u = 0; u < kIlp; ++u) {
                const int i = pos + u * 32 + lane;
                c[u] = i < m ? cd[i] : Cand{-1, 0};
            }
            int32_t xx[kIlp], id[kIlp];
#pragma unroll
            for (int u = 0; u < kIlp; ++u) {
                const int32_t row = c[u].row >= 0 ? c[u].row : 0;
                xx[u] = (M == kL2) ? __ldg(a.db_sqnorm + row) : 0;
                id[u] = a.row_ids ? __ldg(a.row_ids + row) : row;
            }
#pragma unroll
            for (int u = 0; u < kIlp; ++u) {
                const bool valid = c[u].row >= 0;
                unsigned long long key = 0;
                if (valid) {
                    int32_t sc;
                    if constexpr (M == kIP)
                        sc = (int32_t)(0u - (uint32_t)c[u].dot);
                    else
                        sc = (int32_t)((uint32_t)qq + (uint32_t)xx[u] - 2u * (uint32_t)c[u].dot);
                    key = (skey_from_int(sc) << 32) | (uint32_t)id[u];
                }
                const bool keep = valid && key < kth;
                nvalid += __popc(__ballot_sync(0xffffffffu, valid));
                const unsigned bb = __ballot_sync(0xffffffffu, keep);
                if (keep) U[nu + __popc(bb & ((1u << lane) - 1))] = key;
                nu += __popc(bb);
            }
            __syncwarp();
            if (nu + 32 * kIlp > kRadixCap && nu > k) {
                kth = radix_keep_k(U, nu, k, hist);
                nu = k;
            }
        }
        if (nu > k) {
            radix_keep_k(U, nu, k, hist);
            nu = k;
        }
        cur = nu;
        if (lane == 0 && a.cand_count) atomicAdd(a.cand_count, (unsigned long long)nvalid);
    }
    if (a.next_fill >= 0 && lane == 0) a.ccount_reset[q] = a.next_fill;
    RKey64 t[R];
    if (total > 0) {
        // the kept keys, sorted once
#pragma unroll
        for (int e = 0; e < R; ++e) {
            const int i = e * 32 + lane;
            t[e].k = i < cur ? U[i] : ~0ull;
        }
        rsort(t);
#pragma unroll
        for (int e = 0; e < R; ++e) {
            const int i = e * 32 + lane;
            if (i < cur) st[i] = from_key(t[e]);
        }
        if (cur == k) {
            const RKey64 v = rget(t, k - 1);
            if (lane == 0) a.thr[q] = threshold_of<M>(from_key(v), qq, 1.0f);
        }
        if (lane == 0) a.state_cnt[q] = cur;
    }
    if (a.est_j > 0) {
        // fused threshold estimate (see select_reg_kernel)
        const int j = (int)a.est_j;
        const int cnt = total > 0 ? cur : scur;
        if (cnt < j) {
            if (lane == 0 && !a.est_combine) a.est[q] = ~0ull;
            return;
        }
        const Entry e = total > 0 ? from_key(rget(t, j - 1)) : a.state[q * a.k + j - 1];
        if (lane == 0) {
            a.thr[q] = threshold_of<M>(e, qq, 1.0f);
            const unsigned long long prev = a.est[q];
            a.est[q] = (a.est_combine && prev != ~0ull && prev < e.skey) ? prev : e.skey;
        }
    }
}

// One CTA (4 warps) per query: the candidate gathers, the histogram passes
// and the compaction of the radix select above spread over 128 threads; the
// final 32R-wide sort and the state update stay with warp 0.  One warp per
// query left 1024 warps on 148 SMs, each a serial chain of dependent global
// loads and shared-memory passes (40 us per 1024-query batch of cfg2, as long
// as a fifth of the filter pass it follows).
#ifndef QA_RB_THREADS
#define QA_RB_THREADS 128
#endif
constexpr int kRbThreads = QA_RB_THREADS;
constexpr int kRbWarps = kRbThreads / 32;
constexpr int kRbCap = 2048;  // keys per query buffer

// block-wide: the k smallest of U[0, nu) (unique keys) moved to U[0, k) in
// any order; returns an upper bound T of the k-th smallest with exactly k
// keys <= T.  All threads call it; `red` is a 256-int scratch, `ctl` 8 ints.
__device__ unsigned long long radix_keep_k_block(unsigned long long *U, int nu, int k, int *hist,
                                                 unsigned long long *red64, int *ctl) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long kmin = ~0ull, kmax0 = 0;
    for (int i = tid; i < nu; i += kRbThreads) {
        const unsigned long long key = U[i];
        kmin = key < kmin ? key : kmin;
        kmax0 = key > kmax0 ? key : kmax0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a0 = __shfl_xor_sync(0xffffffffu, kmin, o);
        const unsigned long long b0 = __shfl_xor_sync(0xffffffffu, kmax0, o);
        kmin = a0 < kmin ? a0 : kmin;
        kmax0 = b0 > kmax0 ? b0 : kmax0;
    }
    if (lane == 0) {
        red64[warp] = kmin;
        red64[kRbWarps + warp] = kmax0;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < kRbThreads / 32; ++w) {
        kmin = red64[w] < kmin ? red64[w] : kmin;
        kmax0 = red64[kRbWarps + w] > kmax0 ? red64[kRbWarps + w] : kmax0;
    }
    const int hi = 63 - __clzll((long long)(kmin ^ kmax0) | 1ll);  // highest differing bit
    const int shift0 = (hi / 8) * 8;
    unsigned long long mask = shift0 == 56 ? 0ull : ~0ull << (shift0 + 8);
    unsigned long long prefix = kmin & mask;
    int want = k;  // rank still to place among keys matching prefix
    for (int shift = shift0; shift >= 0; shift -= 8) {
        for (int b = tid; b < 256; b += kRbThreads) hist[b] = 0;
        __syncthreads();
        for (int i = tid; i < nu; i += kRbThreads) {
            const unsigned long long key = U[i];
            if ((key & mask) == prefix) atomicAdd(hist + (int)((key >> shift) & 255), 1);
        }
        __syncthreads();
        if (warp == 0) {
            int h[8], sum = 0;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                h[b] = hist[lane * 8 + b];
                sum += h[b];
            }
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const int excl = incl - sum;
            if (excl < want && incl >= want) {  // the lane whose bins hold rank `want`
                int c = excl;
                bool found = false;
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    if (!found && c + h[b] >= want) {
                        found = true;
                        ctl[0] = lane * 8 + b;
                        ctl[1] = c;
                        ctl[2] = h[b];
                    }
                    c += h[b];
                }
            }
        }
        __syncthreads();
        const int d = ctl[0], below = ctl[1], eq = ctl[2];
        want -= below;
        prefix |= (unsigned long long)d << shift;
        mask |= 255ull << shift;
        __syncthreads();  // ctl and hist are rewritten by the next pass
        if (eq == want) break;  // every key with this prefix is kept
    }
    const unsigned long long T = prefix | ~mask;  // keep keys <= T: exactly k of them
    // every thread reads its keys, then (after a barrier) the kept ones are
    // written back through a shared counter (the order does not matter)
    constexpr int kPer = kRbCap / kRbThreads;
    unsigned long long mine[kPer];
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
        const int i = e * kRbThreads + tid;
        mine[e] = i < nu ? U[i] : ~0ull;
    }
    if (tid == 0) ctl[4] = 0;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
        const int i = e * kRbThreads + tid;
        const bool keep = i < nu && mine[e] <= T;
        const unsigned bb = __ballot_sync(0xffffffffu, keep);
        int base = 0;
        if (lane == 0 && bb) base = atomicAdd(ctl + 4, __popc(bb));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) U[base + __popc(bb & ((1u << lane) - 1))] = mine[e];
    }
    __syncthreads();
    return T;
}

template <int M, int R>
__global__ void __launch_bounds__(kRbThreads) select_radix_block_kernel(SelectArgs a) {
    static_assert(M == kIP || M == kL2, "integer scores");
    __shared__ unsigned long long U[kRbCap];
    __shared__ int hist[256];
    __shared__ unsigned long long red64[2 * kRbWarps];
    __shared__ int ctl[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t q = blockIdx.x;
    const int k = (int)a.k;
    const int32_t total = a.ccount[q];
    Entry *st = a.state + q * a.k;
    const int scur = a.state_cnt[q];
    const int32_t qq = (M == kL2) ? a.q_sqnorm[q] : 0;
    int cur = scur;
    if (total > 0) {
        const int m = (int)min((int64_t)total, a.cap);
        if (total > a.cap && tid == 0) {
            a.overflow[q] = 1;
            atomicExch(a.any_overflow, 1);
        }
        for (int i = tid; i < scur; i += kRbThreads) {
            RKey64 r;
            to_key<M>(st[i], r);
            U[i] = r.k;
        }
        if (tid == 0) ctl[5] = scur;  // keys in U
        if (tid == 0) ctl[6] = 0;     // valid candidates seen
        __syncthreads();
        unsigned long long kth = scur == k ? U[k - 1] : ~0ull;  // the state is sorted
        const Cand *cd = a.cand + q * a.cap;
        constexpr int kIlp = 4;
        int nvalid = 0;
        for (int pos = 0; pos < m;) {
            // a round gathers what the buffer can take on top of its keys
            int nu = ctl[5];
            const int room = kRbCap - nu;
            const int end = min(m, pos + room);
            __syncthreads();  // ctl[5] read by everyone before it moves
            for (int p0 = pos; p0 < end; p0 += kRbThreads * kIlp) {
                Cand c[kIlp];
#pragma unroll
                for (int u = 0; u < kIlp; ++u) {
                    const int i = p0 + u * kRbThreads + tid;
                    c[u] = i < end ? cd[i] : Cand{-1, 0};
                }
                int32_t xx[kIlp], id[kIlp];
#pragma unroll
                for (int u = 0; u < kIlp; ++u) {
                    const int32_t row = c[u].row >= 0 ? c[u].row : 0;
                    xx[u] = (M == kL2) ? __ldg(a.db_sqnorm + row) : 0;
                    id[u] = a.row_ids ? __ldg(a.row_ids + row) : row;
                }
#pragma unroll
                for (int u = 0; u < kIlp; ++u) {
                    const bool valid = c[u].row >= 0;
                    unsigned long long key = 0;
                    if (valid) {
                        int32_t sc;
                        if constexpr (M == kIP)
                            sc = (int32_t)(0u - (uint32_t)c[u].dot);
                        else
                            sc = (int32_t)((uint32_t)qq + (uint32_t)xx[u] - 2u * (uint32_t)c[u].dot);
                        key = (skey_from_int(sc) << 32) | (uint32_t)id[u];
                    }
                    const bool keep = valid && key <= kth;
                    nvalid += valid ? 1 : 0;
                    const unsigned bb = __ballot_sync(0xffffffffu, keep);
                    int base = 0;
                    if (lane == 0 && bb) base = atomicAdd(ctl + 5, __popc(bb));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (keep) U[base + __popc(bb & ((1u << lane) - 1))] = key;
                }
            }
            pos = end;
            __syncthreads();
            nu = ctl[5];
            if (nu > k) {
                kth = radix_keep_k_block(U, nu, k, hist, red64, ctl);
                if (tid == 0) ctl[5] = k;
                __syncthreads();
            }
        }
        cur = min(ctl[5], k);
        // valid-candidate count (statistics)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nvalid += __shfl_xor_sync(0xffffffffu, nvalid, o);
        if (lane == 0 && a.cand_count && nvalid) atomicAdd(a.cand_count, (unsigned long long)nvalid);
    }
    if (warp != 0) return;  // the sort and the state update: one warp
    if (a.next_fill >= 0 && lane == 0) a.ccount_reset[q] = a.next_fill;
    RKey64 t[R];
    if (total > 0) {
#pragma unroll
        for (int e = 0; e < R; ++e) {
            const int i = e * 32 + lane;
            t[e].k = i < cur ? U[i] : ~0ull;
        }
        rsort(t);
#pragma unroll
        for (int e = 0; e < R; ++e) {
            const int i = e * 32 + lane;
            if (i < cur) st[i] = from_key(t[e]);
        }
        if (cur == k) {
            const RKey64 v = rget(t, k - 1);
            if (lane == 0) a.thr[q] = threshold_of<M>(from_key(v), qq, 1.0f);
        }
        if (lane == 0) a.state_cnt[q] = cur;
    }
    if (a.est_j > 0) {
        // fused threshold estimate (see select_reg_kernel)
        const int j = (int)a.est_j;
        const int cnt = total > 0 ? cur : scur;
        if (cnt < j) {
            if (lane == 0 && !a.est_combine) a.est[q] = ~0ull;
            return;
        }
        const Entry e = total > 0 ? from_key(rget(t, j - 1)) : a.state[q * a.k + j - 1];
        if (lane == 0) {
            a.thr[q] = threshold_of<M>(e, qq, 1.0f);
            const unsigned long long prev = a.est[q];
            a.est[q] = (a.est_combine && prev != ~0ull && prev < e.skey) ? prev : e.skey;
        }
    }
}

__global__ void reset_kernel(int32_t *p, int64_t n, int32_t v) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void init_state_kernel(int32_t *state_cnt, int32_t *thr, int64_t nq,
                                  int32_t pass_all, int32_t *ovf, int32_t *flags,
                                  int32_t *ccount = nullptr, int32_t fill0 = 0,
                                  unsigned *sched = nullptr, int nsched = 0) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (sched && i < nsched) sched[i] = 0;
    if (i < nq) {
        state_cnt[i] = 0;
        thr[i] = pass_all;
        if (ovf) ovf[i] = 0;
        if (ccount) ccount[i] = fill0;
    }
    if (flags && i < 16) flags[i] = 0;
}

template <int M>
__global__ void finalize_kernel(const Entry *__restrict__ state, int64_t nq, int64_t k,
                                int64_t keff, int64_t id_offset, double *__restrict__ out_scores,
                                int32_t *__restrict__ out_ids, const int32_t *__restrict__ state_cnt,
                                const unsigned long long *__restrict__ est,
                                int32_t *__restrict__ redo, int32_t *__restrict__ any_redo) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nq * keff) return;
    int64_t q = t / keff, j = t - q * keff;
    if (est && j == 0) {
        // the estimate check (see check_estimate_kernel), fused
        const unsigned long long ev = est[q];
        if (ev != ~0ull && !(state_cnt[q] >= k && state[q * k + k - 1].skey <= ev)) {
            redo[q] = 1;
            atomicExch(any_redo, 1);
        }
    }
    Entry e = state[q * k + j];
    double s;
    if constexpr (M == kIP) {
        const int32_t v = int_from_skey(e.skey);  // = -dot
        s = v == 0 ? -0.0 : (double)v;            // -(double)0 is -0.0 in _core.pyx:95
    } else if constexpr (M == kL2) {
        s = (double)int_from_skey(e.skey);
    } else {
        s = double_from_skey(e.skey);
    }
    out_scores[t] = s;
    out_ids[t] = (int32_t)(e.id + id_offset);
}

struct MEntry {
    unsigned long long skey;
    int32_t id;
    int32_t pad;
    double score;
};
struct MEntryLess {
    __device__ bool operator()(const MEntry &a, const MEntry &b) const {
        return a.skey < b.skey || (a.skey == b.skey && a.id < b.id);
    }
};

__global__ void __launch_bounds__(256) merge_kernel(const double *__restrict__ in_scores,
                                                    const int32_t *__restrict__ in_ids, int64_t G,
                                                    int64_t nq, int64_t kin, int64_t k,
                                                    double *__restrict__ out_scores,
                                                    int32_t *__restrict__ out_ids, int sz) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MEntry *buf = reinterpret_cast<MEntry *>(smem_raw);
    const int64_t q = blockIdx.x;
    if (q >= nq) return;
    int cur = 0;
    for (int64_t g = 0; g < G; ++g) {
        const double *sg = in_scores + (g * nq + q) * kin;
        const int32_t *ig = in_ids + (g * nq + q) * kin;
        int64_t pos = 0;
        while (pos < kin) {
            const int take = (int)min(kin - pos, (int64_t)(sz - cur));
            for (int i = threadIdx.x; i < take; i += blockDim.x) {
                MEntry e;
                e.score = sg[pos + i];
                e.skey = skey_from_double(e.score + 0.0);  // -0.0 ties +0.0 (float64 ==)
                e.id = ig[pos + i];
                e.pad = 0;
                buf[cur + i] = e;
            }
            const int tot = cur + take;
            const int P = next_pow2(tot);
            for (int i = tot + threadIdx.x; i < P; i += blockDim.x) {
                buf[i].skey = ~0ull;
                buf[i].id = INT32_MAX;
            }
            __syncthreads();
            block_bitonic_sort(buf, P, MEntryLess());
            cur = (int)min((int64_t)tot, k);
            pos += take;
        }
    }
    for (int i = threadIdx.x; i < cur; i += blockDim.x) {
        out_scores[q * k + i] = buf[i].score;
        out_ids[q * k + i] = buf[i].id;
    }
}

// Large k: merge two per-query sorted lists A [nq, la] and B [nq, lb] (score,
// id order) into the first k of their union, by merge path: an element's
// output rank is its own index plus the count of the other list's elements
// before it (A first on equal keys, so padding duplicates never collide).
__device__ __forceinline__ bool mkey_less(double sa, int32_t ia, double sb, int32_t ib) {
    const unsigned long long ka = skey_from_double(sa + 0.0), kb = skey_from_double(sb + 0.0);
    return ka < kb || (ka == kb && ia < ib);
}

__global__ void merge_pair_kernel(const double *__restrict__ as, const int32_t *__restrict__ ai,
                                  int64_t la, int64_t lda, const double *__restrict__ bs,
                                  const int32_t *__restrict__ bi, int64_t lb, int64_t ldb,
                                  int64_t k, double *__restrict__ os, int32_t *__restrict__ oi,
                                  int64_t ldo) {
    const int64_t q = blockIdx.y;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= la + lb) return;
    const double *A = as + q * lda, *B = bs + q * ldb;
    const int32_t *Ai = ai + q * lda, *Bi = bi + q * ldb;
    double x;
    int32_t xi;
    int64_t r;
    if (t < la) {
        x = A[t];
        xi = Ai[t];
        int64_t lo = 0, hi = lb;  // #{B < x}
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (mkey_less(B[mid], Bi[mid], x, xi)) lo = mid + 1; else hi = mid;
        }
        r = t + lo;
    } else {
        const int64_t j = t - la;
        x = B[j];
        xi = Bi[j];
        int64_t lo = 0, hi = la;  // #{A <= x}
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (!mkey_less(x, xi, A[mid], Ai[mid])) lo = mid + 1; else hi = mid;
        }
        r = j + lo;
    }
    if (r < k) {
        os[q * ldo + r] = x;
        oi[q * ldo + r] = xi;
    }
}


// ------------------------------------------------------------ repair --
//
// Device-side recompute of the queries a search flagged (candidate list
// overflow or a failed threshold-estimate check; flag[q] != 0), so that an
// asynchronous search needs no host round trip.  Two launches, both cheap
// when nothing is flagged:
//   compact   flagged query list + count (one CTA);
//   partial   work items (flagged query f < min(count, kRepMaxQ), row part p
//             of P): every row of the part is scored exactly (dp4a int32
//             dots, the float64 scores of make_entry) and a sorted top-keff
//             kept in shared memory; the partial list goes to scratch, and
//             the LAST part to finish for f merges the P lists (merge-path
//             levels, in scratch) into the query's output row.  Flagged
//             queries beyond kRepMaxQ are scanned whole by one CTA each
//             (pathological inputs only: slow, still exact).
// Exact by construction: every row of a flagged query is scored.
constexpr int kRepChunk = 1024;
constexpr int kRepThreads = 256;
constexpr int kRepMaxQ = 64;       // flagged queries repaired part-parallel
constexpr int kRepMaxParts = 128;

__device__ __forceinline__ int32_t rep_dot(const int8_t *__restrict__ x, const int8_t *__restrict__ q,
                                           int64_t ld) {
    const int4 *x4 = reinterpret_cast<const int4 *>(x);
    const int4 *q4 = reinterpret_cast<const int4 *>(q);
    int32_t acc = 0;
    for (int64_t w = 0; w < (ld >> 4); ++w) {
        const int4 a = __ldg(x4 + w), b = __ldg(q4 + w);
        acc = __dp4a(a.x, b.x, acc);
        acc = __dp4a(a.y, b.y, acc);
        acc = __dp4a(a.z, b.z, acc);
        acc = __dp4a(a.w, b.w, acc);
    }
    return acc;
}

int rep_parts(int64_t n) {
    int64_t P = n / 8192;
    if (P < 1) P = 1;
    if (P > kRepMaxParts) P = kRepMaxParts;
    return (int)P;
}

struct RepLayout {
    int32_t *flist, *count, *done;
    double *ps;      // [kRepMaxQ][P][keff] partial scores, then merge levels
    int32_t *pi;
    double *ms;      // [kRepMaxQ][P/2 + 1][keff] merge ping-pong
    int32_t *mi;
};

__host__ __device__ inline RepLayout rep_layout(void *scratch, int64_t nq, int64_t keff, int P) {
    RepLayout L;
    char *c = (char *)scratch;
    auto take = [&](size_t b) {
        char *r = c;
        c += (b + 255) / 256 * 256;
        return r;
    };
    L.flist = (int32_t *)take((size_t)nq * 4);
    L.count = (int32_t *)take(8);
    L.done = (int32_t *)take((size_t)kRepMaxQ * 4);
    const size_t lists = (size_t)kRepMaxQ * P * keff, half = (size_t)kRepMaxQ * (P / 2 + 1) * keff;
    L.ps = (double *)take(lists * 8);
    L.pi = (int32_t *)take(lists * 4);
    L.ms = (double *)take(half * 8);
    L.mi = (int32_t *)take(half * 4);
    return L;
}

__global__ void __launch_bounds__(1024) repair_compact_kernel(const int32_t *__restrict__ flag,
                                                              int64_t nq, RepLayout L) {
    __shared__ int base_s;
    __shared__ int warp_cnt[32];
    if (threadIdx.x == 0) base_s = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t c0 = 0; c0 < nq; c0 += 1024) {
        const int64_t i = c0 + threadIdx.x;
        const bool f = i < nq && flag[i] != 0;
        const unsigned b = __ballot_sync(0xffffffffu, f);
        if (lane == 0) warp_cnt[warp] = __popc(b);
        __syncthreads();
        int before = 0;
        for (int w = 0; w < warp; ++w) before += warp_cnt[w];
        if (f) L.flist[base_s + before + __popc(b & ((1u << lane) - 1))] = (int32_t)i;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < 32; ++w) tot += warp_cnt[w];
            base_s += tot;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *L.count = base_s;
    for (int i = threadIdx.x; i < kRepMaxQ; i += blockDim.x) L.done[i] = 0;
}

// top-keff of query q over rows [lo, hi) into state (shared memory); returns
// the number kept.  Block-wide (all threads).
template <int M>
__device__ int rep_scan_rows(const RepairArgs &r, int64_t q, int64_t lo, int64_t hi, Entry *state,
                             Entry *buf, Entry *tmp, int *buf_n) {
    const int keff = (int)r.keff;
    const int8_t *qrow = r.q + q * r.ld;
    const int32_t qq = (M == kL2) ? r.q_sqnorm[q] : 0;
    const float qn = (M == kAngular) ? r.q_norm[q] : 1.0f;
    int cnt = 0;
    for (int64_t c0 = lo; c0 < hi; c0 += kRepChunk) {
        if (threadIdx.x == 0) *buf_n = 0;
        __syncthreads();
        const bool full = cnt == keff;
        const Entry kth = full ? state[keff - 1] : Entry{~0ull, INT32_MAX, -1};
        for (int i = threadIdx.x; i < kRepChunk && c0 + i < hi; i += blockDim.x) {
            const int32_t row = (int32_t)(c0 + i);
            const int32_t dot = rep_dot(r.db + (int64_t)row * r.ld, qrow, r.ld);
            Entry e;
            e.row = row;
            e.id = r.row_ids ? __ldg(r.row_ids + row) : row;
            if constexpr (M == kIP) {
                e.skey = skey_from_int((int32_t)(0u - (uint32_t)dot));
            } else if constexpr (M == kL2) {
                e.skey = skey_from_int(
                    (int32_t)((uint32_t)qq + (uint32_t)__ldg(r.db_sqnorm + row) - 2u * (uint32_t)dot));
            } else {
                e.skey = skey_from_double(angular_score(dot, qn, __ldg(r.db_norm + row)));
            }
            if (!full || entry_less(e, kth)) buf[atomicAdd(buf_n, 1)] = e;
        }
        __syncthreads();
        const int ns = *buf_n;
        if (ns == 0) continue;
        int P = 2;
        while (P < ns) P <<= 1;
        for (int i = ns + threadIdx.x; i < P; i += blockDim.x) buf[i] = Entry{~0ull, INT32_MAX, -1};
        __syncthreads();
        block_bitonic_sort(buf, P, EntryLess());
        const int newcnt = min(keff, cnt + ns);  // merge state + buf (ids unique)
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const int rk = i + count_less(buf, ns, state[i]);
            if (rk < newcnt) tmp[rk] = state[i];
        }
        for (int i = threadIdx.x; i < ns; i += blockDim.x) {
            const int rk = i + count_less(state, cnt, buf[i]);
            if (rk < newcnt) tmp[rk] = buf[i];
        }
        __syncthreads();
        for (int i = threadIdx.x; i < newcnt; i += blockDim.x) state[i] = tmp[i];
        cnt = newcnt;
        __syncthreads();
    }
    return cnt;
}

template <int M>
__device__ __forceinline__ double rep_score(unsigned long long k) {
    if constexpr (M == kIP) {
        const int32_t v = int_from_skey(k);
        return v == 0 ? -0.0 : (double)v;  // -(double)0 is -0.0 in _core.pyx:95
    } else if constexpr (M == kL2) {
        return (double)int_from_skey(k);
    } else {
        return double_from_skey(k);
    }
}

template <int M>
__global__ void __launch_bounds__(kRepThreads) repair_kernel(RepairArgs r, RepLayout L, int P) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int keff = (int)r.keff;
    Entry *state = reinterpret_cast<Entry *>(smem_raw);   // [keff]
    Entry *buf = state + keff;                             // [kRepChunk]
    Entry *tmp = buf + kRepChunk;                          // [keff]
    __shared__ int buf_n, last_s;
    const int count = *L.count;
    const int fast = min(count, kRepMaxQ);
    const int64_t items = (int64_t)fast * P + (count - fast);
    for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
        if (w < (int64_t)fast * P) {
            // part p of flagged query f
            const int f = (int)(w / P), p = (int)(w % P);
            const int64_t q = L.flist[f];
            const int64_t lo = r.n * p / P, hi = r.n * (p + 1) / P;
            const int cnt = rep_scan_rows<M>(r, q, lo, hi, state, buf, tmp, &buf_n);
            double *os = L.ps + ((int64_t)f * P + p) * keff;
            int32_t *oi = L.pi + ((int64_t)f * P + p) * keff;
            for (int j = threadIdx.x; j < keff; j += blockDim.x) {
                os[j] = j < cnt ? rep_score<M>(state[j].skey) : INFINITY;
                oi[j] = j < cnt ? state[j].id : INT32_MAX;
            }
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) last_s = atomicAdd(L.done + f, 1) == P - 1;
            __syncthreads();
            if (!last_s) continue;
            __threadfence();
            // the last part merges the P sorted lists of f, pairwise levels
            const double *cs = L.ps + (int64_t)f * P * keff;
            const int32_t *ci = L.pi + (int64_t)f * P * keff;
            double *bs[2] = {L.ms + (int64_t)f * (P / 2 + 1) * keff, L.ps + (int64_t)f * P * keff};
            int32_t *bi[2] = {L.mi + (int64_t)f * (P / 2 + 1) * keff, L.pi + (int64_t)f * P * keff};
            int lists = P, pp = 0;
            while (lists > 1) {
                const int pairs = lists / 2, outl = pairs + (lists & 1);
                double *ts = bs[pp];
                int32_t *ti = bi[pp];
                if (cs == ts) {  // never write over the level being read
                    ts = bs[pp ^ 1];
                    ti = bi[pp ^ 1];
                }
                for (int64_t t = threadIdx.x; t < (int64_t)lists * keff; t += blockDim.x) {
                    const int li = (int)(t / keff), e = (int)(t % keff);
                    const int pr = li >> 1, other = li ^ 1;
                    const double x = cs[(int64_t)li * keff + e];
                    const int32_t xi = ci[(int64_t)li * keff + e];
                    int64_t rk = e;
                    if (other < lists) {
                        const double *O = cs + (int64_t)other * keff;
                        const int32_t *Oi = ci + (int64_t)other * keff;
                        int lo2 = 0, hi2 = keff;
                        if (li & 1) {  // B side: #{A <= x}
                            while (lo2 < hi2) {
                                const int mid = (lo2 + hi2) >> 1;
                                if (!mkey_less(x, xi, O[mid], Oi[mid])) lo2 = mid + 1; else hi2 = mid;
                            }
                        } else {       // A side: #{B < x}
                            while (lo2 < hi2) {
                                const int mid = (lo2 + hi2) >> 1;
                                if (mkey_less(O[mid], Oi[mid], x, xi)) lo2 = mid + 1; else hi2 = mid;
                            }
                        }
                        rk += lo2;
                    }
                    if (rk < keff) {
                        ts[(int64_t)pr * keff + rk] = x;
                        ti[(int64_t)pr * keff + rk] = xi;
                    }
                }
                __syncthreads();
                cs = ts;
                ci = ti;
                lists = outl;
                pp ^= 1;
            }
            for (int j = threadIdx.x; j < keff; j += blockDim.x) {
                r.out_scores[q * keff + j] = cs[j];
                r.out_ids[q * keff + j] = (int32_t)(ci[j] + r.id_offset);
            }
            __syncthreads();
        } else {
            // flagged queries beyond kRepMaxQ: one CTA scans all rows
            const int64_t q = L.flist[kRepMaxQ + (w - (int64_t)fast * P)];
            const int cnt = rep_scan_rows<M>(r, q, 0, r.n, state, buf, tmp, &buf_n);
            for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
                r.out_scores[q * keff + j] = rep_score<M>(state[j].skey);
                r.out_ids[q * keff + j] = (int32_t)(state[j].id + r.id_offset);
            }
            __syncthreads();
        }
    }
}

int pow2_at_least(int64_t v, int64_t cap) {
    int64_t p = 32;
    while (p < v && p < cap) p <<= 1;
    return (int)p;
}

template <int M>
cudaError_t launch_select_t(const SelectArgs &a, cudaStream_t st) {
    static const bool radix_on = [] {
        const char *v = getenv("QA_B200_SEL_RADIX");  // diagnostics: 0 = merge-per-chunk select
        return !(v && strcmp(v, "0") == 0);
    }();
    if constexpr (M != kAngular) {
        // large batches, integer scores: one warp per query, radix select
        static const bool block_on = [] {
            const char *v = getenv("QA_B200_SEL_BLOCK");  // diagnostics: 0 = one warp per query
            return !(v && strcmp(v, "0") == 0);
        }();
        static const int64_t block_minq = [] {  // diagnostics: smallest batch for the CTA-per-query select
            const char *v = getenv("QA_B200_SEL_BLOCK_MINQ");
            return v ? (int64_t)atoll(v) : (int64_t)256;
        }();
        // small batches too once k > 32: the register select's 64/128-wide
        // networks per candidate chunk cost more than the radix passes (cfg4
        // k = 100: 0.27-0.33 -> 0.25-0.29 ms; k = 10 keeps the register select)
        if (radix_on && block_on && a.k <= 128 && (a.nq >= block_minq || a.k > 32) &&
            a.nq <= 65535 * 16) {
            const unsigned grid = (unsigned)a.nq;
            if (a.k <= 32)
                select_radix_block_kernel<M, 1><<<grid, kRbThreads, 0, st>>>(a);
            else if (a.k <= 64)
                select_radix_block_kernel<M, 2><<<grid, kRbThreads, 0, st>>>(a);
            else
                select_radix_block_kernel<M, 4><<<grid, kRbThreads, 0, st>>>(a);
            return cudaGetLastError();
        }
        if (radix_on && a.k <= 128 && a.nq >= 256) {
            const unsigned grid = (unsigned)((a.nq + kRadixWarps - 1) / kRadixWarps);
            if (a.k <= 32)
                select_radix_kernel<M, 1><<<grid, kRadixWarps * 32, 0, st>>>(a);
            else if (a.k <= 64)
                select_radix_kernel<M, 2><<<grid, kRadixWarps * 32, 0, st>>>(a);
            else
                select_radix_kernel<M, 4><<<grid, kRadixWarps * 32, 0, st>>>(a);
            return cudaGetLastError();
        }
    }
    if (a.k <= 128) {
        // warps per query: enough warps in flight to cover ~5 blocks of 8
        // per SM (the candidate stream is latency-bound per warp)
        const int64_t slots = (int64_t)num_sms() * QA_SEL_MINB * 8;
        int wpq = 1;
        while (wpq < 8 && a.nq * wpq * 2 <= slots) wpq *= 2;
        if (const char *v = getenv("QA_B200_SEL_WPQ")) wpq = atoi(v);  // diagnostics
        const unsigned grid = (unsigned)((a.nq + (8 / wpq) - 1) / (8 / wpq));
        // k <= 32: one register per lane (32-wide sort networks, ~8x fewer
        // instructions than the 128-wide ones)
        if (a.k <= 32) {
            if constexpr (M == kAngular)
                select_reg_kernel<M, RKey96, 1><<<grid, 256, 0, st>>>(a, wpq);
            else
                select_reg_kernel<M, RKey64, 1><<<grid, 256, 0, st>>>(a, wpq);
        } else if (a.k <= 64) {
            if constexpr (M == kAngular)
                select_reg_kernel<M, RKey96, 2><<<grid, 256, 0, st>>>(a, wpq);
            else
                select_reg_kernel<M, RKey64, 2><<<grid, 256, 0, st>>>(a, wpq);
        } else {
            if constexpr (M == kAngular)
                select_reg_kernel<M, RKey96, 4><<<grid, 256, 0, st>>>(a, wpq);
            else
                select_reg_kernel<M, RKey64, 4><<<grid, 256, 0, st>>>(a, wpq);
        }
        return cudaGetLastError();
    }
    const int kpad = (int)((a.k + 31) / 32 * 32);
    const size_t per_warp = (size_t)(2 * kpad + kChunk) * sizeof(Entry);
    int warps = (int)std::min<size_t>(kWarpsMax, (160 * 1024) / per_warp);
    if (warps < 1) warps = 1;
    const size_t smem = per_warp * warps;
    cudaError_t e = cudaFuncSetAttribute(select_kernel<M>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)((a.nq + warps - 1) / warps);
    select_kernel<M><<<grid, warps * 32, smem, st>>>(a, kpad);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_select(const SelectArgs &a_in, cudaStream_t st) {
    if (a_in.nq == 0) return cudaSuccess;
    SelectArgs a = a_in;
    if (a.k > 128) {  // the shared-memory select has no fused estimate / fill
        a.est_j = 0;
        a.next_fill = -1;
    }
    switch (a.metric) {
        case kIP: return launch_select_t<kIP>(a, st);
        case kL2: return launch_select_t<kL2>(a, st);
        default: return launch_select_t<kAngular>(a, st);
    }
}

size_t repair_scratch_bytes(int64_t n, int64_t nq, int64_t keff) {
    const int P = rep_parts(n);
    const size_t lists = (size_t)kRepMaxQ * P * keff, half = (size_t)kRepMaxQ * (P / 2 + 1) * keff;
    return (size_t)nq * 4 + 8 + kRepMaxQ * 4 + lists * 12 + half * 12 + 8 * 256;
}

cudaError_t launch_repair(const RepairArgs &r, cudaStream_t st) {
    if (r.nq == 0 || r.keff == 0 || r.n == 0) return cudaSuccess;
    if (r.keff > kMaxK || r.ld % 16 != 0 || !r.scratch) return cudaErrorNotSupported;
    const int P = rep_parts(r.n);
    const RepLayout L = rep_layout(r.scratch, r.nq, r.keff, P);
    repair_compact_kernel<<<1, 1024, 0, st>>>(r.flag, r.nq, L);
    const size_t smem = (size_t)(2 * r.keff + kRepChunk) * sizeof(Entry);
    auto go = [&](auto kern) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        kern<<<(unsigned)(num_sms() * 2), kRepThreads, smem, st>>>(r, L, P);
        return cudaGetLastError();
    };
    if (r.metric == kIP) return go(repair_kernel<kIP>);
    if (r.metric == kL2) return go(repair_kernel<kL2>);
    return go(repair_kernel<kAngular>);
}

cudaError_t launch_fill(int32_t *p, int64_t n, int32_t v, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    reset_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, n, v);
    return cudaGetLastError();
}

// Threshold estimate for the final pass: the j-th best score of the prefix
// scanned so far (j < k), a bound that about j * n / prefix rows of the whole
// set reach.  est[q] keeps its order key for the check after the pass;
// ~0 = no estimate (fewer than j entries: the k-th threshold stays).
template <int M>
__global__ void estimate_kernel(const Entry *__restrict__ state,
                                const int32_t *__restrict__ state_cnt, int32_t *__restrict__ thr,
                                unsigned long long *__restrict__ est, int64_t nq, int64_t k,
                                int64_t j, const int32_t *__restrict__ q_sqnorm,
                                const float *__restrict__ q_norm, bool combine) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    if (state_cnt[q] < j) {
        if (!combine) est[q] = ~0ull;
        return;
    }
    const Entry e = state[q * k + j - 1];
    const int32_t qq = (M == kL2) ? q_sqnorm[q] : 0;
    const float qn = (M == kAngular) ? q_norm[q] : 1.0f;
    thr[q] = threshold_of<M>(e, qq, qn);
    // rows that failed an earlier estimated pass are only known to be worse
    // than THAT estimate: the final check needs the k-th at least as good as
    // every estimate used
    const unsigned long long prev = est[q];
    est[q] = (combine && prev != ~0ull && prev < e.skey) ? prev : e.skey;
}

// After the final pass: the result is exact iff the k-th kept score is at
// least the estimate's score (every row that failed the estimate's bound is
// strictly worse).  Queries where it is not are flagged for recomputation.
__global__ void check_estimate_kernel(const Entry *__restrict__ state,
                                      const int32_t *__restrict__ state_cnt,
                                      const unsigned long long *__restrict__ est, int64_t nq,
                                      int64_t k, int32_t *__restrict__ redo,
                                      int32_t *__restrict__ any_redo) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const unsigned long long e = est[q];
    if (e == ~0ull) return;
    const bool ok = state_cnt[q] >= k && state[q * k + k - 1].skey <= e;
    if (!ok) {
        redo[q] = 1;
        atomicExch(any_redo, 1);
    }
}

cudaError_t launch_estimate(const Entry *state, const int32_t *state_cnt, int32_t *thr,
                            unsigned long long *est, int64_t nq, int64_t k, int64_t j, int metric,
                            const int32_t *q_sqnorm, const float *q_norm, bool combine,
                            cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    const unsigned grid = (unsigned)((nq + 255) / 256);
    switch (metric) {
        case kIP:
            estimate_kernel<kIP><<<grid, 256, 0, st>>>(state, state_cnt, thr, est, nq, k, j,
                                                       q_sqnorm, q_norm, combine);
            break;
        case kL2:
            estimate_kernel<kL2><<<grid, 256, 0, st>>>(state, state_cnt, thr, est, nq, k, j,
                                                       q_sqnorm, q_norm, combine);
            break;
        default:
            estimate_kernel<kAngular><<<grid, 256, 0, st>>>(state, state_cnt, thr, est, nq, k, j,
                                                            q_sqnorm, q_norm, combine);
    }
    return cudaGetLastError();
}

// Threshold estimate from a sampled pass (filter mode 4): per query, the
// j-th largest of its nb bucket keys (order-preserving int32 "goodness",
// qa_filter_tc.cu) by an MSB-first radix select, turned into the final pass's
// threshold and the order key the check after it compares with.  The key is
// a real row's goodness and at least j distinct rows reach it, so it plays the
// role of the j-th best prefix score (estimate_kernel).  Angular goodness is
// float(dot) / xn, so its score is approximate; the estimate is a heuristic
// and exactness rests on the check (finalize_kernel), not on it.
template <int M>
__global__ void __launch_bounds__(256) est_select_kernel(
    const int32_t *__restrict__ keys, int64_t ld, int64_t nb, int64_t j,
    const int32_t *__restrict__ q_sqnorm, const float *__restrict__ q_norm,
    int32_t *__restrict__ thr, unsigned long long *__restrict__ est) {
    __shared__ unsigned hist[256];
    __shared__ unsigned s_digit, s_want;
    const int64_t q = blockIdx.x;
    const int32_t *kq = keys + q * ld;
    unsigned prefix = 0, mask = 0, want = (unsigned)j;  // rank from the top, 1-based
    for (int shift = 24; shift >= 0; shift -= 8) {
        hist[threadIdx.x] = 0;
        __syncthreads();
        for (int64_t i = threadIdx.x; i < nb; i += 256) {
            const unsigned u = (unsigned)__ldg(kq + i) ^ 0x80000000u;
            if ((u & mask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // lane l owns digits 255 - 8l .. 248 - 8l (descending)
            const int lane = threadIdx.x;
            unsigned c[8], tot = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                c[i] = hist[255 - 8 * lane - i];
                tot += c[i];
            }
            unsigned incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const unsigned excl = incl - tot;
            const unsigned hitm = __ballot_sync(0xffffffffu, incl >= want && excl < want);
            if (hitm) {
                const int src = __ffs(hitm) - 1;
                if (lane == src) {
                    unsigned acc = excl;
                    int i = 0;
                    while (acc + c[i] < want) acc += c[i++];
                    s_digit = 255u - 8u * (unsigned)lane - (unsigned)i;
                    s_want = want - acc;
                }
            } else if (lane == 0) {
                s_digit = 0xffffffffu;  // fewer than `want` keys match
            }
        }
        __syncthreads();
        const unsigned dg = s_digit;
        want = s_want;
        __syncthreads();
        if (dg == 0xffffffffu) {
            if (threadIdx.x == 0) est[q] = ~0ull;  // thr keeps its pass-all init
            return;
        }
        prefix |= dg << shift;
        mask |= 255u << shift;
    }
    if (threadIdx.x != 0) return;
    const int32_t g = (int32_t)(prefix ^ 0x80000000u);
    if (g == INT32_MIN) {  // the j-th bucket saw no row
        est[q] = ~0ull;
        return;
    }
    Entry e;
    e.id = 0;
    e.row = 0;
    int32_t qq = 0;
    float qn = 1.0f;
    if constexpr (M == kIP) {
        e.skey = skey_from_int((int32_t)(0u - (uint32_t)g));  // score = -dot
    } else if constexpr (M == kL2) {
        qq = q_sqnorm[q];
        e.skey = skey_from_int((int32_t)((uint32_t)qq - (uint32_t)g));  // qq + xx - 2 dot
    } else {
        qn = q_norm[q];
        const int32_t fb = g < 0 ? (g ^ 0x7fffffff) : g;
        e.skey = skey_from_double(1.0 - (double)__int_as_float(fb) / (double)qn);
    }
    thr[q] = threshold_of<M>(e, qq, qn);
    est[q] = e.skey;
}

cudaError_t launch_est_select(const int32_t *keys, int64_t ld, int64_t nb, int64_t nq, int64_t j,
                              int metric, const int32_t *q_sqnorm, const float *q_norm,
                              int32_t *thr, unsigned long long *est, cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    if (nq > 0x7fffffff || j < 1) return cudaErrorInvalidValue;
    const unsigned grid = (unsigned)nq;
    switch (metric) {
        case kIP:
            est_select_kernel<kIP><<<grid, 256, 0, st>>>(keys, ld, nb, j, q_sqnorm, q_norm, thr, est);
            break;
        case kL2:
            est_select_kernel<kL2><<<grid, 256, 0, st>>>(keys, ld, nb, j, q_sqnorm, q_norm, thr, est);
            break;
        default:
            est_select_kernel<kAngular><<<grid, 256, 0, st>>>(keys, ld, nb, j, q_sqnorm, q_norm,
                                                              thr, est);
    }
    return cudaGetLastError();
}

cudaError_t launch_check_estimate(const Entry *state, const int32_t *state_cnt,
                                  const unsigned long long *est, int64_t nq, int64_t k,
                                  int32_t *redo, int32_t *any_redo, cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    check_estimate_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(state, state_cnt, est, nq,
                                                                       k, redo, any_redo);
    return cudaGetLastError();
}

cudaError_t launch_init_state(int32_t *state_cnt, int32_t *thr, int64_t nq, int metric,
                              cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    int32_t pass = metric == kIP ? kThrPassIP
                                 : (metric == kL2 ? kThrPassL2 : (int32_t)kThrPassAngBits);
    init_state_kernel<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(state_cnt, thr, nq, pass,
                                                                    nullptr, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_init_state_full(int32_t *state_cnt, int32_t *thr, int64_t nq, int metric,
                                   int32_t *ovf, int32_t *flags, int32_t *ccount, int32_t fill0,
                                   cudaStream_t st, unsigned *sched, int nsched) {
    int32_t pass = metric == kIP ? kThrPassIP
                                 : (metric == kL2 ? kThrPassL2 : (int32_t)kThrPassAngBits);
    int64_t m = nq > 16 ? nq : 16;
    if (m < nsched) m = nsched;
    init_state_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(state_cnt, thr, nq, pass, ovf,
                                                                   flags, ccount, fill0, sched,
                                                                   nsched);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const Entry *state, int64_t nq, int64_t k, int64_t keff, int metric,
                            int64_t id_offset, double *out_scores, int32_t *out_ids,
                            cudaStream_t st, const int32_t *state_cnt,
                            const unsigned long long *est, int32_t *redo, int32_t *any_redo) {
    int64_t total = nq * keff;
    if (total == 0) return cudaSuccess;
    unsigned grid = (unsigned)((total + 255) / 256);
    switch (metric) {
        case kIP:
            finalize_kernel<kIP><<<grid, 256, 0, st>>>(state, nq, k, keff, id_offset, out_scores,
                                                       out_ids, state_cnt, est, redo, any_redo);
            break;
        case kL2:
            finalize_kernel<kL2><<<grid, 256, 0, st>>>(state, nq, k, keff, id_offset, out_scores,
                                                       out_ids, state_cnt, est, redo, any_redo);
            break;
        default:
            finalize_kernel<kAngular><<<grid, 256, 0, st>>>(state, nq, k, keff, id_offset,
                                                            out_scores, out_ids, state_cnt, est,
                                                            redo, any_redo);
    }
    return cudaGetLastError();
}

size_t merge_scratch_bytes(int64_t G, int64_t nq, int64_t kin, int64_t k) {
    if (k <= kMaxK && k + kin <= kSortMax) return 0;
    const int64_t len = std::min<int64_t>(k, 2 * kin);
    return (size_t)2 * ((G + 1) / 2) * nq * len * 12 + 256;
}

cudaError_t launch_merge(const double *in_scores, const int32_t *in_ids, int64_t G, int64_t nq,
                         int64_t kin, int64_t k, double *out_scores, int32_t *out_ids,
                         cudaStream_t st, void *scratch) {
    if (nq == 0 || k == 0) return cudaSuccess;
    if (k > kMaxK || k + kin > kSortMax) {
        // pairwise merge-path tree; level buffers [lists, nq, len] x 2 in scratch
        if (!scratch) return cudaErrorInvalidValue;
        const int64_t cap = std::min<int64_t>(k, 2 * kin);
        const int64_t half = (G + 1) / 2;
        double *bs[2] = {(double *)scratch, (double *)scratch + half * nq * cap};
        int32_t *bi[2] = {(int32_t *)(bs[1] + half * nq * cap),
                          (int32_t *)(bs[1] + half * nq * cap) + half * nq * cap};
        const double *cs = in_scores;
        const int32_t *ci = in_ids;
        std::vector<int64_t> lens((size_t)G, kin);  // valid entries per list
        int64_t ld = kin;
        int buf = 0;
        while (true) {
            const int64_t lists = (int64_t)lens.size();
            const bool last = lists <= 2;
            const int64_t nlen = last ? k : cap;
            double *os = last ? out_scores : bs[buf];
            int32_t *oi = last ? out_ids : bi[buf];
            const int64_t ldo = nlen;
            std::vector<int64_t> nl;
            for (int64_t p = 0; 2 * p < lists; ++p) {
                const int64_t a0 = 2 * p, b0 = 2 * p + 1;
                const int64_t la = lens[a0], lb = b0 < lists ? lens[b0] : 0;
                const int64_t outn = std::min<int64_t>(nlen, la + lb);
                dim3 grid((unsigned)((la + lb + 255) / 256), (unsigned)nq);
                merge_pair_kernel<<<grid, 256, 0, st>>>(
                    cs + a0 * nq * ld, ci + a0 * nq * ld, la, ld,
                    cs + (b0 < lists ? b0 : a0) * nq * ld, ci + (b0 < lists ? b0 : a0) * nq * ld,
                    lb, ld, outn, os + p * nq * ldo, oi + p * nq * ldo, ldo);
                nl.push_back(outn);
            }
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) return e;
            if (last) break;
            cs = os;
            ci = oi;
            lens.swap(nl);
            ld = ldo;
            buf ^= 1;
        }
        return cudaSuccess;
    }
    const int sz = pow2_at_least(k + kin, kSortMax);
    const size_t smem = (size_t)sz * sizeof(MEntry);
    cudaError_t e = cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    merge_kernel<<<(unsigned)nq, 256, smem, st>>>(in_scores, in_ids, G, nq, kin, k, out_scores,
                                                  out_ids, sz);
    return cudaGetLastError();
}

}  // namespace qa
