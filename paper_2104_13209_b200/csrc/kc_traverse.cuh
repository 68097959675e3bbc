// kc_traverse.cuh -- warp-level search-tree traversals (K5 orient, K6/K7 pivot).
//
// One warp walks one level-1 subtree of a task's induced sub-graph.  A
// candidate set over the d locals is a *lane-distributed bitset*: lane l holds
// words l, l+32, ... (WPL words per lane, W = ceil(d/32) <= 32*WPL), so
// AND-ing a set with a bitmap row is one coalesced shared-memory load per lane
// and emptiness / next-vertex selection are __ballot_sync + __ffs + __shfl_sync
// (PAPER.md:405-418, :461-465).  Local ids ascend with (word, bit), so
// next_bit() enumerates a set in ascending local id -- the reference's order
// (engine_orient.py:51-60, engine_pivot.py:140-150).
//
// The hot primitive of both engines is "score every v of a set C against C":
//   orient, last level (engine_orient.py:64-69): sum_v popc(C & row v)
//   pivot selection  (engine_pivot.py:82-101):   argmax_v popc(C & row v)
// It runs lane-parallel over v (C compacted into a per-warp list, lane j takes
// the j-th member) and word-sparse over C: only the nonzero words of C
// (one ballot) are visited, each broadcast from its owner lane by __shfl_sync.
//
// Work accounting: `work` counts tree units (a visit, or one candidate
// scored by a pivot choice); the kernels scale a task's units by its row
// width ceil(d/32), which is SURVEY.md §8(d)'s algorithmic word count.
//
// Frames of the explicit DFS stack hold only the candidate set (and, for the
// pivot engine, the branch set and two scalars); the "remaining" cursor set is
// recomputed from the last expanded vertex, so a frame is 32*WPL (+32*WPL+4)
// words.  The first `nsm` frames of a warp live in shared memory, deeper
// ones in a per-warp global slot (L1-cached).
#pragma once

#include "kc_internal.cuh"

namespace kct {

typedef unsigned long long ull;
constexpr unsigned FULL = 0xffffffffu;

// explicit shared-memory accesses for data the compiler only sees through
// generic pointers (it would emit LD.E / ST.E with long-scoreboard waits)
__device__ __forceinline__ unsigned smem_addr(const void *p) {
    return unsigned(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds32(unsigned a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds64(unsigned a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts64(unsigned a, uint2 v) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(v.x), "r"(v.y) : "memory");
}

template <int WPL>
struct Set {
    uint32_t w[WPL];
};

// bits of a 32-bit word (local ids w*32 .. w*32+31) strictly above local id c
__device__ __forceinline__ uint32_t above_mask(int word, int c) {
    const int lo = word << 5;
    if (c < lo) return FULL;
    if (c >= lo + 31) return 0u;
    return ~((2u << (c - lo)) - 1u);
}
// bits strictly below local id v
__device__ __forceinline__ uint32_t below_mask(int word, int v) {
    const int lo = word << 5;
    if (v >= lo + 32) return FULL;
    if (v <= lo) return 0u;
    return (1u << (v - lo)) - 1u;
}

template <int WPL>
__device__ __forceinline__ Set<WPL> load_row(const uint32_t *__restrict__ rows, int RS, int W,
                                             int v, int lane) {
    Set<WPL> r;
    const uint32_t *rv = rows + v * RS;
#pragma unroll
    for (int p = 0; p < WPL; ++p) {
        const int w = p * 32 + lane;
        r.w[p] = w < W ? rv[w] : 0u;
    }
    return r;
}

template <int WPL>
__device__ __forceinline__ bool any_set(const Set<WPL> &s) {
    uint32_t x = 0;
#pragma unroll
    for (int p = 0; p < WPL; ++p) x |= s.w[p];
    return __ballot_sync(FULL, x != 0) != 0;
}

// keep only local id v in R (lane-distributed)
template <int WPL>
__device__ __forceinline__ void restrict_to(Set<WPL> &R, int v, int lane) {
#pragma unroll
    for (int p = 0; p < WPL; ++p)
        R.w[p] &= (p * 32 + lane == (v >> 5)) ? (1u << (v & 31)) : 0u;
}

template <int WPL>
__device__ __forceinline__ int popc_set(const Set<WPL> &s) {  // per-lane part
    int c = 0;
#pragma unroll
    for (int p = 0; p < WPL; ++p) c += __popc(s.w[p]);
    return c;
}

template <int WPL>
__device__ __forceinline__ void store_set(uint32_t *f, const Set<WPL> &S, int lane) {
#pragma unroll
    for (int p = 0; p < WPL; ++p) f[p * 32 + lane] = S.w[p];
}
template <int WPL>
__device__ __forceinline__ Set<WPL> load_set(const uint32_t *f, int lane) {
    Set<WPL> S;
#pragma unroll
    for (int p = 0; p < WPL; ++p) S.w[p] = f[p * 32 + lane];
    return S;
}

// lowest member of R (ascending local id), removed from R; -1 if empty
template <int WPL>
__device__ __forceinline__ int next_bit(Set<WPL> &R, int lane) {
#pragma unroll
    for (int p = 0; p < WPL; ++p) {
        const unsigned b = __ballot_sync(FULL, R.w[p] != 0);
        if (b) {
            const int L = __ffs(b) - 1;
            const uint32_t x = __shfl_sync(FULL, R.w[p], L);
            if (lane == L) R.w[p] = x & (x - 1u);
            return ((p * 32 + L) << 5) + __ffs(x) - 1;
        }
    }
    return -1;
}

// position of the k-th (0-based) set bit of x (k < popc(x)); branch-free
__device__ __forceinline__ int nth_bit(uint32_t x, int k) {
    int p = 0;
#pragma unroll
    for (int w = 16; w; w >>= 1) {
        const int c = __popc(x & ((1u << w) - 1u));
        if (k >= c) {
            k -= c;
            x >>= w;
            p += w;
        }
    }
    return p;
}

// lanes per member so that `cnt` members fill the warp: 32 / pow2ceil(cnt)
__device__ __forceinline__ int lanes_per_member_log2(int cnt) {
    return cnt > 16 ? 0 : cnt > 8 ? 1 : cnt > 4 ? 2 : cnt > 2 ? 3 : cnt > 1 ? 4 : 5;
}
// bits b of a word with b % 2^lg == sub
__device__ __forceinline__ uint32_t id_stripe(int lg, int sub) {
    const uint32_t rep = lg == 5 ? 1u : 0xffffffffu / ((1u << (1 << lg)) - 1u);
    return rep << sub;
}

// compact the members of a set of at most four words (C lane-distributed:
// lane w holds word w) into list[0..n): lane L owns bits [4L, 4L+4), so every
// lane does at most four iterations (the word-per-lane loop below leaves 28
// lanes idle for such sets)
__device__ __forceinline__ int compact4(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                        int *list, int lane) {
    const int wsel = lane >> 3;
    const uint32_t word = wsel == 0 ? c0 : wsel == 1 ? c1 : wsel == 2 ? c2 : c3;
    uint32_t nib = (word >> ((lane & 7) << 2)) & 15u;
    const int c = __popc(nib);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    int off = incl - c;
    while (nib) {
        list[off++] = (lane << 2) + __ffs(nib) - 1;
        nib &= nib - 1u;
    }
    const int n = __shfl_sync(FULL, incl, 31);
    __syncwarp();
    return n;
}

// members of an eight-word set (words replicated in every lane: c[0..8)):
// lane L owns bits [8L, 8L+8)
__device__ __forceinline__ int compact8(const uint32_t (&c)[8], int *list, int lane) {
    const int wsel = lane >> 2;
    uint32_t word = c[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) word = wsel == i ? c[i] : word;
    uint32_t byte = (word >> ((lane & 3) << 3)) & 255u;
    const int cnt = __popc(byte);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    int off = incl - cnt;
    while (byte) {
        list[off++] = (lane << 3) + __ffs(byte) - 1;
        byte &= byte - 1u;
    }
    const int n = __shfl_sync(FULL, incl, 31);
    __syncwarp();
    return n;
}

// compact the members of C (ascending) into list[0..n); returns n (uniform)
template <int WPL>
__device__ __forceinline__ int compact(const Set<WPL> &C, int *list, int lane, int W = 32 * WPL) {
    if (WPL == 1 && W <= 4)
        return compact4(__shfl_sync(FULL, C.w[0], 0), __shfl_sync(FULL, C.w[0], 1),
                        __shfl_sync(FULL, C.w[0], 2), __shfl_sync(FULL, C.w[0], 3), list, lane);
    int n = 0;
#pragma unroll
    for (int p = 0; p < WPL; ++p) {
        uint32_t x = C.w[p];
        const int c = __popc(x);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        int off = n + incl - c;
        const int base = (p * 32 + lane) << 5;
        while (x) {
            list[off++] = base + __ffs(x) - 1;
            x &= x - 1u;
        }
        n += __shfl_sync(FULL, incl, 31);
    }
    __syncwarp();
    return n;
}

// popc(C & row v) for this lane's v (valid) over the nonzero words of C.
// All lanes must call it (shuffles); invalid lanes pass v = 0, valid = false.
template <int WPL>
__device__ __forceinline__ int cover(const uint32_t *__restrict__ rows, int RS,
                                     const Set<WPL> &C, int v, bool valid) {
    int cov = 0;
    const uint32_t *rv = rows + v * RS;
#pragma unroll
    for (int p = 0; p < WPL; ++p) {
        unsigned nz = __ballot_sync(FULL, C.w[p] != 0);
        while (nz) {
            const int L = __ffs(nz) - 1;
            nz &= nz - 1u;
            const uint32_t cw = __shfl_sync(FULL, C.w[p], L);
            if (valid) cov += __popc(cw & rv[p * 32 + L]);
        }
    }
    return cov;
}

// sum over v in C of popc(C & row v); the sum lands in the calling lanes'
// accumulators (reduced at kernel end).  Returns |C| (uniform).
template <int WPL>
__device__ __forceinline__ int score_sum(const uint32_t *__restrict__ rows, int RS,
                                         const Set<WPL> &C, int *list, int lane, ull &acc,
                                         ull &work, int W) {
    const int n = compact<WPL>(C, list, lane);
    for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        const bool ok = i < n;
        const int v = ok ? list[i] : 0;
        acc += ull(cover<WPL>(rows, RS, C, v, ok));
    }
    if (lane == 0) work += ull(n);
    __syncwarp();
    return n;
}

// The last TWO orientation levels at once, lane-parallel over v in C
// (frame last-1 = C): every v in C is a visit, each x in X_v = C & row v is a
// visit of the last frame contributing popc(X_v & row x).  Lane j owns the
// j-th member v of C and walks X_v itself (3-way AND + POPC per word), so the
// per-visit ballot/shuffle work of the sequential walk disappears for the two
// levels that hold almost all visits.  cbuf: per-warp copy of C (32*WPL words).
// Harley-Seal carry-save popcount accumulator.  The last orientation level
// sums popc(C & row x) over many words; instead of one POPC per word (the
// XU pipe, 16 lanes/clk/SM -- the measured bound of the pair loops) the words
// go through full adders (two LOP3 each, 64 lanes/clk/SM) into weight-1 and
// weight-2 bit planes, and only the weight-4 carries are popcounted: one POPC
// per four words.  The sum is exact: total = popc(ones) + 2 popc(twos) + 4 fours.
struct CsaAcc {
    uint32_t ones = 0, twos = 0;
    unsigned fours = 0;
    __device__ __forceinline__ static void fa(uint32_t &carry, uint32_t &sum, uint32_t a,
                                              uint32_t b, uint32_t c) {
        const uint32_t u = a ^ b;
        carry = (a & b) | (u & c);
        sum = u ^ c;
    }
    __device__ __forceinline__ void add4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
        uint32_t ca, cb, c4;
        fa(ca, ones, ones, a, b);
        fa(cb, ones, ones, c, d);
        fa(c4, twos, twos, ca, cb);
        fours += unsigned(__popc(c4));
    }
    __device__ __forceinline__ void add2(uint32_t a, uint32_t b) {
        uint32_t ca;
        fa(ca, ones, ones, a, b);
        const uint32_t c4 = twos & ca;
        twos ^= ca;
        fours += unsigned(__popc(c4));
    }
    __device__ __forceinline__ unsigned total() const {
        return 4u * fours + unsigned(__popc(ones)) + 2u * unsigned(__popc(twos));
    }
};

// Warp tier, rows of at most four words with a 16-byte stride: the members v
// of C are spread so that each gets 32 / pow2ceil(#members) lanes (a sub-warp
// group), and the lanes of a group split v's walk over X_v = C & row v by
// member id (id stripes); every (v, x) pair costs one LDS.128 and a
// carry-save add of four words.  Counts and visits are sums, hence unchanged.
__device__ __forceinline__ void score_pairs4(const uint32_t *__restrict__ rows, const Set<1> &C,
                                             int *list, int lane, ull &acc, ull &visits,
                                             ull &work) {
    const uint32_t c0 = __shfl_sync(FULL, C.w[0], 0), c1 = __shfl_sync(FULL, C.w[0], 1);
    const uint32_t c2 = __shfl_sync(FULL, C.w[0], 2), c3 = __shfl_sync(FULL, C.w[0], 3);
    const int n = compact4(c0, c1, c2, c3, list, lane);
    if (lane == 0) visits += ull(n);
    unsigned a32 = 0;
    for (int base = 0; base < n; base += 32) {
        const int cnt = n - base < 32 ? n - base : 32;
        const int lg = lanes_per_member_log2(cnt);
        const int mi = lane >> lg, sub = lane & ((1 << lg) - 1);
        if (mi >= cnt) continue;
        const int v = list[base + mi];
        const uint4 rv = *reinterpret_cast<const uint4 *>(rows + (v << 2));
        const uint32_t cm0 = c0 & rv.x, cm1 = c1 & rv.y, cm2 = c2 & rv.z, cm3 = c3 & rv.w;
        if (sub == 0) {
            const ull xs = ull(__popc(cm0) + __popc(cm1) + __popc(cm2) + __popc(cm3));
            visits += xs;
            work += 1 + xs;
        }
        const uint32_t st = id_stripe(lg, sub);
        CsaAcc h;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            uint32_t m = (w == 0 ? cm0 : w == 1 ? cm1 : w == 2 ? cm2 : cm3) & st;
            while (m) {
                const int b = 31 - __clz(m);
                m ^= 1u << b;
                const uint4 r = *reinterpret_cast<const uint4 *>(rows + (((w << 5) + b) << 2));
                h.add4(cm0 & r.x, cm1 & r.y, cm2 & r.z, cm3 & r.w);
            }
        }
        a32 += h.total();
    }
    acc += a32;
    __syncwarp();
}

// score_pairs4 for eight-word rows (stride 8, two LDS.128 per row): the
// pair level of a CTA-tier set compressed to 129..256 members
__device__ __forceinline__ void score_pairs8(const uint32_t *__restrict__ rows, int n, int *list,
                                             int lane, ull &acc, ull &visits, ull &work) {
    uint32_t c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int lo = i << 5;
        c[i] = lo >= n ? 0u : (lo + 32 <= n ? FULL : ((1u << (n - lo)) - 1u));
    }
    if (lane == 0) visits += ull(n);
    unsigned a32 = 0;
    for (int base = 0; base < n; base += 32) {
        const int cnt = n - base < 32 ? n - base : 32;
        const int lg = lanes_per_member_log2(cnt);
        const int mi = lane >> lg, sub = lane & ((1 << lg) - 1);
        if (mi >= cnt) continue;
        const int v = base + mi;  // members are 0..n-1
        const uint4 ra = *reinterpret_cast<const uint4 *>(rows + (v << 3));
        const uint4 rb = *reinterpret_cast<const uint4 *>(rows + (v << 3) + 4);
        const uint32_t cm[8] = {c[0] & ra.x, c[1] & ra.y, c[2] & ra.z, c[3] & ra.w,
                                c[4] & rb.x, c[5] & rb.y, c[6] & rb.z, c[7] & rb.w};
        if (sub == 0) {
            unsigned xs = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) xs += unsigned(__popc(cm[i]));
            visits += ull(xs);
            work += 1 + ull(xs);
        }
        const uint32_t st = id_stripe(lg, sub);
        CsaAcc h;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            uint32_t m = cm[w] & st;
            while (m) {
                const int b = 31 - __clz(m);
                m ^= 1u << b;
                const uint32_t *rx = rows + (((w << 5) + b) << 3);
                const uint4 xa = *reinterpret_cast<const uint4 *>(rx);
                const uint4 xb = *reinterpret_cast<const uint4 *>(rx + 4);
                h.add4(cm[0] & xa.x, cm[1] & xa.y, cm[2] & xa.z, cm[3] & xa.w);
                h.add4(cm[4] & xb.x, cm[5] & xb.y, cm[6] & xb.z, cm[7] & xb.w);
            }
        }
        a32 += h.total();
    }
    acc += a32;
    __syncwarp();
}

// Pair level of a wide task (rows of W > 4 words, the CTA tier) whose set X
// has 33..256 members: relabel X's members 0..n-1 (ascending local id) and
// compress their rows restricted to X into 16- or 32-byte rows (mrow), then
// run the four- / eight-word pair loop over them.  Compression is a parallel
// bit extract per word (Hacker's Delight 7-4 "compress": five shift/mask steps
// whose masks depend only on X's word, built once per set), the extracted
// pieces funnelled into the output row at the running offset -- a fixed cost
// per (member, word) with no divergence between lanes (the earlier per-bit
// loop ran at ~2 active lanes: ncu, profiles/r2b_ncu_cta_orient_rmat22.md).
// Counts and visits are order-free sums, hence unchanged.
// words of the compressed rows of a pair level of at most mid_max members
__host__ __device__ constexpr int mid_rows_words(int mid_max) { return mid_max <= 128 ? 512 : 2048; }

__device__ __forceinline__ void compress_masks(uint32_t m, uint32_t (&mv)[5]) {
    uint32_t mk = ~m << 1;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        uint32_t mp = mk ^ (mk << 1);
        mp ^= mp << 2;
        mp ^= mp << 4;
        mp ^= mp << 8;
        mp ^= mp << 16;
        mv[i] = mp & m;
        m = (m ^ mv[i]) | (mv[i] >> (1 << i));
        mk &= ~mp;
    }
}

template <int WPL>
__device__ __forceinline__ void score_pairs_mid(const uint32_t *__restrict__ rows, int RS, int W,
                                                const Set<WPL> &X, int *list, uint32_t *cbuf,
                                                uint32_t *mrow, int mid_max, int lane, ull &acc,
                                                ull &visits, ull &work) {
    (void)cbuf;
    const int n = compact<WPL>(X, list, lane, W);
    // per word w of X: [X_w, popc(X_w), mv0..mv4, -] (two 16-byte loads)
    uint32_t *tab = mrow + mid_rows_words(mid_max);
#pragma unroll
    for (int p = 0; p < WPL; ++p) {
        const int w = p * 32 + lane;
        if (w < W) {
            uint32_t mv[5];
            compress_masks(X.w[p], mv);
            *reinterpret_cast<uint4 *>(tab + w * 8) =
                make_uint4(X.w[p], uint32_t(__popc(X.w[p])), mv[0], mv[1]);
            *reinterpret_cast<uint4 *>(tab + w * 8 + 4) = make_uint4(mv[2], mv[3], mv[4], 0u);
        }
    }
    __syncwarp();
    const int RSM = n <= 128 ? 4 : 8;  // compressed row stride (words)
    for (int i = lane; i < n; i += 32) {
        const uint32_t *ri = rows + list[i] * RS;
        uint32_t *out = mrow + i * RSM;
        uint32_t lo = 0u, hi = 0u;
        int fill = 0, q = 0;
        for (int w = 0; w < W; ++w) {
            const uint4 a = *reinterpret_cast<const uint4 *>(tab + w * 8);
            if (a.x == 0u) continue;  // uniform: depends on X only
            uint32_t x = ri[w] & a.x;
            if (a.x != FULL) {
                const uint4 b = *reinterpret_cast<const uint4 *>(tab + w * 8 + 4);
                uint32_t t;
                t = x & a.z;  x = (x ^ t) | (t >> 1);
                t = x & a.w;  x = (x ^ t) | (t >> 2);
                t = x & b.x;  x = (x ^ t) | (t >> 4);
                t = x & b.y;  x = (x ^ t) | (t >> 8);
                t = x & b.z;  x = (x ^ t) | (t >> 16);
            }
            lo |= x << fill;
            hi |= __funnelshift_l(x, 0u, fill);  // bits of x shifted past bit 31
            fill += int(a.y);
            if (fill >= 32) {  // uniform
                out[q++] = lo;
                lo = hi;
                hi = 0u;
                fill -= 32;
            }
        }
        if (fill > 0) out[q++] = lo;
        while (q < RSM) out[q++] = 0u;
    }
    __syncwarp();
    if (RSM == 8) {
        score_pairs8(mrow, n, list, lane, acc, visits, work);
        return;
    }
    Set<1> all;
    {
        const int lo = lane << 5;
        all.w[0] = lo >= n ? 0u : (lo + 32 <= n ? FULL : ((1u << (n - lo)) - 1u));
    }
    score_pairs4(mrow, all, list, lane, acc, visits, work);
}

template <int WPL>
__device__ __forceinline__ void score_pairs(const uint32_t *__restrict__ rows, int RS, int W,
                                            const Set<WPL> &C, int *list, uint32_t *cbuf,
                                            int lane, ull &acc, ull &visits, ull &work) {
    if (WPL == 1 && W >= 2 && W <= 4 && RS == 4) {
        score_pairs4(rows, reinterpret_cast<const Set<1> &>(C), list, lane, acc, visits, work);
        return;
    }
    const int n = compact<WPL>(C, list, lane, W);
    store_set<WPL>(cbuf, C, lane);
    __syncwarp();
    visits += ull(popc_set<WPL>(C));
    for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        if (i >= n) break;
        const int v = list[i];
        const uint32_t *rv = rows + v * RS;
        ull a = 0, x_seen = 0;
        if (W == 1) {
            const uint32_t cm = cbuf[0] & rv[0];
            uint32_t m = cm;
            x_seen = __popc(m);
            while (m) {
                const int x = __ffs(m) - 1;
                m &= m - 1u;
                a += __popc(cm & rows[x * RS]);
            }
        } else if (WPL == 1 && W <= 4) {
            // rows of at most 4 words (the warp tier): C & row v in registers,
            // fully unrolled 3-way AND + POPC per member x
            uint32_t cm[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) cm[w] = w < W ? (cbuf[w] & rv[w]) : 0u;
            unsigned a32 = 0;
            if (RS == 4) {  // 16-byte rows (warp tier, orientation): one LDS.128 per member
                // members in any order (the sum is order-free): top bit first
                // needs one FLO, no BREV; words summed through CsaAcc
                CsaAcc h;
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    uint32_t m = cm[w];
                    x_seen += __popc(m);
                    while (m) {
                        const int b = 31 - __clz(m);
                        m ^= 1u << b;
                        const uint4 r = *reinterpret_cast<const uint4 *>(rows + ((w << 5) + b) * 4);
                        h.add4(cm[0] & r.x, cm[1] & r.y, cm[2] & r.z, cm[3] & r.w);
                    }
                }
                a32 = h.total();
            } else {
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    uint32_t m = cm[w];
                    x_seen += __popc(m);
                    while (m) {
                        const int x = (w << 5) + __ffs(m) - 1;
                        m &= m - 1u;
                        const uint32_t *rx = rows + x * RS;
                        unsigned c = __popc(cm[0] & rx[0]);
                        if (W > 1) c += __popc(cm[1] & rx[1]);
                        if (W > 2) c += __popc(cm[2] & rx[2]);
                        if (W > 3) c += __popc(cm[3] & rx[3]);
                        a32 += c;
                    }
                }
            }
            a += a32;
        } else if (WPL == 1) {
            // word-sparse: only words where C & row v is nonzero matter
            uint32_t nzm = 0;
            for (int w = 0; w < W; ++w) nzm |= (cbuf[w] & rv[w]) ? (1u << w) : 0u;
            uint32_t ws = nzm;
            while (ws) {
                const int w = __ffs(ws) - 1;
                ws &= ws - 1u;
                uint32_t m = cbuf[w] & rv[w];
                x_seen += __popc(m);
                while (m) {
                    const int x = (w << 5) + __ffs(m) - 1;
                    m &= m - 1u;
                    const uint32_t *rx = rows + x * RS;
                    uint32_t w2s = nzm;
                    int c = 0;
                    while (w2s) {
                        const int w2 = __ffs(w2s) - 1;
                        w2s &= w2s - 1u;
                        c += __popc(cbuf[w2] & rv[w2] & rx[w2]);
                    }
                    a += c;
                }
            }
        } else {
            for (int w = 0; w < W; ++w) {
                uint32_t m = cbuf[w] & rv[w];
                x_seen += __popc(m);
                while (m) {
                    const int x = (w << 5) + __ffs(m) - 1;
                    m &= m - 1u;
                    const uint32_t *rx = rows + x * RS;
                    int c = 0;
                    for (int w2 = 0; w2 < W; ++w2) c += __popc(cbuf[w2] & rv[w2] & rx[w2]);
                    a += c;
                }
            }
        }
        acc += a;
        visits += x_seen;
        work += ull(1 + x_seen);
    }
    __syncwarp();
}

// argmax over v in C of popc(C & row v), lowest v on ties (engine_pivot.py:82-101)
template <int WPL>
__device__ __forceinline__ int select_pivot(const uint32_t *__restrict__ rows, int RS,
                                            const Set<WPL> &C, int *list, int lane, ull &work,
                                            int W) {
    const int n = compact<WPL>(C, list, lane, W);
    ull best = 0;
    for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        const bool ok = i < n;
        const int v = ok ? list[i] : 0;
        const int cov = cover<WPL>(rows, RS, C, v, ok);
        const ull key = ok ? ((ull(cov + 1) << 32) | ull(0xffffffffu - uint32_t(v))) : 0ull;
        best = key > best ? key : best;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const ull y = __shfl_xor_sync(FULL, best, o);
        best = y > best ? y : best;
    }
    if (lane == 0) work += ull(n);
    __syncwarp();
    return int(0xffffffffu - uint32_t(best & 0xffffffffull));
}

// ---------------------------------------------------------------------------
// S-tier: sets of at most 32 members.  Once a candidate set X is that small,
// its members are relabelled 0..n-1 in ascending local id (order, and hence
// every tie-break, is preserved) and the induced rows are compressed to one
// 32-bit word each (srow[i], per-warp shared memory; lane i also keeps its
// own row in a register).  The rest of the subtree then runs on uniform
// 32-bit scalars: next vertex = __ffs, child = one AND, pivot choice = one
// POPC per lane + __reduce_max_sync, last two orientation levels = per-lane
// bit loops.  The reference's visit order and counts are unchanged.
// ---------------------------------------------------------------------------
template <int WPL>
__device__ __forceinline__ int warp_count(const Set<WPL> &X) {
    return int(__reduce_add_sync(FULL, unsigned(popc_set<WPL>(X))));
}

// compress X (|X| <= 32) into srow; returns n; lane i (< n) row in *myrow
template <int WPL>
__device__ __forceinline__ int compress(const uint32_t *__restrict__ rows, int RS,
                                        const Set<WPL> &X, int *list, uint32_t *srow, int lane,
                                        uint32_t &myrow, int W = 32 * WPL) {
    const int n = compact<WPL>(X, list, lane, W);
    uint32_t r = 0;
    if (lane < n) {
        const uint32_t *rc = rows + list[lane] * RS;
        for (int j = 0; j < n; ++j) {
            const int cj = list[j];
            r |= ((rc[cj >> 5] >> (cj & 31)) & 1u) << j;
        }
    }
    srow[lane] = r;
    myrow = r;
    __syncwarp();
    return n;
}

// ---------------------------------------------------------------------------
// Sub-warp groups for the orientation engine's S-tier.
//
// In a compressed (<= 32 member) subtree the levels above the last two are
// walked by the whole warp as uniform scalar code; the last two levels --
// where almost all visits are -- are split over sub-warp groups of G lanes
// (G = 32, 16, 8, 4, 2, 1): at a frame (C, R) of level last-2 the 32/G groups
// take different children v of R (id stripes), and the G lanes of a group
// split the members x of that child's set X = C & row(v) (id stripes again);
// each lane adds popc(X & row x & row y) over y in X & row x through the
// carry-save accumulator.  G = 32 is one child at a time over the whole warp
// (pairs_small); G = 1 is one child per lane.  Counts and visits are sums, so
// they do not depend on G (engine_orient.py:32-79: visit = node expanded,
// last level = popcount).
// ---------------------------------------------------------------------------
template <int NW>
struct Bits {
    uint32_t w[NW];
};

template <int NW>
__device__ __forceinline__ Bits<NW> bits_all(int d) {
    Bits<NW> b;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        const int lo = i << 5;
        b.w[i] = lo >= d ? 0u : (lo + 32 <= d ? FULL : ((1u << (d - lo)) - 1u));
    }
    return b;
}

template <int NW>
__device__ __forceinline__ Bits<NW> bits_row(const uint32_t *__restrict__ rows, int v) {
    Bits<NW> b;
    if (NW == 4) {
        const uint4 r = *reinterpret_cast<const uint4 *>(rows + (v << 2));
        b.w[0] = r.x;
        b.w[NW > 1 ? 1 : 0] = r.y;
        b.w[NW > 2 ? 2 : 0] = r.z;
        b.w[NW > 3 ? 3 : 0] = r.w;
    } else {
        b.w[0] = rows[v];
    }
    return b;
}

template <int NW>
__device__ __forceinline__ Bits<NW> bits_and(const Bits<NW> &a, const Bits<NW> &b) {
    Bits<NW> c;
#pragma unroll
    for (int i = 0; i < NW; ++i) c.w[i] = a.w[i] & b.w[i];
    return c;
}

template <int NW>
__device__ __forceinline__ bool bits_any(const Bits<NW> &a) {
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) x |= a.w[i];
    return x != 0;
}

template <int NW>
__device__ __forceinline__ unsigned bits_popc(const Bits<NW> &a) {
    unsigned c = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) c += unsigned(__popc(a.w[i]));
    return c;
}

// highest member, removed from a (a must be nonempty)
template <int NW>
__device__ __forceinline__ int bits_pop_top(Bits<NW> &a) {
#pragma unroll
    for (int i = NW - 1; i > 0; --i) {
        if (a.w[i]) {
            const int b = 31 - __clz(a.w[i]);
            a.w[i] ^= 1u << b;
            return (i << 5) + b;
        }
    }
    const int b = 31 - __clz(a.w[0]);
    a.w[0] ^= 1u << b;
    return b;
}

// bits b of a 32-bit word with b % n == r (n a power of two dividing 32)
__device__ __forceinline__ uint32_t stripe32(int n, int r) {
    uint32_t m = 0;
    for (int b = r; b < 32; b += n) m |= 1u << b;
    return m;
}

template <int NW>
__device__ __forceinline__ Bits<NW> bits_stripe(const Bits<NW> &a, uint32_t s) {
    Bits<NW> c;
#pragma unroll
    for (int i = 0; i < NW; ++i) c.w[i] = a.w[i] & s;
    return c;
}

template <int NW>
__device__ __forceinline__ Bits<NW> bits_shfl(const Bits<NW> &a, int src) {
    Bits<NW> c;
#pragma unroll
    for (int i = 0; i < NW; ++i) c.w[i] = __shfl_sync(FULL, a.w[i], src);
    return c;
}

// the last two levels below the members xs of X (xs = this lane's share):
// per x a visit, X & row x its child set (each member a visit), and
// popc(X & row x & row y) cliques per y in it
template <int NW>
__device__ __forceinline__ void score_share(const uint32_t *__restrict__ rows, const Bits<NW> &X,
                                            Bits<NW> xs, unsigned &a, unsigned &vs) {
    while (bits_any<NW>(xs)) {
        const int x = bits_pop_top<NW>(xs);
        const Bits<NW> cm = bits_and<NW>(X, bits_row<NW>(rows, x));
        vs += 1u + bits_popc<NW>(cm);
        CsaAcc h;
        Bits<NW> m = cm;
        if (NW == 1) {
            uint32_t mm = m.w[0];
            while (mm) {  // two members per trip: independent loads in flight
                const int y0 = 31 - __clz(mm);
                mm ^= 1u << y0;
                const uint32_t r0 = rows[y0];
                uint32_t r1 = 0;
                if (mm) {
                    const int y1 = 31 - __clz(mm);
                    mm ^= 1u << y1;
                    r1 = rows[y1];
                }
                h.add2(cm.w[0] & r0, cm.w[0] & r1);
            }
        } else {
            while (bits_any<NW>(m)) {
                const int y = bits_pop_top<NW>(m);
                const Bits<NW> r = bits_row<NW>(rows, y);
                h.add4(cm.w[0] & r.w[0], cm.w[NW > 1 ? 1 : 0] & r.w[NW > 1 ? 1 : 0],
                       cm.w[NW > 2 ? 2 : 0] & r.w[NW > 2 ? 2 : 0],
                       cm.w[NW > 3 ? 3 : 0] & r.w[NW > 3 ? 3 : 0]);
            }
        }
        a += h.total();
    }
}

// children v of R under frame C (level last-2), split over sub-warp groups
template <int G, int NW>
__device__ __forceinline__ void pair_batch(const uint32_t *__restrict__ rows, const Bits<NW> &C,
                                           const Bits<NW> &R, int lane, ull &acc, ull &visits) {
    constexpr int NG = 32 / G;
    const Bits<NW> mine = bits_stripe<NW>(R, stripe32(NG, lane / G));
    const uint32_t xstripe = stripe32(G, lane % G);
    unsigned a = 0, vs = 0;
    Bits<NW> gen = mine;
    while (bits_any<NW>(gen)) {
        const int v = bits_pop_top<NW>(gen);
        const Bits<NW> X = bits_and<NW>(C, bits_row<NW>(rows, v));
        score_share<NW>(rows, X, bits_stripe<NW>(X, xstripe), a, vs);
    }
    acc += a;
    visits += vs;
}

// orientation, last two levels over compressed set C (C = frame last-1)
__device__ __forceinline__ void pairs_small(const uint32_t *srow, uint32_t C, int lane, ull &acc,
                                            ull &visits, ull &work) {
    // each member gets 32 / pow2ceil(|C|) lanes; the lanes of a member split
    // its walk over C & row v by member id
    const int cnt = __popc(C);
    const int lg = lanes_per_member_log2(cnt);
    const int mi = lane >> lg, sub = lane & ((1 << lg) - 1);
    if (mi < cnt) {
        const int v = nth_bit(C, mi);
        const uint32_t cm = C & srow[v];
        if (sub == 0) {
            const int xs = __popc(cm);
            visits += ull(1 + xs);
            work += ull(1 + xs);
        }
        uint32_t m = cm & id_stripe(lg, sub);
        // two members per trip: independent shared loads in flight; the
        // words go through CsaAcc (one POPC per four members)
        CsaAcc h;
        while (m) {
            const int x0 = 31 - __clz(m);
            m ^= 1u << x0;
            const uint32_t r0 = srow[x0];
            uint32_t r1 = 0;
            if (m) {
                const int x1 = 31 - __clz(m);
                m ^= 1u << x1;
                r1 = srow[x1];
            }
            h.add2(cm & r0, cm & r1);
        }
        acc += ull(h.total());
    }
}

// orientation walk of a compressed subtree; C is frame s (s <= last - 1).
// The scalar frame stack lives in registers: lane j holds frame s0+j (the
// depth of a <= 32-member subtree is < 32), pushed with a predicated move and
// popped with two shuffles -- no shared memory, no warp barrier.
template <int G = 32>
__device__ void orient_small(const uint32_t *srow, uint32_t C, int s, int last, uint32_t *sstk,
                             int lane, ull &acc, ull &visits, ull &work) {
    (void)sstk;
    if (s == last - 1) {
        pairs_small(srow, C, lane, acc, visits, work);
        __syncwarp();
        return;
    }
    const int s0 = s;
    uint32_t R = C;
    uint32_t fC = 0, fR = 0;  // this lane's frame (depth s0 + lane)
    unsigned uvis = 0;        // uniform visit count of the sequential levels
    for (;;) {
        if (G < 32 && s + 2 == last) {
            // the children of this frame are scored by sub-warp groups
            const ull v0 = visits;
            Bits<1> c1, r1;
            c1.w[0] = C;
            r1.w[0] = R;
            pair_batch<G, 1>(srow, c1, r1, lane, acc, visits);
            work += visits - v0;
            uvis += unsigned(__popc(R));
            R = 0;
            __syncwarp();
        }
        if (R == 0) {
            if (s == s0) break;
            --s;
            C = __shfl_sync(FULL, fC, s - s0);
            R = __shfl_sync(FULL, fR, s - s0);
            continue;
        }
        // orientation counts and visits do not depend on the branch order:
        // take the top member (one FLO, no BREV)
        const int v = 31 - __clz(R);
        R ^= 1u << v;
        ++uvis;
        const uint32_t X = C & srow[v];
        if (!X) continue;
        if (s + 2 == last) {
            pairs_small(srow, X, lane, acc, visits, work);
            __syncwarp();
            continue;
        }
        if (lane == s - s0) {
            fC = C;
            fR = R;
        }
        ++s;
        C = X;
        R = X;
    }
    if (lane == 0) {
        visits += uvis;
        work += uvis;
    }
}

__device__ __forceinline__ int select_small(uint32_t C, uint32_t myrow, int lane) {
    const unsigned key = ((C >> lane) & 1u) ? ((unsigned(__popc(C & myrow)) + 1u) << 5) |
                                                  unsigned(31 - lane)
                                            : 0u;
    return 31 - int(__reduce_max_sync(FULL, key) & 31u);
}

// Pivot leaves are binned per (path length, pivot count).  Each warp owns a
// u32 histogram for len < kLeafHL in shared memory, written by lane 0 only --
// no atomics (64-bit shared atomicAdd is a CAS spin loop on sm_100) -- and
// flushed to the global u64 L x L histogram at 2^31 and at kernel end.
constexpr int kLeafHL = 32;
constexpr int kLeafCells = kLeafHL * (kLeafHL + 1) / 2;

// ---------------------------------------------------------------------------
// GPU-wide subtree queue (pivot engine).  A busy warp that creates a child
// set X of kPushMin..kGItemMax members while some warp of the warp-tier
// kernel is hungry hands X over as an explicit, self-contained item: the
// sorted GLOBAL vertex ids of X plus (depth, pivot count).  The thief builds
// the sub-graph induced by exactly those vertices (ascending compact id, so
// the relabelling preserves the reference's order and tie-breaks) and walks
// X's subtree -- no dependence on the donor's task or bitmap.  Protocol
// (stack slots under one global spin lock, low traffic; the `busy` and
// `hungry` counters only ever change by atomics): `busy` counts warps that
// may still push, `hungry` counts warps waiting for items; a hungry warp
// leaves only under the lock with the stack empty, so a pusher -- which
// re-checks `hungry` under the lock -- can never strand an item.
// ---------------------------------------------------------------------------
constexpr int kGItemMax = 128;
constexpr int kGItemWords = 4 + kGItemMax;  // [n | X][s][npv][kind][ids | srow]
// item kinds: 0 = sorted global vertex ids (the thief rebuilds the induced
// sub-graph); 1 = compressed S-tier subtree: the 32 compressed rows travel
// with the set X, so the thief only copies 32 words
constexpr int kPushMin = 12;      // smaller children are cheaper to walk than to rebuild
constexpr int kPushCooldown = 256;  // child decisions between two hand-overs of one warp
constexpr int kPushRoom = 4;        // hand over only where >= 4 levels remain to target t
struct GQueue {
    uint32_t *items;  // cap x kGItemWords
    int *ctl;         // [0] lock [1] size [2] hungry [3] busy [4] pushes [5] pops [6] closed
    int cap;
    __device__ __forceinline__ void acquire() const {
        while (atomicCAS(ctl, 0, 1) != 0) __nanosleep(64);
        __threadfence();
    }
    __device__ __forceinline__ void release() const {
        __threadfence();
        atomicExch(ctl, 0);
    }
    __device__ __forceinline__ int vol(int i) const { return *(volatile int *)(ctl + i); }
    __device__ __forceinline__ void set(int i, int v) const { *(volatile int *)(ctl + i) = v; }
};

// ---------------------------------------------------------------------------
// Bounded pivot walks with spilling (round-based work distribution).  A walk
// (one task, or one spilled item) may expand at most `budget` branches; past
// that, every pending child -- the frames' remaining branches, the per-lane
// node stack -- is written out as a self-contained ITEM instead of being
// walked, and the next round's launches walk the items (again bounded).  A
// subtree of X depends only on the sub-graph induced by X and on (depth,
// pivot count), so visits and leaves are exactly the unbounded walk's
// (engine_pivot.py:117-233); only who walks which subtree changes.  Items:
//   kind 0: [0, n, s, npv] + the n global vertex ids of X, ascending;
//           n <= big_thr -> small list (warp tier), else big list (CTA tier)
//   kind 2: [2, m, 0, 0] + 32 compressed rows + m nodes (C, s | npv << 16)
//           of one S-tier universe (the per-lane walk's pending stack)
// Offsets are appended with atomics; a full buffer makes the emitter walk
// the child itself (never lost, only slower).
// ---------------------------------------------------------------------------
constexpr int kSpillBatch = 64;  // S-tier nodes per kind-2 item
struct Spill {
    uint32_t *buf;     // item words
    ull *ctl;          // [0] word cursor [1] small items [2] big items [3] failed [4] max big n
    uint32_t *small_off, *big_off;
    ull cap_words;
    uint32_t cap_small, cap_big;
    int big_thr;
    // lane 0: reserve an item of `words` words; ~0u when full
    __device__ __forceinline__ uint32_t reserve(int words, bool big, int n) const {
        const ull off = atomicAdd(&ctl[0], ull(words));
        if (off + ull(words) > cap_words) {
            atomicAdd(&ctl[3], 1ull);
            return 0xffffffffu;
        }
        const ull idx = atomicAdd(&ctl[big ? 2 : 1], 1ull);
        if (idx >= ull(big ? cap_big : cap_small)) {
            atomicAdd(&ctl[3], 1ull);
            return 0xffffffffu;
        }
        (big ? big_off : small_off)[idx] = uint32_t(off);
        if (big) atomicMax(&ctl[4], ull(n));
        return uint32_t(off);
    }
};

struct PivotLeafSink {
    uint32_t *whist;  // this warp's kLeafCells counters
    ull *g_hist;      // global L x L histogram
    int L;
    // GPU-wide work sharing (nullptr: off)
    const GQueue *gq;
    bool eager;          // CTA tier: push large children without rate limit
    const int32_t *l2g;  // local id -> global vertex id of the current universe
    int *hc;             // per-warp smem: [0] countdown [1] cached hungry
    int push_min = kPushMin, cooldown = kPushCooldown, room_min = kPushRoom;
    // bounded walks (nullptr: unbounded).  hc[2] = remaining budget of this
    // warp's walk, hc[3] = 1 after a failed emission (walk on unbounded);
    // cta_flag: CTA tier -- once one warp of the task is over budget, all are
    const Spill *sp = nullptr;
    int *cta_flag = nullptr;
    __device__ __forceinline__ void set_budget(int b, int lane) const {
        if (lane == 0) {
            hc[2] = b;
            hc[3] = 0;
        }
        __syncwarp();
    }
    // uniform: charge n expanded branches; true once the budget is spent
    __device__ __forceinline__ bool spend(int n, int lane) const {
        if (!sp) return false;
        int r = 0;
        if (lane == 0) {
            if (hc[3]) {
                r = 1;
            } else {
                r = (hc[2] -= n);
                if (cta_flag) {
                    if (r < 0) *(volatile int *)cta_flag = 1;
                    else if (*(volatile int *)cta_flag) r = -1;
                }
            }
        }
        return __shfl_sync(0xffffffffu, r, 0) < 0;
    }
    __device__ __forceinline__ void no_spill(int lane) const {
        if (lane == 0) hc[3] = 1;
        __syncwarp();
    }
    // kind-0 item: the global ids of X (lane-distributed over this universe)
    template <int WPL>
    __device__ __forceinline__ bool spill_ids(const Set<WPL> &X, int n, int s, int npv, int *list,
                                              int lane) const;
    // kind-2 item: an S-tier universe (32 compressed rows) with nb pending nodes
    __device__ __forceinline__ bool spill_batch(const uint32_t *srow, const uint2 *nodes, int nb,
                                                int lane) const {
        uint32_t off = 0;
        if (lane == 0) off = sp->reserve(4 + 32 + 2 * nb, false, 0);
        off = __shfl_sync(0xffffffffu, off, 0);
        if (off == 0xffffffffu) return false;
        uint32_t *it = sp->buf + off;
        if (lane == 0) {
            it[0] = 2u;
            it[1] = uint32_t(nb);
            it[2] = 0u;
            it[3] = 0u;
        }
        it[4 + lane] = srow[lane];
        for (int i = lane; i < nb; i += 32) {
            const uint2 nd = nodes[i];
            it[36 + 2 * i] = nd.x;
            it[37 + 2 * i] = nd.y;
        }
        __syncwarp();
        return true;
    }
    // uniform: should a child of n members be handed to a hungry warp?
    // Rate-limited: at most one hand-over per kPushCooldown decisions, so a
    // donor keeps doing its own work and thieves get substantial subtrees.
    __device__ __forceinline__ bool want_push(int n, int room, int lane) const {
        if (!gq || n < push_min || n > kGItemMax) return false;
        if (eager) {
            // CTA tier: hand every large (L-tier) child to a hungry warp-tier
            // warp -- its W <= 4 universe walks it far cheaper than this one
            if (n <= 32) return false;
        } else if (room < room_min) {
            return false;  // shallow remaining tree: cheaper to walk
        }
        if (lane == 0 && --hc[0] <= 0) {
            hc[0] = eager ? 16 : cooldown;
            hc[1] = gq->vol(2);
        }
        __syncwarp();
        const bool w = hc[1] > 0;
        __syncwarp();
        if (w && lane == 0 && !eager) hc[1] = 0;  // one hand-over per cooldown window
        return w;
    }
    // reserve a slot (lock held by lane 0 on success); -1 when full / nobody hungry
    __device__ __forceinline__ int reserve(int lane) const {
        int slot = -1;
        if (lane == 0) {
            gq->acquire();
            // only while more warps are hungry than items are waiting
            const int sz = gq->vol(1);
            if (!gq->vol(6) && sz < gq->cap && sz < gq->vol(2)) slot = sz;  // [6]: closed
            else gq->release();
        }
        return __shfl_sync(0xffffffffu, slot, 0);
    }
    __device__ __forceinline__ void publish(int slot, int n, int s, int npv, int lane) const {
        uint32_t *it = gq->items + int64_t(slot) * kGItemWords;
        if (lane == 0) {
            it[0] = uint32_t(n);
            it[1] = uint32_t(s);
            it[2] = uint32_t(npv);
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            gq->set(1, slot + 1);
            atomicAdd(gq->ctl + 4, 1);  // pushes (diagnostics)
            gq->release();
        }
        __syncwarp();
    }
    // compressed S-tier child X over the compressed rows srow
    __device__ __forceinline__ bool push_compressed(const uint32_t *srow, uint32_t X, int s,
                                                    int npv, int lane) const {
        const int slot = reserve(lane);
        if (slot < 0) return false;
        uint32_t *it = gq->items + int64_t(slot) * kGItemWords;
        it[4 + lane] = srow[lane];
        if (lane == 0) it[3] = 1u;
        publish(slot, int(X), s, npv, lane);
        return true;
    }
    // S-tier child X (compressed ids; map = compressed -> local, nullptr = identity)
    __device__ __forceinline__ bool push_small(uint32_t X, const int *map, int s, int npv,
                                               int lane) const {
        const int slot = reserve(lane);
        if (slot < 0) return false;
        uint32_t *ids = gq->items + int64_t(slot) * kGItemWords + 4;
        if (lane == 0) ids[-1] = 0u;  // kind 0
        if ((X >> lane) & 1u) {
            const int local = map ? map[lane] : lane;
            ids[__popc(X & ((1u << lane) - 1u))] = uint32_t(l2g[local]);
        }
        publish(slot, __popc(X), s, npv, lane);
        return true;
    }
    __device__ __forceinline__ void add(int len, int np) const {
        if (len < kLeafHL) {
            uint32_t &c = whist[len * (len + 1) / 2 + np];
            if (++c == 0x80000000u) {
                atomicAdd(&g_hist[int64_t(len) * L + np], 0x80000000ull);
                c = 0;
            }
        } else {
            atomicAdd(&g_hist[int64_t(len) * L + np], 1ull);
        }
    }
    // any lane, concurrently with other lanes (per-lane walks): 32-bit shared
    // atomics (native), the cell handed to the global u64 histogram at 2^31
    __device__ __forceinline__ void add_atomic(int len, int np) const {
        if (len < kLeafHL) {
            uint32_t *c = &whist[len * (len + 1) / 2 + np];
            if (atomicAdd(c, 1u) == 0x7fffffffu) {
                atomicAdd(&g_hist[int64_t(len) * L + np], 0x80000000ull);
                atomicSub(c, 0x80000000u);
            }
        } else {
            atomicAdd(&g_hist[int64_t(len) * L + np], 1ull);
        }
    }
    // whole warp: add the per-warp counters to the global histogram
    __device__ __forceinline__ void flush(int lane) const {
        __syncwarp();
        for (int i = lane; i < kLeafCells; i += 32) {
            const uint32_t x = whist[i];
            if (!x) continue;
            int len = int((sqrtf(8.0f * i + 1.0f) - 1.0f) * 0.5f);
            while (len * (len + 1) / 2 > i) --len;
            while ((len + 1) * (len + 2) / 2 <= i) ++len;
            const int np = i - len * (len + 1) / 2;
            atomicAdd(&g_hist[int64_t(len) * L + np], ull(x));
            whist[i] = 0;
        }
        __syncwarp();
    }
};

template <int WPL>
__device__ __forceinline__ bool PivotLeafSink::spill_ids(const Set<WPL> &X, int n, int s, int npv,
                                                        int *list, int lane) const {
    const bool big = n > sp->big_thr;
    uint32_t off = 0;
    if (lane == 0) off = sp->reserve(4 + n, big, n);
    off = __shfl_sync(0xffffffffu, off, 0);
    if (off == 0xffffffffu) return false;
    compact<WPL>(X, list, lane);
    uint32_t *it = sp->buf + off;
    if (lane == 0) {
        it[0] = 0u;
        it[1] = uint32_t(n);
        it[2] = uint32_t(s);
        it[3] = uint32_t(npv);
    }
    for (int i = lane; i < n; i += 32) it[4 + i] = uint32_t(l2g[list[i]]);
    __syncwarp();
    return true;
}

// Take the lowest pending branch v of the shallowest stored frame (lane j
// holds frame s0+j; `depth` frames are stored) and hand its child to the
// queue.  A pruned / leaf / dead branch is consumed inline instead (it is
// ordinary work: a visit and maybe a leaf); when the queue refuses the item
// the branch is put back.  Ascending order within the frame is kept, so the
// reference's "pruned bits below v" rule (engine_pivot.py:158-166) holds.
template <typename Sink>
__device__ __forceinline__ void donate_bottom(const uint32_t *srow, const int *map, int depth,
                                              int s0, int t, bool allk, uint32_t fC, uint32_t fP,
                                              uint32_t &fR, uint32_t fPN, const Sink &sink,
                                              int lane, unsigned &uvis) {
    const unsigned has = __ballot_sync(FULL, lane < depth && fR != 0);
    if (!has) return;
    const int j = __ffs(has) - 1;
    const uint32_t jC = __shfl_sync(FULL, fC, j), jP = __shfl_sync(FULL, fP, j);
    const uint32_t jR = __shfl_sync(FULL, fR, j), pn = __shfl_sync(FULL, fPN, j);
    const int v = __ffs(jR) - 1;
    if (lane == j) fR = jR & (jR - 1u);
    const int sj = s0 + j, jpiv = int(pn & 0xffu), jnpv = int(pn >> 8);
    const int np2 = jnpv + (v == jpiv ? 1 : 0);
    if (!allk && sj + 1 - t > np2) return;  // pruned: not a visit
    const uint32_t X = jC & srow[v] & ~(jP & ((1u << v) - 1u));
    if (!X) {
        ++uvis;
        if ((allk || sj + 1 >= t) && lane == 0) sink.add(sj + 1, np2);
        return;
    }
    if (!allk && sj + 2 - t > np2 + 1) {  // dead child
        ++uvis;
        return;
    }
    if (__popc(X) >= sink.push_min && sink.push_compressed(srow, X, sj + 1, np2, lane)) {
        ++uvis;
        return;
    }
    if (lane == j) fR = jR;  // refused: the branch stays with this warp
}

// pivot walk of a compressed subtree rooted at a fresh child set C (frame s,
// pivot count npv).  Frame stack in registers (lane j = frame s0+j, see
// orient_small); visit / work counters uniform, added by lane 0 at the end.
template <typename Sink>
__device__ void pivot_small(const uint32_t *srow, uint32_t myrow, uint32_t C, int s, int npv,
                            int t, bool allk, uint32_t *sstk, const Sink &sink, int lane,
                            ull &visits, ull &work, const int *map = nullptr) {
    (void)sstk;
    const int s0 = s;
    int piv = select_small(C, myrow, lane);
    uint32_t P = C & ~srow[piv];
    // engine_pivot.py:152-153 prunes branch v iff s+1-t > npv + [v == piv]:
    // a frame with deficit npv+1 can only branch on its pivot (always in P)
    uint32_t R = (!allk && s + 1 - t > npv) ? (P & (1u << piv)) : P;
    unsigned uvis = 0, uwork = unsigned(__popc(C));
    uint32_t fC = 0, fP = 0, fR = 0, fPN = 0;  // this lane's frame; fPN = piv | npv << 8
    for (;;) {
        if (R == 0) {
            if (s == s0) break;
            --s;
            const int j = s - s0;
            C = __shfl_sync(FULL, fC, j);
            P = __shfl_sync(FULL, fP, j);
            R = __shfl_sync(FULL, fR, j);
            const uint32_t pn = __shfl_sync(FULL, fPN, j);
            piv = int(pn & 0xffu);
            npv = int(pn >> 8);
            continue;
        }
        const int v = __ffs(R) - 1;
        R &= R - 1u;
        const int np2 = npv + (v == piv ? 1 : 0);
        if (!allk && s + 1 - t > np2) continue;
        ++uvis;
        const uint32_t X = C & srow[v] & ~(P & ((1u << v) - 1u));
        if (X) {
            // a child whose every branch would be pruned adds neither visits
            // nor leaves: do not build it
            if (!allk && s + 2 - t > np2 + 1) continue;
            // GPU-wide work sharing: while some warp is hungry, donate the
            // SHALLOWEST pending branch (the biggest subtree this warp still
            // owns), classic work stealing from the bottom of the stack
            if (sink.gq && s > s0 && sink.want_push(sink.push_min, allk ? 1 << 20 : t - s0, lane))
                donate_bottom(srow, map, s - s0, s0, t, allk, fC, fP, fR, fPN, sink, lane, uvis);
            if (lane == s - s0) {
                fC = C;
                fP = P;
                fR = R;
                fPN = uint32_t(piv) | (uint32_t(npv) << 8);
            }
            ++s;
            npv = np2;
            C = X;
            piv = select_small(C, myrow, lane);
            P = C & ~srow[piv];
            R = (!allk && s + 1 - t > npv) ? (P & (1u << piv)) : P;
            uwork += unsigned(__popc(C));
        } else if (allk || s + 1 >= t) {
            if (lane == 0) sink.add(s + 1, np2);
        }
    }
    if (lane == 0) {
        visits += uvis;
        work += ull(uvis) + uwork;
    }
}

// Per-lane walk of a compressed (<= 32 member) pivot subtree: sub-warp
// groups of ONE lane (pivoting favours group size 1,
// PAPER.md:720).  Pending nodes (C, s | npv << 8) sit in a per-warp stack in
// shared memory; every round each lane pops one node and expands it itself --
// pivot = argmax |C & row v| over v in C (lowest id on ties,
// engine_pivot.py:82-101), P = C \ row(pivot), the branches of P under the
// pruning rule (engine_pivot.py:152-153), child C & row v minus the pruned
// bits below v (:158-166), leaves binned by (length, pivots) -- and the
// children are pushed back (counted first, then written at scanned offsets).
// 32 nodes advance per round instead of one; counts and visits are sums over
// nodes, so the traversal order does not change them.  When the stack is
// nearly full a node's subtree is walked by the uniform path instead; while
// some warp is hungry the bottom (shallowest) node is handed to the GPU-wide
// queue as a compressed item.
// nstk[0..size) already holds the pending nodes (a spilled batch, or the root)
template <typename Sink>
__device__ void pivot_lanes_run(const uint32_t *srow, int size, int t, bool allk, uint2 *nstk,
                                int ncap, const Sink &sink, int lane, ull &visits, ull &work) {
    unsigned vis = 0, wk = 0, vis0 = 0;
    // srow and nstk live in shared memory: explicit ld/st.shared (through the
    // generic pointers the compiler emitted LD.E, long-scoreboard waits)
    const unsigned sb = smem_addr(srow), nb0 = smem_addr(nstk);
    auto row = [&](int v) { return lds32(sb + 4u * unsigned(v)); };
    auto node = [&](int i) { return lds64(nb0 + 8u * unsigned(i)); };
    const uint32_t myrow = row(lane);
    const bool sp_on = sink.sp != nullptr, gq_on = sink.gq != nullptr;
    int rounds = 0;
    for (;;) {
        if (size == 0) break;
        if (sp_on && (++rounds & 7) == 0) {
            // bounded walk: charge the branches of the last 8 rounds; once the
            // budget is spent the whole pending stack leaves as kind-2 items
            const int rv = int(__reduce_add_sync(FULL, vis - vis0));
            vis0 = vis;
            if (sink.spend(rv, lane)) {
                while (size > 0) {
                    const int nb = size < kSpillBatch ? size : kSpillBatch;
                    if (!sink.spill_batch(srow, nstk + size - nb, nb, lane)) break;
                    size -= nb;
                }
                if (size == 0) break;
                sink.no_spill(lane);  // buffer full: walk the rest here
            }
        }
        if (gq_on && size >= 2 && sink.want_push(sink.push_min, 1 << 20, lane)) {
            const uint2 nb = node(0);  // bottom: the shallowest pending node
            if (__popc(nb.x) >= sink.push_min &&
                sink.push_compressed(srow, nb.x, int(nb.y & 0xffffu), int(nb.y >> 16), lane)) {
                __syncwarp();
                if (lane == 0) sts64(nb0, node(size - 1));
                __syncwarp();
                --size;
                continue;
            }
        }
        const int free_slots = ncap - size;
        // take the top k nodes whose children fit: a node pushes at most |C|
        // children (its branches are members of C), so k is the longest run
        // of top nodes with sum |C| <= free slots (deep nodes are small: most
        // rounds run all 32 lanes; the old bound of 32 children per node
        // allowed at most ncap / 32 = 16)
        const int cand = size < 32 ? size : 32;
        const uint2 ndc = lane < cand ? node(size - 1 - lane) : make_uint2(0u, 0u);
        int need = lane < cand ? __popc(ndc.x) : (1 << 20);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, need, o);
            if (lane >= o) need += y;
        }
        const int k = __popc(__ballot_sync(FULL, need <= free_slots));
        if (k == 0) {
            // no room for the top node's children: walk it uniformly
            const uint32_t tc = __shfl_sync(FULL, ndc.x, 0), ty = __shfl_sync(FULL, ndc.y, 0);
            --size;
            pivot_small(srow, myrow, tc, int(ty & 0xffffu), int(ty >> 16), t, allk, nullptr, sink,
                        lane, visits, work);
            continue;
        }
        uint32_t C = 0;
        int s = 0, npv = 0;
        const bool have = lane < k;
        if (have) {
            C = ndc.x;
            s = int(ndc.y & 0xffffu);
            npv = int(ndc.y >> 16);
        }
        size -= k;
        __syncwarp();
        int piv = 0, nch = 0;
        uint32_t P = 0, R = 0;
        if (have) {
            // pivot: argmax popc(C & row v), lowest v on ties
            unsigned best = 0;
            uint32_t m = C;
            while (m) {
                const int v = __ffs(m) - 1;
                m &= m - 1u;
                const unsigned key = ((unsigned(__popc(C & row(v))) + 1u) << 5) | unsigned(31 - v);
                best = key > best ? key : best;
            }
            piv = 31 - int(best & 31u);
            wk += unsigned(__popc(C));
            P = C & ~row(piv);
            R = (!allk && s + 1 - t > npv) ? (P & (1u << piv)) : P;
            // branches: visits, leaves, and the number of children to push
            uint32_t r = R;
            while (r) {
                const int v = __ffs(r) - 1;
                r &= r - 1u;
                const int np2 = npv + (v == piv ? 1 : 0);
                if (!allk && s + 1 - t > np2) continue;  // pruned: not a visit
                ++vis;
                const uint32_t X = C & row(v) & ~(P & ((1u << v) - 1u));
                if (X) {
                    if (!allk && s + 2 - t > np2 + 1) continue;  // every branch pruned
                    ++nch;
                } else if (allk || s + 1 >= t) {
                    sink.add_atomic(s + 1, np2);
                }
            }
        }
        int incl = nch;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        int at = size + incl - nch;
        size += __shfl_sync(FULL, incl, 31);
        if (nch) {
            uint32_t r = R;
            while (r) {
                const int v = __ffs(r) - 1;
                r &= r - 1u;
                const int np2 = npv + (v == piv ? 1 : 0);
                if (!allk && s + 1 - t > np2) continue;
                const uint32_t X = C & row(v) & ~(P & ((1u << v) - 1u));
                if (!X || (!allk && s + 2 - t > np2 + 1)) continue;
                sts64(nb0 + 8u * unsigned(at++), make_uint2(X, uint32_t(s + 1) | (uint32_t(np2) << 16)));
            }
        }
        __syncwarp();
    }
    visits += vis;
    work += ull(vis) + wk;
}

template <typename Sink>
__device__ void pivot_lanes(const uint32_t *srow, uint32_t C0, int s0, int npv0, int t, bool allk,
                            uint2 *nstk, int ncap, const Sink &sink, int lane, ull &visits,
                            ull &work) {
    if (lane == 0) nstk[0] = make_uint2(C0, uint32_t(s0) | (uint32_t(npv0) << 16));
    __syncwarp();
    pivot_lanes_run(srow, 1, t, allk, nstk, ncap, sink, lane, visits, work);
}

// ---------------------------------------------------------------------------
// frames
// ---------------------------------------------------------------------------
struct Frames {
    uint32_t *sm;  // frames [0, nsm)
    uint32_t *gm;  // frames [nsm, ...)
    int nsm;
    int fw;  // words per frame
    __device__ __forceinline__ uint32_t *at(int s) const {
        return s < nsm ? sm + s * fw : gm + int64_t(s - nsm) * fw;
    }
};

// per-warp scratch: compressed S-tier rows, and the hash table of the
// warp-tier sub-graph builder (kMapSlots int32 keys + kMapSlots u8 values)
struct SmallScratch {
    uint32_t *srow;  // 32 words
    uint32_t *sstk;  // kMapWords words: LocalMap storage
    uint2 *nstk = nullptr;  // pivot per-lane node stack (warp tier), nullptr: uniform walks
    int ncap = 0;
    uint32_t *mrow = nullptr;  // mid_words(WPL, mid_max): compressed pair level (CTA tier)
    int mid_max = 0;           // largest set compressed there (128 or 256)
};
// 256 rows of 8 words + the per-word compress table of a set (8 words per word)
constexpr int mid_words(int wpl, int mid_max) { return mid_rows_words(mid_max) + 8 * 32 * wpl; }
constexpr int kNodeCap = 512;  // pivot_lanes stack capacity (nodes of 2 words)
constexpr int kMapSlots = 256;
constexpr int kMapWords = kMapSlots + kMapSlots / 4;
constexpr int kSmallWords = 32 + kMapWords;

// global vertex id -> local index of the <= 128 sorted locals of a warp-tier
// task: open addressing, load factor <= 1/2, so a miss (most out-neighbours
// are not locals) costs ~2.5 probes instead of a 7-step binary search
struct LocalMap {
    int32_t *key;
    uint8_t *val;
    __device__ __forceinline__ static uint32_t slot(int32_t x) {
        return (uint32_t(x) * 0x9E3779B1u) >> 24;  // 8 bits: kMapSlots = 256
    }
    // whole warp; l2g[0..d) distinct, d <= kMapSlots / 2
    __device__ __forceinline__ void build(const int32_t *l2g, int d, int lane) const {
        for (int i = lane; i < kMapSlots; i += 32) key[i] = -1;
        __syncwarp();
        for (int i = lane; i < d; i += 32) {
            const int32_t x = l2g[i];
            uint32_t h = slot(x);
            while (atomicCAS(key + h, -1, x) != -1) h = (h + 1) & (kMapSlots - 1);
            val[h] = uint8_t(i);
        }
        __syncwarp();
    }
    __device__ __forceinline__ int find(int32_t x) const {
        uint32_t h = slot(x);
        for (;;) {
            const int32_t k = key[h];
            if (k == x) return val[h];
            if (k < 0) return -1;
            h = (h + 1) & (kMapSlots - 1);
        }
    }
};

// ---------------------------------------------------------------------------
// orient: one level-1 subtree (engine_orient.py:32-79).  The caller expanded
// root-level vertex u (and counted its visit); C = row(u) is frame 1.
// last = t - 2 >= 1.  Orient frame layout: [C: 32*WPL][cursor].
// ---------------------------------------------------------------------------
// hand a set X at frame s (s <= last-1) to the S-tier if it has <= 32
// members; returns false (nothing done) otherwise
template <int WPL, int G = 32>
__device__ __forceinline__ bool orient_try_small(const uint32_t *__restrict__ rows, int RS, int W,
                                                 const Set<WPL> &X, int s, int last, int *list,
                                                 const SmallScratch &S, int lane, ull &acc,
                                                 ull &visits, ull &work) {
    if (W == 1) {  // rows are already one word: identity relabelling
        orient_small<G>(rows, __shfl_sync(FULL, X.w[0], 0), s, last, S.sstk, lane, acc, visits,
                     work);
        return true;
    }
    if (warp_count<WPL>(X) > 32) return false;
    uint32_t myrow;
    const int n = compress<WPL>(rows, RS, X, list, S.srow, lane, myrow, W);
    orient_small<G>(S.srow, n == 32 ? FULL : ((1u << n) - 1u), s, last, S.sstk, lane, acc, visits,
                 work);
    return true;
}

template <int WPL, int G = 32>
__device__ void orient_subtree(const uint32_t *__restrict__ rows, int RS, int W, int last, int u,
                               const Frames &F, int *list, uint32_t *cbuf, const SmallScratch &SS,
                               ull &acc, ull &visits, ull &work) {
    const int lane = threadIdx.x & 31;
    Set<WPL> C = load_row<WPL>(rows, RS, W, u, lane);
    if (last == 1) {  // frame 1 is the last level
        visits += ull(popc_set<WPL>(C));
        score_sum<WPL>(rows, RS, C, list, lane, acc, work, W);
        return;
    }
    if (!any_set<WPL>(C)) return;
    if (orient_try_small<WPL, G>(rows, RS, W, C, 1, last, list, SS, lane, acc, visits, work))
        return;
    if (last == 2) {  // frame 1 is the next-to-last level
        if (W > 4 && SS.mrow && warp_count<WPL>(C) <= SS.mid_max)
            score_pairs_mid<WPL>(rows, RS, W, C, list, cbuf, SS.mrow, SS.mid_max, lane, acc,
                                 visits, work);
        else
            score_pairs<WPL>(rows, RS, W, C, list, cbuf, lane, acc, visits, work);
        return;
    }
    int s = 1;
    Set<WPL> R = C;
    store_set<WPL>(F.at(1), C, lane);
    const int cur = 32 * WPL;  // cursor word offset inside a frame
    for (;;) {
        const int v = next_bit<WPL>(R, lane);
        if (v < 0) {
            if (--s == 0) break;
            const uint32_t *f = F.at(s);
            C = load_set<WPL>(f, lane);
            const int c = int(f[cur]);
#pragma unroll
            for (int p = 0; p < WPL; ++p) R.w[p] = C.w[p] & above_mask(p * 32 + lane, c);
            continue;
        }
        if (lane == 0) {
            ++visits;
            work += 1;
        }
        Set<WPL> X;
        const uint32_t *rv = rows + v * RS;
#pragma unroll
        for (int p = 0; p < WPL; ++p) {
            const int w = p * 32 + lane;
            X.w[p] = w < W ? (C.w[p] & rv[w]) : 0u;
        }
        if (!any_set<WPL>(X)) continue;
        if (orient_try_small<WPL, G>(rows, RS, W, X, s + 1, last, list, SS, lane, acc, visits,
                                     work))
            continue;
        if (s + 2 == last) {  // X is the next-to-last frame
            if (W > 4 && SS.mrow && warp_count<WPL>(X) <= SS.mid_max)
                score_pairs_mid<WPL>(rows, RS, W, X, list, cbuf, SS.mrow, SS.mid_max, lane, acc,
                                     visits,
                                     work);
            else
                score_pairs<WPL>(rows, RS, W, X, list, cbuf, lane, acc, visits, work);
            continue;
        }
        uint32_t *f = F.at(s);
        if (lane == 0) f[cur] = uint32_t(v);
        ++s;
        C = X;
        R = X;
        store_set<WPL>(F.at(s), C, lane);
    }
}

// ---------------------------------------------------------------------------
// pivot: one root-level branch v0 (engine_pivot.py:117-233).  The caller
// passes the root frame's sets S0 (all locals) and P0 (branch set) via smem
// pointers.  Pivot frame layout: [C: 32*WPL][P: 32*WPL][piv, npv, cursor, -].
// Leaves are binned as hist[(path length, pivots)] (expanded exactly on the
// host).  t: target; allk: no stopping rule.
// ---------------------------------------------------------------------------

// hand a fresh child set X (frame s, pivot count npv) to the S-tier if it
// has <= 32 members
template <int WPL>
__device__ __forceinline__ bool pivot_try_small(const uint32_t *__restrict__ rows, int RS, int W,
                                                const Set<WPL> &X, int s, int npv, int t,
                                                bool allk, int *list, const SmallScratch &S,
                                                const PivotLeafSink &sink, int lane, ull &visits,
                                                ull &work) {
    if (W == 1) {  // rows are already one word: identity relabelling
        const uint32_t c = __shfl_sync(FULL, X.w[0], 0);
        if (S.nstk && RS == 1 && __isShared(rows)) {  // per-lane walks read rows as shared
            pivot_lanes(rows, c, s, npv, t, allk, S.nstk, S.ncap, sink, lane, visits, work);
            return true;
        }
        const uint32_t myrow = ((c >> lane) & 1u) ? rows[lane * RS] : 0u;
        pivot_small(rows, myrow, c, s, npv, t, allk, S.sstk, sink, lane, visits, work);
        return true;
    }
    if (warp_count<WPL>(X) > 32) return false;
    uint32_t myrow;
    const int n = compress<WPL>(rows, RS, X, list, S.srow, lane, myrow, W);
    if (S.nstk) {
        pivot_lanes(S.srow, n == 32 ? FULL : ((1u << n) - 1u), s, npv, t, allk, S.nstk, S.ncap,
                    sink, lane, visits, work);
        return true;
    }
    pivot_small(S.srow, myrow, n == 32 ? FULL : ((1u << n) - 1u), s, npv, t, allk, S.sstk, sink,
                lane, visits, work, list);
    return true;
}

// ---------------------------------------------------------------------------
// CTA-local work sharing for the pivot walk of a big task.  A warp that has
// run out of root branches parks as idle; a busy warp that creates an
// L-tier child while some warp is idle hands the child (its set, depth and
// pivot count -- everything the subtree needs) to a shared-memory stack
// instead of descending into it.  All state changes happen under a spin lock
// held by lane 0; termination = every warp idle and the stack empty.
// ---------------------------------------------------------------------------
struct StealStack {
    uint32_t *items;  // cap x iw words: [C: 32*WPL][s][npv]
    int *lock, *size, *idle;
    int cap, iw, nwarps;
    __device__ __forceinline__ void acquire() const {
        while (atomicCAS(lock, 0, 1) != 0) __nanosleep(32);
        __threadfence_block();
    }
    __device__ __forceinline__ void release() const {
        __threadfence_block();
        atomicExch(lock, 0);
    }
};

template <int WPL>
__device__ __forceinline__ bool steal_push(const StealStack &q, const Set<WPL> &X, int s, int npv,
                                           int lane) {
    // heuristic pre-check without the lock
    if (*(volatile int *)q.idle == 0 || *(volatile int *)q.size >= q.cap) return false;
    int slot = -1;
    if (lane == 0) {
        q.acquire();
        if (*(volatile int *)q.size < q.cap) slot = *(volatile int *)q.size;
        else q.release();
    }
    slot = __shfl_sync(FULL, slot, 0);
    if (slot < 0) return false;
    uint32_t *it = q.items + slot * q.iw;
    store_set<WPL>(it, X, lane);
    if (lane == 0) {
        it[32 * WPL] = uint32_t(s);
        it[32 * WPL + 1] = uint32_t(npv);
    }
    __syncwarp();
    if (lane == 0) {
        __threadfence_block();
        *(volatile int *)q.size = slot + 1;
        q.release();
    }
    __syncwarp();
    return true;
}

// hand an L-tier child X (local ids of the current universe) to the queue
template <int WPL>
__device__ __forceinline__ bool push_large(const PivotLeafSink &sink, const Set<WPL> &X, int *list,
                                           int s, int npv, int lane) {
    const int slot = sink.reserve(lane);
    if (slot < 0) return false;
    const int n = compact<WPL>(X, list, lane);
    uint32_t *ids = sink.gq->items + int64_t(slot) * kGItemWords + 4;
    if (lane == 0) ids[-1] = 0u;  // kind 0
    for (int i = lane; i < n; i += 32) ids[i] = uint32_t(sink.l2g[list[i]]);
    sink.publish(slot, n, s, npv, lane);
    return true;
}

// L-tier bottom-of-stack donation: find the shallowest stored frame sf in
// [s0, s_top) with a pending branch v, and hand v's child set to the queue as
// a global-id item (same rules as donate_bottom for the S-tier).  Frames keep
// (C, P, piv, npv, cursor); advancing the cursor to v marks v as taken.
template <int WPL>
__device__ __forceinline__ void donate_bottom_L(const uint32_t *__restrict__ rows, int RS, int W,
                                                int t, bool allk, const Frames &F, int s0,
                                                int s_top, int *list, const PivotLeafSink &sink,
                                                int lane, ull &visits) {
    const int PO = 32 * WPL, SC = 64 * WPL;
    for (int sf = s0; sf < s_top; ++sf) {
        uint32_t *f = F.at(sf - s0);
        const Set<WPL> Cf = load_set<WPL>(f, lane), Pf = load_set<WPL>(f + PO, lane);
        const int piv = int(f[SC]), npv = int(f[SC + 1]), c = int(f[SC + 2]);
        Set<WPL> R;
#pragma unroll
        for (int p = 0; p < WPL; ++p) R.w[p] = Pf.w[p] & above_mask(p * 32 + lane, c);
        if (!allk && sf + 1 - t > npv) restrict_to(R, piv, lane);
        const int v = next_bit<WPL>(R, lane);
        if (v < 0) continue;
        const int np2 = npv + (v == piv ? 1 : 0);
        if (!allk && sf + 1 - t > np2) {  // pruned (not a visit): just take it
            __syncwarp();
            if (lane == 0) f[SC + 2] = uint32_t(v);
            __syncwarp();
            return;
        }
        Set<WPL> X;
        const uint32_t *rv = rows + v * RS;
#pragma unroll
        for (int p = 0; p < WPL; ++p) {
            const int w = p * 32 + lane;
            X.w[p] = w < W ? (Cf.w[p] & rv[w] & ~(Pf.w[p] & below_mask(w, v))) : 0u;
        }
        const int n = warp_count<WPL>(X);
        const bool dead = !allk && sf + 2 - t > np2 + 1;
        bool taken = false;
        if (n == 0) {
            if ((allk || sf + 1 >= t) && lane == 0) sink.add(sf + 1, np2);
            taken = true;
        } else if (dead) {
            taken = true;
        } else if (n >= sink.push_min && n <= kGItemMax) {
            taken = push_large<WPL>(sink, X, list, sf + 1, np2, lane);
        }
        if (taken) {
            if (lane == 0) {
                ++visits;
                f[SC + 2] = uint32_t(v);
            }
            __syncwarp();
        }
        return;  // only the shallowest pending branch is considered
    }
}

// Walk the subtree of a fresh child set C (nonempty, not dead) at frame s0
// with pivot count npv (engine_pivot.py:117-233 from that node down).
template <int WPL>
__device__ void pivot_from(const uint32_t *__restrict__ rows, int RS, int W, int t, bool allk,
                           Set<WPL> C, const int s0, int npv, const Frames &F, int *list,
                           const SmallScratch &SS, const PivotLeafSink &sink,
                           const StealStack *q, ull &visits, ull &work) {
    const int lane = threadIdx.x & 31;
    if (pivot_try_small<WPL>(rows, RS, W, C, s0, npv, t, allk, list, SS, sink, lane, visits, work))
        return;
    if (sink.sp && sink.spend(0, lane)) {
        // this walk's budget is already spent: hand C itself over
        if (sink.spill_ids<WPL>(C, warp_count<WPL>(C), s0, npv, list, lane)) return;
        sink.no_spill(lane);
    }
    // frames are indexed relative to the walk's first frame s0: a spilled or
    // handed-over subtree starts deep in its task's tree (RMAT-22: depth
    // ~150) while a warp holds frames for one universe (<= its size + 2)
    auto fr = [&](int x) { return F.at(x - s0); };
    int pend = 0;           // branches not yet charged to the budget (uniform)
    bool spilling = false;  // budget spent: children leave as items
    const int PO = 32 * WPL, SC = 64 * WPL;  // P offset, scalars offset
    int s = s0;
    int piv = select_pivot<WPL>(rows, RS, C, list, lane, work, W);
    Set<WPL> P;
    {
        const Set<WPL> rp = load_row<WPL>(rows, RS, W, piv, lane);
#pragma unroll
        for (int p = 0; p < WPL; ++p) P.w[p] = C.w[p] & ~rp.w[p];
    }
    Set<WPL> R = P;
    // engine_pivot.py:152-153: a frame with deficit npv+1 only branches on its pivot
    if (!allk && s + 1 - t > npv) restrict_to(R, piv, lane);
    {
        uint32_t *f = fr(s);
        store_set<WPL>(f, C, lane);
        store_set<WPL>(f + PO, P, lane);
        if (lane == 0) {
            f[SC] = uint32_t(piv);
            f[SC + 1] = uint32_t(npv);
        }
    }
    for (;;) {
        const int v = next_bit<WPL>(R, lane);
        if (v < 0) {
            if (s == s0) break;
            --s;
            const uint32_t *f = fr(s);
            C = load_set<WPL>(f, lane);
            P = load_set<WPL>(f + PO, lane);
            piv = int(f[SC]);
            npv = int(f[SC + 1]);
            const int c = int(f[SC + 2]);
#pragma unroll
            for (int p = 0; p < WPL; ++p) R.w[p] = P.w[p] & above_mask(p * 32 + lane, c);
            if (!allk && s + 1 - t > npv) restrict_to(R, piv, lane);
            continue;
        }
        const int np2 = npv + (v == piv ? 1 : 0);
        if (!allk && s + 1 - t > np2) continue;
        if (lane == 0) {
            ++visits;
            work += 1;
        }
        if (sink.sp && !spilling && ++pend >= 16) {
            spilling = sink.spend(pend, lane);
            pend = 0;
        }
        Set<WPL> X;
        const uint32_t *rv = rows + v * RS;
#pragma unroll
        for (int p = 0; p < WPL; ++p) {
            const int w = p * 32 + lane;
            // engine_pivot.py:158-166: drop already-branched pivot-set bits below v
            X.w[p] = w < W ? (C.w[p] & rv[w] & ~(P.w[p] & below_mask(w, v))) : 0u;
        }
        if (any_set<WPL>(X)) {
            // a child whose every branch would be pruned adds neither visits nor leaves
            if (!allk && s + 2 - t > np2 + 1) continue;
            if (spilling) {
                // over budget: the child leaves as an item instead of being
                // walked (<= 32 members: the S-tier walk below spills it)
                const int nx = warp_count<WPL>(X);
                if (nx > 32) {
                    if (sink.spill_ids<WPL>(X, nx, s + 1, np2, list, lane)) continue;
                    sink.no_spill(lane);
                    spilling = false;
                }
            }
            {
                const int nx = warp_count<WPL>(X);
                if (WPL == 1 && sink.want_push(nx, allk ? 1 << 20 : t - s0, lane)) {
                    // donate the shallowest pending branch if there is one
                    // below this frame, else this child (CTA tier: this child)
                    if (sink.eager) {
                        if (push_large<WPL>(sink, X, list, s + 1, np2, lane)) continue;
                    } else if (s > s0) {
                        if (lane == 0) fr(s)[SC + 2] = uint32_t(v);  // cursor of the top frame
                        __syncwarp();
                        donate_bottom_L<WPL>(rows, RS, W, t, allk, F, s0, s, list, sink, lane,
                                             visits);
                    } else if (push_large<WPL>(sink, X, list, s + 1, np2, lane)) {
                        continue;
                    }
                }
                if (q && nx > 32 && steal_push<WPL>(*q, X, s + 1, np2, lane)) continue;
            }
            if (pivot_try_small<WPL>(rows, RS, W, X, s + 1, np2, t, allk, list, SS, sink, lane,
                                     visits, work))
                continue;
            if (lane == 0) fr(s)[SC + 2] = uint32_t(v);
            ++s;
            npv = np2;
            C = X;
            piv = select_pivot<WPL>(rows, RS, C, list, lane, work, W);
            const Set<WPL> rp = load_row<WPL>(rows, RS, W, piv, lane);
#pragma unroll
            for (int p = 0; p < WPL; ++p) P.w[p] = C.w[p] & ~rp.w[p];
            R = P;
            if (!allk && s + 1 - t > npv) restrict_to(R, piv, lane);
            uint32_t *f = fr(s);
            store_set<WPL>(f, C, lane);
            store_set<WPL>(f + PO, P, lane);
            if (lane == 0) {
                f[SC] = uint32_t(piv);
                f[SC + 1] = uint32_t(npv);
            }
        } else if (allk || s + 1 >= t) {
            if (lane == 0) sink.add(s + 1, np2);
        }
    }
}

// One root-level branch v0 of the task (frame 0 sets S0 / P0 in smem).
template <int WPL>
__device__ void pivot_subtree(const uint32_t *__restrict__ rows, int RS, int W, int t, bool allk,
                              int v0, int piv0, const uint32_t *S0, const uint32_t *P0,
                              const Frames &F, int *list, const SmallScratch &SS,
                              const PivotLeafSink &sink, ull &visits, ull &work,
                              const StealStack *q = nullptr, int s0 = 0, int npv0 = 0) {
    // (s0, npv0): depth and pivot count of the frame S0 (0, 0 for a task root;
    // a spilled item's node otherwise)
    const int lane = threadIdx.x & 31;
    const int np0 = npv0 + (v0 == piv0 ? 1 : 0);
    if (!allk && s0 + 1 - t > np0) return;  // engine_pivot.py:152-153
    if (lane == 0) {
        ++visits;
        work += 1;
    }
    Set<WPL> C;
    {
        const uint32_t *rv = rows + v0 * RS;
#pragma unroll
        for (int p = 0; p < WPL; ++p) {
            const int w = p * 32 + lane;
            C.w[p] = w < W ? (S0[w] & rv[w] & ~(P0[w] & below_mask(w, v0))) : 0u;
        }
    }
    if (!any_set<WPL>(C)) {
        if ((allk || s0 + 1 >= t) && lane == 0) sink.add(s0 + 1, np0);
        return;
    }
    if (!allk && s0 + 2 - t > np0 + 1) return;  // dead child
    pivot_from<WPL>(rows, RS, W, t, allk, C, s0 + 1, np0, F, list, SS, sink, q, visits, work);
}

// Idle loop of the work-sharing protocol: pop and walk stolen subtrees until
// every warp is idle and the stack is empty.
template <int WPL>
__device__ void pivot_steal_loop(const uint32_t *__restrict__ rows, int RS, int W, int t,
                                 bool allk, const Frames &F, int *list, const SmallScratch &SS,
                                 const PivotLeafSink &sink, const StealStack &q, ull &visits,
                                 ull &work) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        q.acquire();
        ++*(volatile int *)q.idle;
        q.release();
    }
    for (;;) {
        int slot = -1, done = 0;
        if (lane == 0) {
            // poll without the lock; lock only to pop or to confirm termination
            while (*(volatile int *)q.size == 0 && *(volatile int *)q.idle < q.nwarps)
                __nanosleep(64);
            q.acquire();
            const int sz = *(volatile int *)q.size;
            if (sz > 0) {
                slot = sz - 1;  // popped under the lock; data read below, lock held
                *(volatile int *)q.idle -= 1;
            } else {
                done = *(volatile int *)q.idle == q.nwarps;
                q.release();
            }
        }
        slot = __shfl_sync(FULL, slot, 0);
        done = __shfl_sync(FULL, done, 0);
        if (done) break;
        if (slot < 0) continue;
        const uint32_t *it = q.items + slot * q.iw;
        const Set<WPL> X = load_set<WPL>(it, lane);
        const int s = int(it[32 * WPL]);
        const int npv = int(it[32 * WPL + 1]);
        __syncwarp();
        if (lane == 0) {
            *(volatile int *)q.size = slot;
            q.release();
        }
        pivot_from<WPL>(rows, RS, W, t, allk, X, s, npv, F, list, SS, sink, &q, visits, work);
        if (lane == 0) {
            q.acquire();
            ++*(volatile int *)q.idle;
            q.release();
        }
    }
}

}  // namespace kct
