// kc_peel.cu -- K3 exact: the reference's sequential heap order
// (orientation.py:81-113: repeatedly remove the live vertex of minimum
// (residual degree, id)) computed in parallel, identical rank for rank.
//
// Why it decomposes (each step below is exact, not a heuristic):
//  1. Phases.  While some live vertex has residual degree <= k the heap pops
//     degree <= k, and removing degree-<=k vertices in any order ends at the
//     (k+1)-core.  So the heap removes the k-shell (core number k) entirely
//     before any vertex of a higher core: order = shells by core number.
//  2. Components.  During phase k only k-shell vertices lose degree, and only
//     through k-shell neighbours.  A connected component C of the graph
//     induced by the k-shell therefore evolves independently: its pops, in
//     their relative order, are those of the heap run on C alone, starting
//     from the degrees in the k-core.
//  3. Merge.  The heap interleaves the components of a phase by always taking
//     the smallest current head.  For such a min-head merge, an element is
//     output in order of E = the maximum key of its component's pops up to
//     and including it (ties only inside one component, kept in pop order):
//     if E_x < E_y, the element of y's component holding E_y cannot be
//     popped while x's component still has x or an earlier element waiting.
// So: core numbers (the bulk peel, K3), the shell-internal CSR, connected
// components (union-find), ONE short sequential heap run per component (a
// warp per component; only a handful of components exceed 32 vertices), and
// a stable sort by (core, E) of the vertices listed in (component, pop)
// order.  The rank equals the reference's array (tests/test_orientation.py
// :77-85), hence the DAG, hence every engine's visits.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "kc_internal.cuh"

namespace {

typedef unsigned long long ull;
constexpr unsigned FULL = 0xffffffffu;
constexpr int kT = 256;
constexpr uint32_t kDead = 0xffffffffu;

inline int grid_for(int64_t n, int sms) {
    int64_t b = (n + kT - 1) / kT;
    if (b > int64_t(sms) * 16) b = int64_t(sms) * 16;
    return int(b < 1 ? 1 : b);
}

// warp per vertex: degree in its own core (neighbours of core >= c) and the
// shell-internal flags of its arcs
__global__ void k_shell_degrees(const int64_t *__restrict__ row_ptr,
                                const int32_t *__restrict__ col, const int32_t *__restrict__ core,
                                int64_t n, int32_t *__restrict__ deg0,
                                uint8_t *__restrict__ flag) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t v = warp; v < n; v += nw) {
        const int32_t c = core[v];
        int cnt = 0;
        for (int64_t e = row_ptr[v] + lane; e < row_ptr[v + 1]; e += 32) {
            const int32_t cw = core[col[e]];
            cnt += cw >= c;
            flag[e] = cw == c;
        }
        cnt = __reduce_add_sync(FULL, unsigned(cnt));
        if (lane == 0) deg0[v] = cnt;
    }
}

__global__ void k_row_ptr32(const int32_t *__restrict__ src, int64_t cnt, int64_t n,
                            int64_t *__restrict__ row_ptr) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v <= n;
         v += int64_t(gridDim.x) * blockDim.x)
        row_ptr[v] = v == n ? cnt : kc_lower_bound_i32(src, cnt, int32_t(v));
}

__global__ void k_iota32(int32_t *__restrict__ a, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        a[i] = int32_t(i);
}

// union-find with parents always smaller than children: a root is the
// smallest id of its tree, so the final label is the component's minimum id
__device__ __forceinline__ int32_t uf_find(int32_t *par, int32_t x) {
    int32_t p = *(volatile int32_t *)(par + x);
    while (p != x) {
        const int32_t gp = *(volatile int32_t *)(par + p);
        if (gp != p) par[x] = gp;  // path halving: gp is an ancestor of x
        x = p;
        p = gp;
    }
    return x;
}

__global__ void k_uf_hook(const int32_t *__restrict__ isrc, const int32_t *__restrict__ icol,
                          int64_t m_int, int32_t *par) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m_int;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int32_t u = isrc[i], w = icol[i];
        if (u > w) continue;  // each edge once
        int32_t a = uf_find(par, u), b = uf_find(par, w);
        while (a != b) {
            if (a > b) {
                const int32_t t = a;
                a = b;
                b = t;
            }
            const int32_t old = atomicCAS(par + b, b, a);  // hook root b under a < b
            if (old == b) break;
            b = uf_find(par, old);
            a = uf_find(par, a);
        }
    }
}

__global__ void k_uf_keys(int32_t *par, int64_t n, int bits, uint64_t *__restrict__ keys) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x) {
        const int32_t r = uf_find(par, int32_t(v));
        keys[v] = (uint64_t(uint32_t(r)) << bits) | uint64_t(v);
    }
}

// sorted (label, v) keys -> cverts (vertices grouped by component, ascending
// id inside) and component-start flags
__global__ void k_groups(const uint64_t *__restrict__ keys, int64_t n, int bits,
                         int32_t *__restrict__ cverts, int32_t *__restrict__ sflag) {
    const uint64_t mask = (uint64_t(1) << bits) - 1;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        cverts[i] = int32_t(keys[i] & mask);
        sflag[i] = (i == 0 || (keys[i] >> bits) != (keys[i - 1] >> bits)) ? 1 : 0;
    }
}

// cid1 = inclusive scan of sflag (1-based component index of position i)
__global__ void k_starts(const int32_t *__restrict__ sflag, const int32_t *__restrict__ cid1,
                         int64_t n, int32_t *__restrict__ cstart) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        if (sflag[i]) cstart[cid1[i] - 1] = int32_t(i);
}

// loc[v] = index of v inside its component; gpos[v] = its position in cverts
__global__ void k_locals(const int32_t *__restrict__ cverts, const int32_t *__restrict__ cid1,
                         const int32_t *__restrict__ cstart, int64_t n, int32_t *__restrict__ loc,
                         int32_t *__restrict__ gpos) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int32_t v = cverts[i];
        loc[v] = int32_t(i) - cstart[cid1[i] - 1];
        gpos[v] = int32_t(i);
    }
}

__global__ void k_iloc(const int32_t *__restrict__ icol, int64_t m_int,
                       const int32_t *__restrict__ loc, int32_t *__restrict__ iloc) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m_int;
         i += int64_t(gridDim.x) * blockDim.x)
        iloc[i] = loc[icol[i]];
}

// Components of at most 32 vertices: one warp each, lane i = the i-th
// smallest id; the residual degrees and the internal adjacency (a 32-bit mask)
// live in registers, a pop is one __reduce_min_sync.
__global__ void k_comp_small(const int32_t *__restrict__ cverts, const int32_t *__restrict__ cstart,
                             int64_t n_comp, int64_t n, const int32_t *__restrict__ core,
                             const int32_t *__restrict__ deg0, const int64_t *__restrict__ irow,
                             const int32_t *__restrict__ iloc, int32_t *__restrict__ pos,
                             ull *__restrict__ ekey, int32_t *__restrict__ err) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t c = warp; c < n_comp; c += nw) {
        const int32_t b = cstart[c];
        const int32_t s = int32_t((c + 1 < n_comp ? cstart[c + 1] : n) - b);
        if (s > 32) continue;  // big components: k_comp_big
        const bool mine = lane < s;
        const int32_t v = mine ? cverts[b + lane] : 0;
        const int32_t k = core[cverts[b]];
        uint32_t deg = mine ? uint32_t(deg0[v]) : 0u, adj = 0;
        if (mine)
            for (int64_t e = irow[v]; e < irow[v + 1]; ++e) adj |= 1u << iloc[e];
        bool live = mine;
        ull emax = 0, my_e = 0;
        int my_pos = 0;
        const uint32_t cap = uint32_t(k) + 1;
        for (int step = 0; step < s; ++step) {
            const uint32_t key = live ? ((deg < cap ? deg : cap) << 5) | uint32_t(lane) : kDead;
            const uint32_t m = __reduce_min_sync(FULL, key);
            const int p = int(m & 31u);
            const uint32_t dp = m >> 5;
            if (dp > uint32_t(k) && lane == 0) atomicExch(err, 1);  // heap pops degree <= k
            const int32_t idp = __shfl_sync(FULL, v, p);
            const ull ek = (ull(dp) << 32) | ull(uint32_t(idp));
            emax = ek > emax ? ek : emax;
            if (lane == p) {
                live = false;
                my_pos = step;
                my_e = emax;
            }
            if (live && ((adj >> p) & 1u)) --deg;
        }
        if (mine) {
            pos[v] = my_pos;
            ekey[v] = my_e;
        }
    }
}

// internal-row bounds of every vertex, in component order (one dependent
// load per heap step instead of cverts -> irow)
__global__ void k_local_rows(const int32_t *__restrict__ cverts, const int64_t *__restrict__ irow,
                             int64_t n, int2 *__restrict__ lrow) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int32_t v = cverts[i];
        lrow[i] = make_int2(int32_t(irow[v]), int32_t(irow[v + 1]));
    }
}

// One big component per CTA (one warp): residual degrees dg[s] (16-bit in
// shared memory when the component's degrees fit, else 32-bit, in shared or
// global memory), the minimum key of every 32-vertex block (bmin) and of
// every 32-block super-block (smin), both in shared memory.  A decrement only
// lowers keys (atomicMin up the two levels); a pop recomputes its own block
// and super-block.  Key = (min(deg, k+1) << lbits) | local index (local order
// = id order).
template <typename DT, bool SMEM>
__global__ void __launch_bounds__(32)
    k_comp_big(const int32_t *__restrict__ big, const int32_t *__restrict__ cverts,
               const int32_t *__restrict__ cstart, int64_t n_comp, int64_t n,
               const int32_t *__restrict__ core, const int32_t *__restrict__ deg0,
               const int2 *__restrict__ lrow, const int32_t *__restrict__ iloc,
               int32_t *__restrict__ pos, ull *__restrict__ ekey, uint32_t *gscratch,
               int64_t gslot, int32_t *__restrict__ err) {
    extern __shared__ uint32_t sm[];
    constexpr DT kDeadT = DT(~DT(0));
    const int lane = threadIdx.x;
    const int64_t c = big[blockIdx.x];
    const int32_t b0 = cstart[c];
    const int32_t s = int32_t((c + 1 < n_comp ? cstart[c + 1] : n) - b0);
    const int nb = (s + 31) >> 5, ns = (nb + 31) >> 5;
    uint32_t *bmin = sm;
    uint32_t *smin = bmin + ((nb + 3) & ~3);
    DT *dg = SMEM ? reinterpret_cast<DT *>(smin + ((ns + 3) & ~3))
                  : reinterpret_cast<DT *>(gscratch + int64_t(blockIdx.x) * gslot);
    int lbits = 0;
    while ((1 << lbits) < s) ++lbits;
    const int32_t k = core[cverts[b0]];
    const uint32_t cap = uint32_t(k) + 1, lmask = (1u << lbits) - 1u;
    if (lane == 0 && (uint64_t(cap) << lbits) >= 0xffffffffull) atomicExch(err, 2);
    auto key_of = [&](int i) -> uint32_t {
        if (i >= s) return kDead;
        const DT d = dg[i];
        return d == kDeadT ? kDead : ((uint32_t(d) < cap ? uint32_t(d) : cap) << lbits) | uint32_t(i);
    };
    for (int i = lane; i < s; i += 32) dg[i] = DT(deg0[cverts[b0 + i]]);
    __syncwarp();
    for (int bb = 0; bb < nb; ++bb) {
        const uint32_t m = __reduce_min_sync(FULL, key_of(bb * 32 + lane));
        if (lane == 0) bmin[bb] = m;
    }
    __syncwarp();
    for (int sb = 0; sb < ns; ++sb) {
        const int j = sb * 32 + lane;
        const uint32_t m = __reduce_min_sync(FULL, j < nb ? bmin[j] : kDead);
        if (lane == 0) smin[sb] = m;
    }
    __syncwarp();
    ull emax = 0;
    for (int step = 0; step < s; ++step) {
        uint32_t m = kDead;
        for (int j = lane; j < ns; j += 32) m = min(m, smin[j]);
        m = __reduce_min_sync(FULL, m);
        const int p = int(m & lmask);
        const uint32_t dp = m >> lbits;
        const int32_t vp = cverts[b0 + p];  // only for the outputs below
        if (lane == 0) {
            if (dp > uint32_t(k)) atomicExch(err, 1);
            const ull ek = (ull(dp) << 32) | ull(uint32_t(vp));
            emax = ek > emax ? ek : emax;
            pos[vp] = step;
            ekey[vp] = emax;
            dg[p] = kDeadT;
        }
        __syncwarp();
        const int2 rb = lrow[b0 + p];
        for (int e = rb.x + lane; e < rb.y; e += 32) {
            const int j = iloc[e];
            const DT d = dg[j];
            if (d == kDeadT) continue;
            dg[j] = DT(d - 1);  // each neighbour appears once in p's row
            const uint32_t d1 = uint32_t(d) - 1u;
            const uint32_t nk = ((d1 < cap ? d1 : cap) << lbits) | uint32_t(j);
            atomicMin(bmin + (j >> 5), nk);
            atomicMin(smin + (j >> 10), nk);
        }
        __syncwarp();
        const int pb = p >> 5;
        const uint32_t kb = __reduce_min_sync(FULL, key_of(pb * 32 + lane));
        if (lane == 0) bmin[pb] = kb;
        __syncwarp();
        const int ps = pb >> 5, j = ps * 32 + lane;
        const uint32_t ks = __reduce_min_sync(FULL, j < nb ? bmin[j] : kDead);
        if (lane == 0) smin[ps] = ks;
        __syncwarp();
    }
}

// max deg0 over vertices of components with more than 32 vertices
__global__ void k_max_deg_big(const int32_t *__restrict__ cverts, const int32_t *__restrict__ cid1,
                              const int32_t *__restrict__ cstart, int64_t n_comp, int64_t n,
                              const int32_t *__restrict__ deg0, int *__restrict__ out) {
    int local = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t c = cid1[i] - 1;
        const int64_t sz = (c + 1 < n_comp ? cstart[c + 1] : n) - cstart[c];
        if (sz > 32) local = max(local, deg0[cverts[i]]);
    }
    local = int(__reduce_max_sync(FULL, unsigned(local)));
    if ((threadIdx.x & 31) == 0 && local) atomicMax(out, local);
}

// slot of v in (component, pop) order; sort key (core, E)
__global__ void k_merge_keys(const int32_t *__restrict__ core, const int32_t *__restrict__ gpos,
                             const int32_t *__restrict__ loc, const int32_t *__restrict__ pos,
                             const ull *__restrict__ ekey, int64_t n, int dbits, int ibits,
                             uint64_t *__restrict__ keys, int32_t *__restrict__ vals) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x) {
        const int64_t slot = int64_t(gpos[v]) - loc[v] + pos[v];
        const ull e = ekey[v];
        keys[slot] = (uint64_t(uint32_t(core[v])) << (dbits + ibits)) | ((e >> 32) << ibits) |
                     (e & 0xffffffffull);
        vals[slot] = int32_t(v);
    }
}

__global__ void k_rank_from_order32(const int32_t *__restrict__ order, int64_t n,
                                    int32_t *__restrict__ rank) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        rank[order[i]] = int32_t(i);
}

struct Buf {
    void *p = nullptr;
    cudaStream_t s;
    Buf(size_t bytes, cudaStream_t st) : s(st) { p = kc_alloc<uint8_t>(bytes, st); }
    ~Buf() { kc_free(p, s); }
    template <typename T>
    T *as() const {
        return reinterpret_cast<T *>(p);
    }
};

}  // namespace

void kc_exact_order_from_cores(kc_graph *g, const int32_t *core, int64_t degeneracy,
                               int32_t *rank_out) {
    const int64_t n = g->n, two_m = 2 * g->m;
    cudaStream_t st = g->stream;
    const int sms = g->num_sms;
    if (n == 0) return;
    // 1. degree in the own core + shell-internal arcs
    Buf deg0(4 * n, st), flag(std::max<int64_t>(two_m, 1), st), err(8, st);
    KC_CUDA(cudaMemsetAsync(err.p, 0, 8, st));
    k_shell_degrees<<<sms * 16, kT, 0, st>>>(g->row_ptr, g->col, core, n, deg0.as<int32_t>(),
                                             flag.as<uint8_t>());
    KC_CUDA(cudaGetLastError());
    // 2. shell-internal CSR (rows keep compact-id order)
    Buf isrc(4 * std::max<int64_t>(two_m, 1), st), icol(4 * std::max<int64_t>(two_m, 1), st),
        cnt(8, st), irow(8 * (n + 1), st);
    int64_t m_int = 0;
    if (two_m > 0) {
        size_t bytes = 0;
        KC_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, g->col, flag.as<uint8_t>(),
                                           icol.as<int32_t>(), cnt.as<int32_t>(), int(two_m), st));
        void *tmp = kc_tmp(g, bytes);
        KC_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, g->col, flag.as<uint8_t>(),
                                           icol.as<int32_t>(), cnt.as<int32_t>(), int(two_m), st));
        KC_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, g->coo_src, flag.as<uint8_t>(),
                                           isrc.as<int32_t>(), cnt.as<int32_t>() + 1, int(two_m),
                                           st));
        int32_t h = 0;
        KC_CUDA(cudaMemcpyAsync(&h, cnt.p, 4, cudaMemcpyDeviceToHost, st));
        KC_CUDA(cudaStreamSynchronize(st));
        m_int = h;
    }
    k_row_ptr32<<<grid_for(n + 1, sms), kT, 0, st>>>(isrc.as<int32_t>(), m_int, n,
                                                     irow.as<int64_t>());
    // 3. connected components of the shell-internal graph
    Buf par(4 * n, st);
    k_iota32<<<grid_for(n, sms), kT, 0, st>>>(par.as<int32_t>(), n);
    if (m_int > 0)
        k_uf_hook<<<grid_for(m_int, sms), kT, 0, st>>>(isrc.as<int32_t>(), icol.as<int32_t>(),
                                                       m_int, par.as<int32_t>());
    const int bits = kc_bits_for(n - 1 > 0 ? n - 1 : 1);
    Buf keys(8 * n, st), keys2(8 * n, st);
    k_uf_keys<<<grid_for(n, sms), kT, 0, st>>>(par.as<int32_t>(), n, bits, keys.as<uint64_t>());
    KC_CUDA(cudaGetLastError());
    {
        size_t bytes = 0;
        KC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys.as<uint64_t>(),
                                               keys2.as<uint64_t>(), int(n), 0, 2 * bits, st));
        void *tmp = kc_tmp(g, bytes);
        KC_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, keys.as<uint64_t>(),
                                               keys2.as<uint64_t>(), int(n), 0, 2 * bits, st));
    }
    // 4. group by component
    Buf cverts(4 * n, st), sflag(4 * n, st), cid1(4 * n, st), loc(4 * n, st), gpos(4 * n, st);
    k_groups<<<grid_for(n, sms), kT, 0, st>>>(keys2.as<uint64_t>(), n, bits,
                                              cverts.as<int32_t>(), sflag.as<int32_t>());
    {
        size_t bytes = 0;
        KC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, sflag.as<int32_t>(),
                                              cid1.as<int32_t>(), int(n), st));
        void *tmp = kc_tmp(g, bytes);
        KC_CUDA(cub::DeviceScan::InclusiveSum(tmp, bytes, sflag.as<int32_t>(), cid1.as<int32_t>(),
                                              int(n), st));
    }
    int32_t n_comp32 = 0;
    KC_CUDA(cudaMemcpyAsync(&n_comp32, cid1.as<int32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
    KC_CUDA(cudaStreamSynchronize(st));
    const int64_t n_comp = n_comp32;
    Buf cstart(4 * (n_comp + 1), st);
    k_starts<<<grid_for(n, sms), kT, 0, st>>>(sflag.as<int32_t>(), cid1.as<int32_t>(), n,
                                              cstart.as<int32_t>());
    k_locals<<<grid_for(n, sms), kT, 0, st>>>(cverts.as<int32_t>(), cid1.as<int32_t>(),
                                              cstart.as<int32_t>(), n, loc.as<int32_t>(),
                                              gpos.as<int32_t>());
    Buf iloc(4 * std::max<int64_t>(m_int, 1), st);
    if (m_int > 0)
        k_iloc<<<grid_for(m_int, sms), kT, 0, st>>>(icol.as<int32_t>(), m_int, loc.as<int32_t>(),
                                                    iloc.as<int32_t>());
    KC_CUDA(cudaGetLastError());
    // 5. the heap run of every component
    std::vector<int32_t> hstart(n_comp + 1);
    KC_CUDA(cudaMemcpyAsync(hstart.data(), cstart.p, 4 * n_comp, cudaMemcpyDeviceToHost, st));
    KC_CUDA(cudaStreamSynchronize(st));
    hstart[n_comp] = int32_t(n);
    std::vector<int32_t> hbig;
    int64_t max_big = 0;
    for (int64_t c = 0; c < n_comp; ++c) {
        const int64_t s = hstart[c + 1] - hstart[c];
        if (s > 32) {
            hbig.push_back(int32_t(c));
            max_big = std::max(max_big, s);
        }
    }
    // largest degree in the own core over the big components (16-bit test)
    int64_t max_deg0_big = 0;
    if (!hbig.empty()) {
        Buf dmax(8, st);
        KC_CUDA(cudaMemsetAsync(dmax.p, 0, 8, st));
        k_max_deg_big<<<grid_for(n, sms), kT, 0, st>>>(cverts.as<int32_t>(), cid1.as<int32_t>(),
                                                       cstart.as<int32_t>(), n_comp, n,
                                                       deg0.as<int32_t>(), dmax.as<int>());
        int hm = 0;
        KC_CUDA(cudaMemcpyAsync(&hm, dmax.p, 4, cudaMemcpyDeviceToHost, st));
        KC_CUDA(cudaStreamSynchronize(st));
        max_deg0_big = hm;
    }
    // largest components first (they are the critical path)
    std::sort(hbig.begin(), hbig.end(), [&](int32_t a, int32_t b) {
        return hstart[a + 1] - hstart[a] > hstart[b + 1] - hstart[b];
    });
    Buf pos(4 * n, st), ekey(8 * n, st);
    {
        const int64_t blocks = std::min<int64_t>((n_comp + 7) / 8, int64_t(sms) * 32);
        k_comp_small<<<int(std::max<int64_t>(blocks, 1)), kT, 0, st>>>(
            cverts.as<int32_t>(), cstart.as<int32_t>(), n_comp, n, core, deg0.as<int32_t>(),
            irow.as<int64_t>(), iloc.as<int32_t>(), pos.as<int32_t>(), ekey.as<ull>(),
            err.as<int32_t>());
        KC_CUDA(cudaGetLastError());
    }
    if (!hbig.empty()) {
        const int64_t nbig = int64_t(hbig.size());
        Buf dbig(4 * nbig, st), lrow(8 * n, st);
        KC_CUDA(cudaMemcpyAsync(dbig.p, hbig.data(), 4 * nbig, cudaMemcpyHostToDevice, st));
        KC_REQUIRE(m_int < (int64_t(1) << 31), KC_EINVAL, "too many shell-internal arcs");
        k_local_rows<<<grid_for(n, sms), kT, 0, st>>>(cverts.as<int32_t>(), irow.as<int64_t>(), n,
                                                     lrow.as<int2>());
        const int64_t nb = (max_big + 31) / 32, ns = (nb + 31) / 32;
        const int64_t lvl_words = ((nb + 3) & ~int64_t(3)) + ((ns + 3) & ~int64_t(3));
        constexpr int64_t kSmemBytes = 200 * 1024;
        // 16-bit residual degrees when every degree of the big components fits
        const bool narrow = max_deg0_big < 0xffff;
        const int64_t dg_bytes = (narrow ? 2 : 4) * ((max_big + 3) & ~int64_t(3));
        const int64_t smem_all = 4 * lvl_words + dg_bytes;
        auto run = [&](auto kern, size_t smem, uint32_t *gsc, int64_t gslot) {
            KC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem)));
            kern<<<int(nbig), 32, smem, st>>>(
                dbig.as<int32_t>(), cverts.as<int32_t>(), cstart.as<int32_t>(), n_comp, n, core,
                deg0.as<int32_t>(), lrow.as<int2>(), iloc.as<int32_t>(), pos.as<int32_t>(),
                ekey.as<ull>(), gsc, gslot, err.as<int32_t>());
        };
        if (smem_all <= kSmemBytes) {
            if (narrow) run(k_comp_big<uint16_t, true>, size_t(smem_all), nullptr, 0);
            else run(k_comp_big<uint32_t, true>, size_t(smem_all), nullptr, 0);
        } else {
            const int64_t gslot = (max_big + 3) & ~int64_t(3);
            Buf gs(4 * size_t(gslot) * size_t(nbig), st);
            run(k_comp_big<uint32_t, false>, size_t(4 * lvl_words), gs.as<uint32_t>(), gslot);
        }
        KC_CUDA(cudaGetLastError());
    }
    // 6. merge: stable sort of the (component, pop)-ordered vertices by (core, E)
    const int dbits = kc_bits_for(degeneracy > 0 ? degeneracy : 1);
    const int ibits = kc_bits_for(n - 1 > 0 ? n - 1 : 1);
    KC_REQUIRE(2 * dbits + ibits <= 64, KC_EINVAL, "degeneracy too large for the exact order key");
    Buf vals(4 * n, st), order(4 * n, st);
    k_merge_keys<<<grid_for(n, sms), kT, 0, st>>>(core, gpos.as<int32_t>(), loc.as<int32_t>(),
                                                  pos.as<int32_t>(), ekey.as<ull>(), n, dbits,
                                                  ibits, keys.as<uint64_t>(), vals.as<int32_t>());
    {
        size_t bytes = 0;
        KC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.as<uint64_t>(),
                                                keys2.as<uint64_t>(), vals.as<int32_t>(),
                                                order.as<int32_t>(), int(n), 0,
                                                2 * dbits + ibits, st));
        void *tmp = kc_tmp(g, bytes);
        KC_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, keys.as<uint64_t>(),
                                                keys2.as<uint64_t>(), vals.as<int32_t>(),
                                                order.as<int32_t>(), int(n), 0,
                                                2 * dbits + ibits, st));
    }
    k_rank_from_order32<<<grid_for(n, sms), kT, 0, st>>>(order.as<int32_t>(), n, rank_out);
    KC_CUDA(cudaGetLastError());
    int32_t herr[2] = {0, 0};
    KC_CUDA(cudaMemcpyAsync(herr, err.p, 8, cudaMemcpyDeviceToHost, st));
    KC_CUDA(cudaStreamSynchronize(st));
    KC_REQUIRE(herr[0] == 0, KC_ECUDA,
               herr[0] == 2 ? "exact peel: component key overflow"
                            : "exact peel: internal invariant violated (pop above the core)");
}
