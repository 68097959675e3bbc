// kc_graph.cu -- K1 csr_build, K2 rank_degree + orient_filter, K3 kcore_peel.
//
// K1 restates graph.py:162-200 (from_edges): id compaction ascending by
//    original id, symmetrize, (src,dst) sort, row_ptr.  Device radix sorts over
//    packed u64 keys; row_ptr by per-vertex lower_bound over the sorted sources.
// K2 restates orientation.py:124-128 (degree rank: sort by (degree, id)) and
//    orientation.py:139-153 (keep e iff rank[src] < rank[dst], stable
//    compaction so segments keep compact-id order; row pointers rebuilt).
// K3 is the paper's bulk-synchronous GPU k-core peel (PAPER.md:316-321,
//    accepted by SPEC.md:129): rounds remove every live vertex of residual
//    degree <= level at once; rank = (round, id).  Its order differs from the
//    sequential heap of orientation.py:81-113, but it is a valid degeneracy
//    order: max out-degree == degeneracy (checked by the parity tests).
//
// All kernels are memory-bound integer passes: grid-stride loops, coalesced
// int32/int64 streams, no shared-memory staging needed.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "kc_internal.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n, int sms) {
    int64_t b = (n + kThreads - 1) / kThreads;
    int64_t cap = int64_t(sms) * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return int(b);
}

struct EventTimer {
    cudaEvent_t a, b;
    cudaStream_t s;
    explicit EventTimer(cudaStream_t st) : s(st) {
        KC_CUDA(cudaEventCreate(&a));
        KC_CUDA(cudaEventCreate(&b));
        KC_CUDA(cudaEventRecord(a, s));
    }
    double stop() {
        KC_CUDA(cudaEventRecord(b, s));
        KC_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        KC_CUDA(cudaEventElapsedTime(&ms, a, b));
        return ms;
    }
    ~EventTimer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
};

// ---- K1 ------------------------------------------------------------------
// map original ids of every pair to compact ids, emit both directions as
// packed keys (src << bits | dst)
__global__ void k_pack_pairs(const int64_t *__restrict__ pairs, int64_t m,
                             const int64_t *__restrict__ ids, int64_t n, int bits,
                             uint64_t *__restrict__ keys) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
         e += int64_t(gridDim.x) * blockDim.x) {
        uint64_t cu = (uint64_t)kc_lower_bound_i64(ids, n, pairs[2 * e]);
        uint64_t cv = (uint64_t)kc_lower_bound_i64(ids, n, pairs[2 * e + 1]);
        keys[e] = (cu << bits) | cv;
        keys[m + e] = (cv << bits) | cu;
    }
}

__global__ void k_unpack_keys(const uint64_t *__restrict__ keys, int64_t cnt, int bits,
                              int32_t *__restrict__ col, int32_t *__restrict__ src) {
    const uint64_t mask = (uint64_t(1) << bits) - 1;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < cnt;
         i += int64_t(gridDim.x) * blockDim.x) {
        uint64_t k = keys[i];
        col[i] = int32_t(k & mask);
        src[i] = int32_t(k >> bits);
    }
}

// row_ptr[v] = first slot whose source >= v (sources sorted ascending)
__global__ void k_row_ptr(const int32_t *__restrict__ src, int64_t cnt, int64_t n,
                          int64_t *__restrict__ row_ptr) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v <= n;
         v += int64_t(gridDim.x) * blockDim.x)
        row_ptr[v] = v == n ? cnt : kc_lower_bound_i32(src, cnt, int32_t(v));
}

__global__ void k_coo_from_rowptr(const int64_t *__restrict__ row_ptr, int64_t n,
                                  int32_t *__restrict__ src) {
    // one warp per vertex writes its source id over its segment
    int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t v = warp; v < n; v += nwarps)
        for (int64_t e = row_ptr[v] + lane; e < row_ptr[v + 1]; e += 32) src[e] = int32_t(v);
}

__global__ void k_degree_stats(const int64_t *__restrict__ row_ptr, int64_t n,
                               unsigned long long *__restrict__ out_max) {
    unsigned long long local = 0;
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x) {
        unsigned long long d = (unsigned long long)(row_ptr[v + 1] - row_ptr[v]);
        local = d > local ? d : local;
    }
    for (int o = 16; o; o >>= 1) {
        unsigned long long x = __shfl_xor_sync(0xffffffffu, local, o);
        local = x > local ? x : local;
    }
    if ((threadIdx.x & 31) == 0 && local) atomicMax(out_max, local);
}

// ---- K2 ------------------------------------------------------------------
__global__ void k_degree_keys(const int64_t *__restrict__ row_ptr, int64_t n, int bits,
                              uint64_t *__restrict__ keys) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x)
        keys[v] = (uint64_t(row_ptr[v + 1] - row_ptr[v]) << bits) | uint64_t(v);
}

__global__ void k_rank_from_sorted(const uint64_t *__restrict__ keys, int64_t n, int bits,
                                   int32_t *__restrict__ rank) {
    const uint64_t mask = (uint64_t(1) << bits) - 1;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        rank[keys[i] & mask] = int32_t(i);
}

// orientation.py:144 keep = rank[src] < rank[dst]; packed (src<<32|dst)
// compaction keeps the undirected CSR order, i.e. compact-id order per segment
__global__ void k_orient_flags(const int32_t *__restrict__ col, const int32_t *__restrict__ src,
                               const int32_t *__restrict__ rank, int64_t cnt,
                               uint8_t *__restrict__ flags) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < cnt;
         e += int64_t(gridDim.x) * blockDim.x)
        flags[e] = rank[src[e]] < rank[col[e]] ? 1 : 0;
}

// ---- K3 ------------------------------------------------------------------
// K3 as ONE persistent cooperative kernel: the whole bulk-synchronous peel
// runs on the device with grid-wide barriers (no host round trip per round).
// order[] receives vertices in removal order; round r's frontier is the slice
// [head, end) of it, and relax appends the next round's frontier at `tail`.
//
// Barrier discipline: the kernel is a sequence of steps separated by
// grid.sync().  Step p appends through counter cnt[p%3] and reports a minimum
// through mn[p%3]; every thread reads both right after the barrier ending
// step p, and slot p%3 is only re-zeroed at the start of step p+2 (after the
// barrier ending step p+1, which no thread passes before finishing its
// reads).  All control values are therefore identical in every thread.
// ctl: [0..2] cnt, [3..5] mn, [6] degeneracy, [7] rounds.
__global__ void k_peel_coop(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                            int64_t n, int32_t *__restrict__ deg, int32_t *__restrict__ round_of,
                            int32_t *__restrict__ order, int32_t *ctl,
                            int32_t *__restrict__ core_of) {
    cg::grid_group grid = cg::this_grid();
    const int64_t gtid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int64_t gsz = int64_t(gridDim.x) * blockDim.x;
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = gtid >> 5, nwarps = gsz >> 5;
    const int32_t BIG = 0x7fffffff;
    volatile int32_t *vctl = ctl;
    int32_t *cnt = ctl, *mn = ctl + 3;
    for (int64_t v = gtid; v < n; v += gsz) {
        deg[v] = int32_t(row_ptr[v + 1] - row_ptr[v]);
        round_of[v] = -1;
    }
    if (gtid == 0)
        for (int i = 0; i < 3; ++i) {
            cnt[i] = 0;
            mn[i] = BIG;
        }
    grid.sync();
    int p = 0;  // step index (uniform)
    auto begin_step = [&]() {
        if (gtid == 0) {
            cnt[(p + 1) % 3] = 0;
            mn[(p + 1) % 3] = BIG;
        }
    };
    int64_t head = 0, tail = 0;
    int32_t level = 0, round = 0, degen = 0;
    while (head < n) {
        // scan step: live vertices of residual degree <= level start a level
        begin_step();
        for (int64_t base = gtid - lane; base < n; base += gsz) {
            const int64_t v = base + lane;
            const bool live = v < n && round_of[v] < 0;
            const int32_t d = live ? deg[v] : BIG;
            const bool take = live && d <= level;
            const unsigned mask = __ballot_sync(0xffffffffu, take);
            int off = 0;
            if (lane == 0 && mask) off = atomicAdd(&cnt[p % 3], __popc(mask));
            off = __shfl_sync(0xffffffffu, off, 0);
            if (take) order[tail + off + __popc(mask & ((1u << lane) - 1))] = int32_t(v);
            int32_t dm = (live && !take) ? d : BIG;
            for (int o = 16; o; o >>= 1) dm = min(dm, __shfl_xor_sync(0xffffffffu, dm, o));
            if (lane == 0 && dm != BIG) atomicMin(&mn[p % 3], dm);
        }
        grid.sync();
        const int32_t added = vctl[p % 3];
        const int32_t mnv = vctl[3 + p % 3];
        ++p;
        if (added == 0) {
            level = mnv;  // no live vertex at this level: jump to the next one
            continue;
        }
        // lower bound of the next level: min degree of the live vertices this
        // scan left, lowered by every decrement of the rounds below; if it
        // undershoots (its vertex got peeled), the next scan finds nothing and
        // falls back to the exact minimum -- rounds and ranks are unchanged
        int32_t next_level = mnv;
        int64_t end = tail + added;
        tail = end;
        degen = level > degen ? level : degen;
        while (end > head) {
            // mark + relax step: warp per frontier vertex marks it removed and
            // decrements its not-yet-removed neighbours; one that crosses
            // level+1 -> level joins the next round's frontier.  Decrementing
            // a vertex of the current frontier (not marked yet) is harmless:
            // its degree is <= level, so it can never cross level+1 -> level.
            begin_step();
            for (int64_t i = head + gwarp; i < end; i += nwarps) {
                const int32_t v = order[i];
                if (lane == 0) {
                    round_of[v] = round;
                    if (core_of) core_of[v] = level;  // core number = level of removal
                }
                for (int64_t e = row_ptr[v] + lane; e < row_ptr[v + 1]; e += 32) {
                    const int32_t w = col[e];
                    if (round_of[w] >= 0) continue;
                    const int32_t old = atomicSub(&deg[w], 1);
                    if (old == level + 1) order[tail + atomicAdd(&cnt[p % 3], 1)] = w;
                    else if (old - 1 > level) atomicMin(&mn[p % 3], old - 1);
                }
            }
            grid.sync();
            const int32_t nxt = vctl[p % 3];
            const int32_t rmin = vctl[3 + p % 3];
            next_level = rmin < next_level ? rmin : next_level;
            ++p;
            head = end;
            end = tail + nxt;
            tail = end;
            ++round;
        }
        level = next_level;  // skip the scan that would only find this minimum
    }
    if (gtid == 0) {
        ctl[6] = degen;
        ctl[7] = round;
    }
}

__global__ void k_peel_keys(const int32_t *__restrict__ round_of, int64_t n, int bits,
                            uint64_t *__restrict__ keys) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x)
        keys[v] = (uint64_t(uint32_t(round_of[v])) << bits) | uint64_t(v);
}

__global__ void k_out_degree_max(const int64_t *__restrict__ orow, int64_t n,
                                 unsigned long long *__restrict__ out) {
    unsigned long long local = 0;
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x) {
        unsigned long long d = (unsigned long long)(orow[v + 1] - orow[v]);
        local = d > local ? d : local;
    }
    for (int o = 16; o; o >>= 1) {
        unsigned long long x = __shfl_xor_sync(0xffffffffu, local, o);
        local = x > local ? x : local;
    }
    if ((threadIdx.x & 31) == 0 && local) atomicMax(out, local);
}

// task list helpers ----------------------------------------------------------
// vertex tasks: make_tasks order = ascending vertex id among out-degree > 0
// (scheduler.py:91-92).  Index i of that order is a shard coordinate.
__global__ void k_vertex_task_flags(const int64_t *__restrict__ orow, int64_t n,
                                    int32_t *__restrict__ flag) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x)
        flag[v] = orow[v + 1] - orow[v] > 0 ? 1 : 0;
}

}  // namespace

// ---------------------------------------------------------------------------
void *kc_tmp(kc_graph *g, size_t bytes) {
    if (bytes > g->tmp_bytes) {
        if (g->tmp) kc_free(g->tmp, g->stream);
        g->tmp = nullptr;
        g->tmp_bytes = 0;
        size_t want = bytes + bytes / 4 + 1024;
        g->tmp = kc_alloc<uint8_t>(want, g->stream);
        g->tmp_bytes = want;
    }
    return g->tmp;
}

static void sort_u64(kc_graph *g, uint64_t *keys_in, uint64_t *keys_out, int64_t cnt, int end_bit) {
    if (cnt <= 1) {
        if (cnt == 1)
            KC_CUDA(cudaMemcpyAsync(keys_out, keys_in, 8, cudaMemcpyDeviceToDevice, g->stream));
        return;
    }
    KC_REQUIRE(cnt < (int64_t(1) << 31), KC_EINVAL, "graph too large for 32-bit sort offsets");
    size_t bytes = 0;
    KC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys_in, keys_out, int(cnt), 0, end_bit,
                                           g->stream));
    void *tmp = kc_tmp(g, bytes);
    KC_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, keys_in, keys_out, int(cnt), 0, end_bit,
                                           g->stream));
}

static void finish_csr_stats(kc_graph *g) {
    unsigned long long *d_max = kc_alloc<unsigned long long>(1, g->stream);
    KC_CUDA(cudaMemsetAsync(d_max, 0, 8, g->stream));
    if (g->n)
        k_degree_stats<<<grid_for(g->n, g->num_sms), kThreads, 0, g->stream>>>(g->row_ptr, g->n,
                                                                              d_max);
    unsigned long long h = 0;
    KC_CUDA(cudaMemcpyAsync(&h, d_max, 8, cudaMemcpyDeviceToHost, g->stream));
    KC_CUDA(cudaStreamSynchronize(g->stream));
    kc_free(d_max, g->stream);
    g->d_max_und = int64_t(h);
}

void kc_build_from_edges(kc_graph *g, const int64_t *pairs, int64_t m, const int64_t *extra,
                         int64_t n_extra) {
    KC_REQUIRE(m >= 0 && n_extra >= 0, KC_EINVAL, "negative sizes");
    EventTimer timer(g->stream);
    int64_t tot = 2 * m + n_extra;
    // ids = union1d(pairs.ravel(), extra)          graph.py:177-181
    int64_t *d_all = kc_alloc<int64_t>(tot, g->stream);
    int64_t *d_sorted = kc_alloc<int64_t>(tot, g->stream);
    if (m) KC_CUDA(cudaMemcpyAsync(d_all, pairs, 16 * m, cudaMemcpyDefault, g->stream));
    if (n_extra)
        KC_CUDA(cudaMemcpyAsync(d_all + 2 * m, extra, 8 * n_extra, cudaMemcpyDefault,
                                g->stream));
    int64_t n = 0;
    if (tot > 0) {
        KC_REQUIRE(tot < (int64_t(1) << 31), KC_EINVAL, "edge list too large");
        size_t bytes = 0;
        KC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, d_all, d_sorted, int(tot), 0, 64,
                                               g->stream));
        void *tmp = kc_tmp(g, bytes);
        KC_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, d_all, d_sorted, int(tot), 0, 64,
                                               g->stream));
        int32_t *d_n = kc_alloc<int32_t>(1, g->stream);
        bytes = 0;
        KC_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, d_sorted, d_all, d_n, int(tot),
                                          g->stream));
        tmp = kc_tmp(g, bytes);
        KC_CUDA(cub::DeviceSelect::Unique(tmp, bytes, d_sorted, d_all, d_n, int(tot), g->stream));
        int32_t hn = 0;
        KC_CUDA(cudaMemcpyAsync(&hn, d_n, 4, cudaMemcpyDeviceToHost, g->stream));
        KC_CUDA(cudaStreamSynchronize(g->stream));
        kc_free(d_n, g->stream);
        n = hn;
    }
    kc_free(d_sorted, g->stream);
    g->n = n;
    g->m = n ? m : 0;
    g->orig_ids = kc_alloc<int64_t>(n, g->stream);
    if (n)
        KC_CUDA(cudaMemcpyAsync(g->orig_ids, d_all, 8 * n, cudaMemcpyDeviceToDevice, g->stream));
    g->row_ptr = kc_alloc<int64_t>(n + 1, g->stream);
    g->col = kc_alloc<int32_t>(2 * g->m, g->stream);
    g->coo_src = kc_alloc<int32_t>(2 * g->m, g->stream);
    if (n == 0) {
        KC_CUDA(cudaMemsetAsync(g->row_ptr, 0, 8, g->stream));
    } else if (g->m == 0) {
        KC_CUDA(cudaMemsetAsync(g->row_ptr, 0, 8 * (n + 1), g->stream));
    } else {
        // raw pairs again (d_all now holds the ids); reuse a fresh buffer
        int64_t *d_pairs = kc_alloc<int64_t>(2 * m, g->stream);
        KC_CUDA(cudaMemcpyAsync(d_pairs, pairs, 16 * m, cudaMemcpyDefault, g->stream));
        int bits = kc_bits_for(n - 1 > 0 ? n - 1 : 1);
        KC_REQUIRE(2 * bits <= 64 && n < (int64_t(1) << 31), KC_EINVAL, "too many vertices");
        uint64_t *keys = kc_alloc<uint64_t>(2 * m, g->stream);
        uint64_t *keys2 = kc_alloc<uint64_t>(2 * m, g->stream);
        k_pack_pairs<<<grid_for(m, g->num_sms), kThreads, 0, g->stream>>>(d_pairs, m, g->orig_ids,
                                                                           n, bits, keys);
        KC_CUDA(cudaGetLastError());
        // lexsort((dst, src))                     graph.py:195
        sort_u64(g, keys, keys2, 2 * m, 2 * bits);
        k_unpack_keys<<<grid_for(2 * m, g->num_sms), kThreads, 0, g->stream>>>(
            keys2, 2 * m, bits, g->col, g->coo_src);
        // bincount + cumsum                        graph.py:198-199
        k_row_ptr<<<grid_for(n + 1, g->num_sms), kThreads, 0, g->stream>>>(g->coo_src, 2 * m, n,
                                                                            g->row_ptr);
        KC_CUDA(cudaGetLastError());
        KC_CUDA(cudaStreamSynchronize(g->stream));
        kc_free(keys, g->stream);
        kc_free(keys2, g->stream);
        kc_free(d_pairs, g->stream);
    }
    kc_free(d_all, g->stream);
    g->build_ms = timer.stop();
    finish_csr_stats(g);
}

void kc_build_from_csr(kc_graph *g, int64_t n, int64_t m, const int64_t *row_ptr,
                       const int32_t *col, const int64_t *orig_ids) {
    KC_REQUIRE(n >= 0 && m >= 0, KC_EINVAL, "negative sizes");
    EventTimer timer(g->stream);
    g->n = n;
    g->m = m;
    g->row_ptr = kc_alloc<int64_t>(n + 1, g->stream);
    g->col = kc_alloc<int32_t>(2 * m, g->stream);
    g->coo_src = kc_alloc<int32_t>(2 * m, g->stream);
    g->orig_ids = kc_alloc<int64_t>(n, g->stream);
    KC_CUDA(cudaMemcpyAsync(g->row_ptr, row_ptr, 8 * (n + 1), cudaMemcpyHostToDevice, g->stream));
    if (m) KC_CUDA(cudaMemcpyAsync(g->col, col, 8 * m, cudaMemcpyHostToDevice, g->stream));
    if (n && orig_ids)
        KC_CUDA(cudaMemcpyAsync(g->orig_ids, orig_ids, 8 * n, cudaMemcpyHostToDevice, g->stream));
    if (n && m)
        k_coo_from_rowptr<<<grid_for(32 * n, g->num_sms), kThreads, 0, g->stream>>>(g->row_ptr, n,
                                                                                   g->coo_src);
    KC_CUDA(cudaGetLastError());
    g->build_ms = timer.stop();
    finish_csr_stats(g);
}

void kc_free_dag(kc_graph *g) {
    if (g->rank) kc_free(g->rank, g->stream);
    if (g->orow_ptr) kc_free(g->orow_ptr, g->stream);
    if (g->ocol) kc_free(g->ocol, g->stream);
    if (g->ocoo) kc_free(g->ocoo, g->stream);
    if (g->esize) kc_free(g->esize, g->stream);
    g->esize = nullptr;
    g->rank = nullptr;
    g->orow_ptr = nullptr;
    g->ocol = nullptr;
    g->ocoo = nullptr;
    g->oriented = 0;
}

// K3: bulk peeling.  Returns rank via sort of (round, id); degeneracy = the
// highest level at which some vertex was removed.  core_of (optional, device
// int32[n]) receives every vertex's core number.
static void degeneracy_rank(kc_graph *g, int64_t *degeneracy, int64_t *rounds_out,
                            int32_t *core_of = nullptr, bool want_rank = true) {
    const int64_t n = g->n;
    KC_REQUIRE(n < (int64_t(1) << 31), KC_EINVAL, "graph too large for 32-bit vertex ids");
    int32_t *deg = kc_alloc<int32_t>(n, g->stream);
    int32_t *round_of = kc_alloc<int32_t>(n, g->stream);
    int32_t *order = kc_alloc<int32_t>(n, g->stream);
    int32_t *ctl = kc_alloc<int32_t>(8, g->stream);
    // one 1024-thread CTA per SM: grid barriers cost grow with the CTA count
    constexpr int kPeelThreads = 1024;
    int per_sm = 0;
    KC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_peel_coop, kPeelThreads, 0));
    KC_REQUIRE(per_sm > 0, KC_ECUDA, "peel kernel cannot be resident");
    int grid = g->num_sms;
    const int64_t want = (n + kPeelThreads - 1) / kPeelThreads;
    if (want < grid) grid = int(want < 1 ? 1 : want);
    const int64_t *rp = g->row_ptr;
    const int32_t *cl = g->col;
    int64_t nn = n;
    void *args[] = {(void *)&rp, (void *)&cl, (void *)&nn, (void *)&deg, (void *)&round_of,
                    (void *)&order, (void *)&ctl, (void *)&core_of};
    KC_CUDA(cudaLaunchCooperativeKernel((void *)k_peel_coop, dim3(grid), dim3(kPeelThreads), args,
                                        0, g->stream));
    int32_t h[8] = {0};
    KC_CUDA(cudaMemcpyAsync(h, ctl, sizeof(h), cudaMemcpyDeviceToHost, g->stream));
    KC_CUDA(cudaStreamSynchronize(g->stream));
    const int32_t round = h[7];
    *degeneracy = h[6];
    *rounds_out = round;
    if (!want_rank) {
        kc_free(deg, g->stream);
        kc_free(round_of, g->stream);
        kc_free(order, g->stream);
        kc_free(ctl, g->stream);
        return;
    }
    // rank = position in (round, id) order
    int bits = kc_bits_for(n - 1 > 0 ? n - 1 : 1);
    int rbits = kc_bits_for(round > 0 ? round : 1);
    KC_REQUIRE(bits + rbits <= 64, KC_EINVAL, "too many peel rounds");
    uint64_t *keys = kc_alloc<uint64_t>(n, g->stream);
    uint64_t *keys2 = kc_alloc<uint64_t>(n, g->stream);
    const int g1 = grid_for(n, g->num_sms);
    k_peel_keys<<<g1, kThreads, 0, g->stream>>>(round_of, n, bits, keys);
    sort_u64(g, keys, keys2, n, bits + rbits);
    k_rank_from_sorted<<<g1, kThreads, 0, g->stream>>>(keys2, n, bits, g->rank);
    KC_CUDA(cudaGetLastError());
    kc_free(keys, g->stream);
    kc_free(keys2, g->stream);
    kc_free(deg, g->stream);
    kc_free(round_of, g->stream);
    kc_free(order, g->stream);
    kc_free(ctl, g->stream);
}

// exact sequential order (reference heap, orientation.py:81-113): core
// numbers from the bulk peel, then the per-shell-component heap runs and
// their merge (kc_peel.cu)
static void exact_degeneracy_rank(kc_graph *g, int64_t *degeneracy, int64_t *rounds) {
    const int64_t n = g->n;
    int32_t *core = kc_alloc<int32_t>(n, g->stream);
    degeneracy_rank(g, degeneracy, rounds, core, false);
    kc_exact_order_from_cores(g, core, *degeneracy, g->rank);
    kc_free(core, g->stream);
}

void kc_do_orient(kc_graph *g, int criterion, const int32_t *rank_in, kc_dag_info *info) {
    KC_REQUIRE(criterion == KC_CRIT_DEGREE || criterion == KC_CRIT_DEGENERACY ||
                   criterion == KC_CRIT_GIVEN || criterion == KC_CRIT_DEGENERACY_EXACT ||
                   criterion == KC_CRIT_DEGENERACY_BULK,
               KC_EINVAL, "unknown orientation criterion");
    KC_REQUIRE(criterion != KC_CRIT_GIVEN || rank_in, KC_EINVAL, "rank_in required");
    kc_free_dag(g);
    const int64_t n = g->n, two_m = 2 * g->m;
    g->rank = kc_alloc<int32_t>(n, g->stream);
    int64_t degen = -1, rounds = 0;
    EventTimer t_rank(g->stream);
    if (n > 0) {
        const int grid = grid_for(n, g->num_sms);
        if (criterion == KC_CRIT_DEGREE) {
            // orientation.py:124-128: lexsort((arange(n), degrees))
            int bits = kc_bits_for(n - 1 > 0 ? n - 1 : 1);
            int dbits = kc_bits_for(g->d_max_und > 0 ? g->d_max_und : 1);
            uint64_t *keys = kc_alloc<uint64_t>(n, g->stream);
            uint64_t *keys2 = kc_alloc<uint64_t>(n, g->stream);
            k_degree_keys<<<grid, kThreads, 0, g->stream>>>(g->row_ptr, n, bits, keys);
            sort_u64(g, keys, keys2, n, bits + dbits);
            k_rank_from_sorted<<<grid, kThreads, 0, g->stream>>>(keys2, n, bits, g->rank);
            KC_CUDA(cudaGetLastError());
            KC_CUDA(cudaStreamSynchronize(g->stream));
            kc_free(keys, g->stream);
            kc_free(keys2, g->stream);
        } else if (criterion == KC_CRIT_DEGENERACY_BULK) {
            degeneracy_rank(g, &degen, &rounds);
        } else if (criterion == KC_CRIT_DEGENERACY || criterion == KC_CRIT_DEGENERACY_EXACT) {
            exact_degeneracy_rank(g, &degen, &rounds);
        } else {
            KC_CUDA(cudaMemcpyAsync(g->rank, rank_in, 4 * n, cudaMemcpyHostToDevice, g->stream));
        }
    } else if (criterion == KC_CRIT_DEGENERACY || criterion == KC_CRIT_DEGENERACY_EXACT ||
               criterion == KC_CRIT_DEGENERACY_BULK) {
        degen = 0;
    }
    double rank_ms = t_rank.stop();

    EventTimer t_orient(g->stream);
    g->orow_ptr = kc_alloc<int64_t>(n + 1, g->stream);
    g->ocol = kc_alloc<int32_t>(g->m, g->stream);
    g->ocoo = kc_alloc<int32_t>(g->m, g->stream);
    int64_t m_dir = 0;
    unsigned long long d_max = 0;
    if (n == 0) {
        KC_CUDA(cudaMemsetAsync(g->orow_ptr, 0, 8, g->stream));
    } else if (two_m == 0) {
        KC_CUDA(cudaMemsetAsync(g->orow_ptr, 0, 8 * (n + 1), g->stream));
    } else {
        uint8_t *flags = kc_alloc<uint8_t>(two_m, g->stream);
        int32_t *d_cnt = kc_alloc<int32_t>(1, g->stream);
        k_orient_flags<<<grid_for(two_m, g->num_sms), kThreads, 0, g->stream>>>(
            g->col, g->coo_src, g->rank, two_m, flags);
        size_t bytes = 0;
        KC_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, g->col, flags, g->ocol, d_cnt,
                                           int(two_m), g->stream));
        void *tmp = kc_tmp(g, bytes);
        KC_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, g->col, flags, g->ocol, d_cnt, int(two_m),
                                           g->stream));
        KC_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, g->coo_src, flags, g->ocoo, d_cnt,
                                           int(two_m), g->stream));
        int32_t h = 0;
        KC_CUDA(cudaMemcpyAsync(&h, d_cnt, 4, cudaMemcpyDeviceToHost, g->stream));
        KC_CUDA(cudaStreamSynchronize(g->stream));
        m_dir = h;
        k_row_ptr<<<grid_for(n + 1, g->num_sms), kThreads, 0, g->stream>>>(g->ocoo, m_dir, n,
                                                                            g->orow_ptr);
        unsigned long long *d_dmax = kc_alloc<unsigned long long>(1, g->stream);
        KC_CUDA(cudaMemsetAsync(d_dmax, 0, 8, g->stream));
        k_out_degree_max<<<grid_for(n, g->num_sms), kThreads, 0, g->stream>>>(g->orow_ptr, n,
                                                                               d_dmax);
        KC_CUDA(cudaMemcpyAsync(&d_max, d_dmax, 8, cudaMemcpyDeviceToHost, g->stream));
        KC_CUDA(cudaGetLastError());
        KC_CUDA(cudaStreamSynchronize(g->stream));
        kc_free(d_dmax, g->stream);
        kc_free(flags, g->stream);
        kc_free(d_cnt, g->stream);
    }
    double orient_ms = t_orient.stop();
    g->m_dir = m_dir;
    g->d_max = int64_t(d_max);
    g->degeneracy = degen;
    g->criterion = criterion;
    g->oriented = 1;
    if (info) {
        info->m_dir = m_dir;
        info->d_max = int64_t(d_max);
        info->degeneracy = degen;
        info->rounds = rounds;
        info->rank_ms = rank_ms;
        info->orient_ms = orient_ms;
    }
}

int64_t kc_task_count(const kc_graph *g, int scheme) {
    if (scheme == KC_SCHEME_EDGE) return g->m_dir;
    if (g->n == 0) return 0;
    int32_t *flag = kc_alloc<int32_t>(g->n, g->stream);
    int32_t *out = kc_alloc<int32_t>(1, g->stream);
    k_vertex_task_flags<<<grid_for(g->n, g->num_sms), kThreads, 0, g->stream>>>(g->orow_ptr, g->n,
                                                                                 flag);
    size_t bytes = 0;
    KC_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, flag, out, int(g->n), g->stream));
    void *tmp = kc_tmp(const_cast<kc_graph *>(g), bytes);
    KC_CUDA(cub::DeviceReduce::Sum(tmp, bytes, flag, out, int(g->n), g->stream));
    int32_t h = 0;
    KC_CUDA(cudaMemcpyAsync(&h, out, 4, cudaMemcpyDeviceToHost, g->stream));
    KC_CUDA(cudaStreamSynchronize(g->stream));
    kc_free(flag, g->stream);
    kc_free(out, g->stream);
    return h;
}
