// kc_count.cu -- K4 induce_bitmap, K5 orient_traverse, K6 pivot_traverse,
// K7 pivot_traverse_allk, K8 u128 limb reduction.
//
// One persistent kernel per (algorithm): CTAs pull tasks (root vertices or
// oriented edges) from a global atomic queue (replacing the
// reference's thread-pool cursor scheduler.py:141-149).  Per task the CTA
//   K4: builds the binary-encoded induced sub-graph of the task's locals in
//       shared memory (bitgraph.py:59-111 semantics: locals ascending by compact
//       id; bit j of row i <=> arc l2g[i]->l2g[j] (directed) / either arc
//       (undirected)); u32 words, LSB-first, rows padded to an odd stride so
//       lane-divergent row reads spread over the 32 banks;
//   K5: orient -- sub-warp groups of G lanes (1..32, per task or fixed,
//       PAPER.md:461-465) take level-2 subtrees from a shared counter and walk
//       them depth-first with a private stack (engine_orient.py:32-79).  Lane g
//       owns words g, g+G, ... of every stack row; candidate selection by
//       __ballot_sync + __shfl_sync + __ffs; the last level is AND+__popc only,
//       accumulated per lane without reductions;
//   K6/K7: pivot -- warps take the root's branch vertices and walk Fig.3
//       (engine_pivot.py:117-233).  Pivot choice scores candidates lane-parallel
//       (argmax |cand & row(v)|, lowest id on ties, engine_pivot.py:82-101).
//       Leaves are binned in a (path length, pivots) histogram; the binomial
//       expansion happens once on the host, exactly (K7 for all k at once).
// K8: per-thread u64 partials -> 32-bit limb sums -> atomics; the host carries
//     them into the exact 128-bit count.  Visited nodes are tallied per SM.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <vector>

#include "kc_internal.cuh"
#include "kc_traverse.cuh"

namespace {

typedef unsigned long long ull;

struct CountParams {
    const int64_t *orow;
    const int32_t *ocol;
    const int32_t *ocoo;
    const int32_t *tasks;
    int64_t n_tasks;
    int scheme;        // KC_SCHEME_*
    int t;             // target inside a task
    int all_k;         // pivot all-k
    int split;         // tasks are out-edges of split vertex roots (see kc_do_count)
    const int32_t *task_w;  // split triples: third vertex w of task (v,u,w), else nullptr;
                            // pivot branch tasks: the root branch v (local index)
    int branch;             // pivot: tasks are root branches (task, v) of split tasks
    int roots_only;         // pivot: compute the root frame of each task (split pass)
    const int32_t *branch_si;   // branch task -> split-task index
    int32_t *root_piv;          // split task -> root pivot (local index)
    uint32_t *root_P;           // split task -> root branch set P0 (4 words)
    int32_t *root_cnt;          // split task -> |P0| (0: task skipped)
    int32_t *overflow;   // warp kernel: edge tasks with more than kWarpD locals
    int32_t *overflow_w;  // and their third vertex (triples)
    ull *overflow_n;
    kct::GQueue gq;      // pivot: GPU-wide subtree queue of the warp-tier kernel
    int use_gq;
    int gq_push_min, gq_cooldown, gq_room;  // hand-over policy (kct::PivotLeafSink)
    int dcap;          // max locals per task
    int wcap;          // ceil(dcap / 32)
    int group_size;    // orientation warp tier: lanes per sub-warp group (1..32)
    int rows_in_smem;  // rows in shared memory, else in rows_global slot
    uint32_t *rows_global;
    int64_t rows_slot;   // u32 words per CTA slot
    int nsm_frames;      // DFS frames per warp held in shared memory
    int fw;              // words per frame
    uint32_t *frames_global;  // deeper frames, one slot per warp
    int64_t frames_slot;      // u32 words per warp slot
    int hist_dim;        // pivot: L (hist is L x L)
    ull *hist;
    int sh_hl;           // pivot: shared histogram side (len < sh_hl)
    const uint32_t *given_rows;  // engine entry: one host-provided matrix
    int given_d;
    int directed_out;            // extract entry: 1 = directed
    uint32_t *extract_rows;      // extract entry outputs
    int32_t *extract_l2g;
    int *extract_d;
    ull *task_counter;
    ull *limbs;          // [4]
    ull *visits_total;
    ull *word_ops;       // roofline counters (kc_count_raw.word_ops / extract_bytes)
    ull *ext_bytes;
    ull *visits_per_sm;
    ull *tasks_run;
    ull *prof;  // KC_TIMING diagnostics (nullptr: off): see kProf* below
    // pivot bounded walks (kct::Spill): items out, and (spill rounds) items in
    kct::Spill spill;
    int use_spill;
    int spill_budget;
    const uint32_t *in_buf;  // spill round: task i is the item at in_buf + in_off[i]
    const uint32_t *in_off;
    int mid_max;  // CTA tier: largest pair-level set compressed (128 or 256; KC_MID_MAX)
};
// prof words: CTA tier build / walk cycles (thread 0), warp tier build / walk
// cycles (lane 0, summed over warps), then a histogram of overflow task sizes
// in buckets of 32 locals
constexpr int kProfCtaBuild = 0, kProfCtaWalk = 1, kProfWarpBuild = 2, kProfWarpWalk = 3,
              kProfOvfHist = 4, kProfGqIdle = 68, kProfGqWalk = 69, kProfGqItems = 70,
              kProfWords = 72;

__host__ __device__ __forceinline__ int row_stride(int W) { return W | 1; }
// warp tier, orientation: rows of 2..4 words padded to 16 bytes so the
// last-two-levels loop reads a row with one 128-bit load (kc_traverse.cuh)
__host__ __device__ __forceinline__ int warp_row_stride(int W, bool orient) {
    return (orient && W >= 2 && W <= 4) ? 4 : row_stride(W);
}

// ---------------------------------------------------------------------------
// K4: locals + bit matrix
// ---------------------------------------------------------------------------
// Ordered block-wide append of flagged values (keeps chunk order).
template <int BLOCK>
__device__ __forceinline__ void block_append(bool flag, int32_t value, int32_t *out, int *s_count,
                                             int *s_warp) {
    constexpr int NW = BLOCK / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned b = __ballot_sync(0xffffffffu, flag);
    if (lane == 0) s_warp[warp] = __popc(b);
    __syncthreads();
    int base = *s_count;
    int off = 0, total = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        int c = s_warp[w];
        off += w < warp ? c : 0;
        total += c;
    }
    if (flag) out[base + off + __popc(b & ((1u << lane) - 1))] = value;
    __syncthreads();
    if (threadIdx.x == 0) *s_count = base + total;
    __syncthreads();
}

__device__ __forceinline__ int smem_find(const int32_t *a, int n, int32_t x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return (lo < n && a[lo] == x) ? lo : -1;
}

__device__ __forceinline__ bool gl_contains(const int32_t *__restrict__ a, int n, int32_t x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < x) lo = mid + 1;
        else hi = mid;
    }
    return lo < n && __ldg(a + lo) == x;
}

template <int BLOCK>
__device__ void rows_from_locals(const CountParams &p, const int32_t *l2g, int d, uint32_t *rows,
                                 int32_t *scratch, bool directed, ull &bytes);

// Returns d (number of locals); fills l2g and (when t >= 2 or pivot) rows.
// scratch must hold >= dcap int32 (used for the edge scheme's second list).
template <int BLOCK>
__device__ int build_task(const CountParams &p, int32_t task, int32_t *l2g, uint32_t *rows,
                          int32_t *scratch, bool need_rows, bool directed, int *s_cnt,
                          int *s_warp, ull &bytes, int32_t w3 = -1) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = BLOCK / 32;
    int d;
    if (p.scheme == KC_SCHEME_VERTEX) {
        // bitgraph.py:59-64 locals = out-neighbours of the root
        const int64_t beg = p.orow[task];
        d = int(p.orow[task + 1] - beg);
        for (int i = tid; i < d; i += BLOCK) l2g[i] = p.ocol[beg + i];
        if (tid == 0) bytes += 4 /*task id*/ + 16 + 4ull * d;
    } else {
        // bitgraph.py:67-86 locals = common out-neighbours of (src, dst);
        // the longer list is staged in smem, the shorter one is probed
        const int32_t u = p.ocoo[task], v = p.ocol[task];
        int64_t ab = p.orow[u], ae = p.orow[u + 1], bb = p.orow[v], be = p.orow[v + 1];
        if (ae - ab > be - bb) {
            int64_t t0 = ab, t1 = ae;
            ab = bb; ae = be; bb = t0; be = t1;
        }
        const int la = int(ae - ab), lb = int(be - bb);
        if (tid == 0) bytes += 4 + 8 + 32 + 4ull * (la + lb);
        for (int i = tid; i < lb; i += BLOCK) scratch[i] = p.ocol[bb + i];
        if (tid == 0) *s_cnt = 0;
        __syncthreads();
        for (int c = 0; c < la; c += BLOCK) {
            int i = c + tid;
            int32_t x = i < la ? p.ocol[ab + i] : 0;
            bool f = i < la && smem_find(scratch, lb, x) >= 0;
            if (w3 >= 0 && f)  // triple (v,u,w): also a out-neighbour of w
                f = gl_contains(p.ocol + p.orow[w3], int(p.orow[w3 + 1] - p.orow[w3]), x);
            block_append<BLOCK>(f, x, l2g, s_cnt, s_warp);
        }
        d = *s_cnt;
    }
    __syncthreads();
    if (!need_rows || d == 0) return d;
    rows_from_locals<BLOCK>(p, l2g, d, rows, scratch, directed, bytes);
    return d;
}

// bit matrix of the sub-graph induced by the sorted vertices l2g[0..d)
// (bitgraph.py:89-111: bit j of row i <=> arc l2g[i] -> l2g[j], or either
// arc when undirected); whole block, ends with a barrier
template <int BLOCK>
__device__ void rows_from_locals(const CountParams &p, const int32_t *l2g, int d, uint32_t *rows,
                                 int32_t *scratch, bool directed, ull &bytes) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = BLOCK / 32;
    const int W = (d + 31) >> 5, RS = row_stride(W);
    for (int i = tid; i < d * RS; i += BLOCK) rows[i] = 0u;
    // orientation: global id -> local index by open addressing over H >= 2d
    // slots in the (now free) staging area -- a miss costs ~2.5 probes, not a
    // binary search.  (The pivot engine keeps its per-warp leaf histograms in
    // that area across tasks, so it searches l2g instead.)
    int hb = 1;
    while ((1 << hb) < 2 * d) ++hb;
    const int H = 1 << hb;
    int32_t *hkey = scratch;
    int16_t *hval = reinterpret_cast<int16_t *>(scratch + H);
    if (directed) {
        for (int i = tid; i < H; i += BLOCK) hkey[i] = -1;
        __syncthreads();
        for (int i = tid; i < d; i += BLOCK) {
            const int32_t x = l2g[i];
            uint32_t h = (uint32_t(x) * 0x9E3779B1u) >> (32 - hb);
            while (atomicCAS(hkey + h, -1, x) != -1) h = (h + 1) & uint32_t(H - 1);
            hval[h] = int16_t(i);
        }
    }
    __syncthreads();
    auto find = [&](int32_t x) -> int {
        if (!directed) return smem_find(l2g, d, x);
        uint32_t h = (uint32_t(x) * 0x9E3779B1u) >> (32 - hb);
        for (;;) {
            const int32_t k = hkey[h];
            if (k == x) return hval[h];
            if (k < 0) return -1;
            h = (h + 1) & uint32_t(H - 1);
        }
    };
    // bitgraph.py:89-111: bit j of row i <=> l2g[j] in N+(l2g[i]); the scan of
    // each local's out-list replaces the reference's pairwise binary searches
    const int32_t lo_id = l2g[0], hi_id = l2g[d - 1];
    for (int i = warp; i < d; i += NW) {
        const int32_t gi = l2g[i];
        const int64_t beg = p.orow[gi], end = p.orow[gi + 1];
        if (lane == 0) bytes += 16 + 4ull * (end - beg);
        for (int64_t e = beg + lane; e < end; e += 32) {
            const int32_t x = p.ocol[e];
            if (x < lo_id || x > hi_id) continue;
            const int j = find(x);
            if (j >= 0) {
                atomicOr(&rows[i * RS + (j >> 5)], 1u << (j & 31));
                if (!directed) atomicOr(&rows[j * RS + (i >> 5)], 1u << (i & 31));
            }
        }
    }
    __syncthreads();
}

// engine entry: load a host-provided matrix instead of extracting
template <int BLOCK>
__device__ int load_given(const CountParams &p, uint32_t *rows) {
    const int d = p.given_d;
    const int W = (d + 31) >> 5, RS = row_stride(W);
    for (int i = threadIdx.x; i < d * RS; i += BLOCK) {
        int r = i / RS, w = i - r * RS;
        rows[i] = w < W ? p.given_rows[r * W + w] : 0u;
    }
    __syncthreads();
    return d;
}

// ---------------------------------------------------------------------------
// block reductions for the K8 epilogue
// ---------------------------------------------------------------------------
template <int BLOCK>
__device__ void flush_block(const CountParams &p, ull acc, ull visits, ull tasks, ull work,
                            ull bytes, ull *s_red) {
    constexpr int NW = BLOCK / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    ull lo = acc & 0xffffffffull, hi = acc >> 32;
    for (int o = 16; o; o >>= 1) {
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
        hi += __shfl_xor_sync(0xffffffffu, hi, o);
        visits += __shfl_xor_sync(0xffffffffu, visits, o);
        tasks += __shfl_xor_sync(0xffffffffu, tasks, o);
        work += __shfl_xor_sync(0xffffffffu, work, o);
        bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
    }
    __syncthreads();
    if (lane == 0) {
        if (work && p.word_ops) atomicAdd(p.word_ops, work);
        if (bytes && p.ext_bytes) atomicAdd(p.ext_bytes, bytes);
        s_red[4 * warp + 0] = lo;
        s_red[4 * warp + 1] = hi;
        s_red[4 * warp + 2] = visits;
        s_red[4 * warp + 3] = tasks;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        ull a = 0, b = 0, c = 0, dd = 0;
        for (int w = 0; w < NW; ++w) {
            a += s_red[4 * w];
            b += s_red[4 * w + 1];
            c += s_red[4 * w + 2];
            dd += s_red[4 * w + 3];
        }
        if (a) atomicAdd(&p.limbs[0], a);
        if (b) atomicAdd(&p.limbs[1], b);
        if (c) {
            atomicAdd(p.visits_total, c);
            if (p.visits_per_sm) atomicAdd(&p.visits_per_sm[kc_smid()], c);
        }
        if (dd) atomicAdd(p.tasks_run, dd);
    }
}

// ---------------------------------------------------------------------------
// K5: orient traversal -- warps take level-1 subtrees (kc_traverse.cuh)
// ---------------------------------------------------------------------------
template <int BLOCK, int WPL>
__device__ void orient_task(const CountParams &p, const uint32_t *rows, int d,
                            const kct::Frames &F, int *list, uint32_t *cbuf,
                            const kct::SmallScratch &SS, int *s_next, ull &acc, ull &visits,
                            ull &work) {
    const int W = (d + 31) >> 5, RS = row_stride(W);
    const int last = p.t - 2;
    if (last == 0) {
        // t == 2: each local u is a visit; count popc(S0 & row u) (engine_orient.py:64-69)
        for (int u = threadIdx.x; u < d; u += BLOCK) {
            const uint32_t *ru = rows + u * RS;
            int c = 0;
            for (int w = 0; w < W; ++w) c += __popc(ru[w]);
            acc += ull(c);
            ++visits;
            work += 1;
        }
        return;
    }
    const int lane = threadIdx.x & 31;
    for (;;) {
        int u = 0;
        if (lane == 0) u = atomicAdd(s_next, 1);
        u = __shfl_sync(kct::FULL, u, 0);
        if (u >= d) break;
        if (lane == 0) {
            ++visits;
            work += 1;
        }
        kct::orient_subtree<WPL>(rows, RS, W, last, u, F, list, cbuf, SS, acc, visits, work);
    }
}

// ---------------------------------------------------------------------------
// K6/K7: pivot traversal -- root frame by the block, branches by warps
// ---------------------------------------------------------------------------
template <int BLOCK, int WPL>
__device__ void pivot_task(const CountParams &p, const uint32_t *rows, int d, uint32_t *S0,
                           uint32_t *P0, const kct::Frames &F, int *list,
                           const kct::SmallScratch &SS, const kct::PivotLeafSink &sink,
                           const kct::StealStack &q, int *s_next, int *s_piv0, ull *s_key,
                           ull &visits, ull &work, int s0 = 0, int npv0 = 0) {
    constexpr int NW = BLOCK / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = (d + 31) >> 5, RS = row_stride(W);
    // root frame (engine_pivot.py:133-136): S0 = all locals, pivot = argmax |row c|
    // (a spilled item: S0 = all members of the item's set, at depth s0 with
    // npv0 pivots)
    for (int w = tid; w < 32 * WPL; w += BLOCK) {
        const int lo = w << 5;
        S0[w] = lo >= d ? 0u : (lo + 32 <= d ? kct::FULL : ((1u << (d - lo)) - 1u));
    }
    ull best = 0;
    for (int c = tid; c < d; c += BLOCK) {
        const uint32_t *rc = rows + c * RS;
        int cov = 0;
        for (int w = 0; w < W; ++w) cov += __popc(rc[w]);
        const ull key = (ull(cov + 1) << 32) | ull(0xffffffffu - uint32_t(c));
        best = key > best ? key : best;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const ull y = __shfl_xor_sync(kct::FULL, best, o);
        best = y > best ? y : best;
    }
    if (lane == 0) s_key[warp] = best;
    __syncthreads();
    if (tid == 0) {
        ull b = 0;
        for (int w = 0; w < NW; ++w) b = s_key[w] > b ? s_key[w] : b;
        *s_piv0 = int(0xffffffffu - uint32_t(b & 0xffffffffull));
        work += ull(d);
    }
    __syncthreads();
    const int piv0 = *s_piv0;
    const uint32_t *rp0 = rows + piv0 * RS;
    for (int w = tid; w < 32 * WPL; w += BLOCK) P0[w] = w < W ? (S0[w] & ~rp0[w]) : 0u;
    if (tid == 0) {
        *q.lock = 0;
        *q.size = 0;
        *q.idle = 0;
    }
    __syncthreads();
    for (;;) {
        int v = 0;
        if (lane == 0) v = atomicAdd(s_next, 1);
        v = __shfl_sync(kct::FULL, v, 0);
        if (v >= d) break;
        if (!((P0[v >> 5] >> (v & 31)) & 1u)) continue;
        kct::pivot_subtree<WPL>(rows, RS, W, p.t, p.all_k != 0, v, piv0, S0, P0, F, list, SS,
                                sink, visits, work, &q, s0, npv0);
    }
    kct::pivot_steal_loop<WPL>(rows, RS, W, p.t, p.all_k != 0, F, list, SS, sink, q, visits, work);
}

// ---------------------------------------------------------------------------
// the persistent kernel
// ---------------------------------------------------------------------------
enum Mode { MODE_ORIENT = 0, MODE_PIVOT = 1, MODE_EXTRACT = 2 };
constexpr int kCtaSmallWords = 32;  // CTA tier per-warp S-tier rows (srow)
constexpr int kStealCap = 16;  // pivot work-sharing stack slots per CTA

template <int BLOCK, int MODE, int WPL, bool GQ = false>
__global__ void __launch_bounds__(BLOCK) k_count(CountParams p) {
    constexpr int NW = BLOCK / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_next, s_piv0, s_cnt, s_task;
    __shared__ int s_warp[NW];
    __shared__ ull s_key[NW];
    __shared__ ull s_red[4 * NW];
    const int tid = threadIdx.x, warp = tid >> 5;
    // layout: [l2g i32 dcap][rows u32][S0 P0][per warp: list, cbuf, S-tier, leaf hist, frames]
    int32_t *l2g = reinterpret_cast<int32_t *>(smem);
    uint32_t *area = reinterpret_cast<uint32_t *>(l2g + ((p.dcap + 3) & ~3));
    uint32_t *rows;
    if (p.rows_in_smem) {
        rows = area;
        area += ((int64_t(p.dcap) * row_stride(p.wcap) + 3) & ~3);
    } else {
        rows = p.rows_global + int64_t(blockIdx.x) * p.rows_slot;
    }
    int32_t *scratch = reinterpret_cast<int32_t *>(area);  // edge-scheme staging (pre-traversal)
    uint32_t *S0 = area, *P0 = area + 32 * WPL;
    kct::StealStack q;
    __shared__ int s_q[3];
    q.lock = s_q;
    q.size = s_q + 1;
    q.idle = s_q + 2;
    q.cap = kStealCap;
    q.iw = 32 * WPL + 4;
    q.nwarps = NW;
    q.items = area + 64 * WPL;
    if (MODE == MODE_PIVOT) area += 64 * WPL + kStealCap * (32 * WPL + 4);
    const int hist_cells = MODE == MODE_PIVOT ? kct::kLeafCells : 0;
    // compressed pair-level rows: only where a pair level exists (t >= 4)
    const int mid_words =
        (MODE == MODE_ORIENT && p.t >= 4) ? kct::mid_words(WPL, p.mid_max) : 0;
    // per-warp S-tier rows only: the CTA tier has no LocalMap (kct::kSmallWords)
    // pivot: per-lane S-tier walks need a node stack per warp
    const int node_words = MODE == MODE_PIVOT ? 2 * kct::kNodeCap : 0;
    const int per_warp = ((p.dcap + 3) & ~3) + 32 * WPL + kCtaSmallWords + hist_cells +
                         mid_words + node_words + p.nsm_frames * p.fw;
    int *list = reinterpret_cast<int *>(area + warp * per_warp);
    uint32_t *cbuf = area + warp * per_warp + ((p.dcap + 3) & ~3);
    kct::SmallScratch SS;
    SS.srow = cbuf + 32 * WPL;
    SS.sstk = nullptr;  // (unused by the CTA-tier walks)
    uint32_t *whist = SS.srow + kCtaSmallWords;
    if (mid_words) {  // compressed pair levels of <= p.mid_max members
        SS.mrow = whist + hist_cells;
        SS.mid_max = p.mid_max;
    }
    if (node_words) {
        SS.nstk = reinterpret_cast<uint2 *>(whist + hist_cells + mid_words);
        SS.ncap = kct::kNodeCap;
    }
    kct::Frames F;
    F.sm = whist + hist_cells + mid_words + node_words;
    F.nsm = p.nsm_frames;
    F.fw = p.fw;
    F.gm = p.frames_global ? p.frames_global + (int64_t(blockIdx.x) * NW + warp) * p.frames_slot
                           : nullptr;
    __shared__ int s_hc[4 * NW];
    __shared__ int s_spill;  // bounded walks: set once a warp of the task is over budget
    kct::PivotLeafSink sink;
    sink.whist = whist;
    sink.g_hist = p.hist;
    sink.L = p.hist_dim;
    // queue / spill descriptors copied to shared memory: taking the address
    // of a kernel parameter would copy the whole CountParams to local memory
    __shared__ kct::GQueue s_gq;
    __shared__ kct::Spill s_sp;
    if (tid == 0) {
        s_gq = p.gq;
        s_sp = p.spill;
    }
    __syncthreads();
    sink.gq = (GQ && MODE == MODE_PIVOT) ? &s_gq : nullptr;  // compile-time off when !GQ
    sink.eager = true;  // CTA tier
    sink.l2g = l2g;
    sink.hc = s_hc + 4 * warp;
    if (MODE == MODE_PIVOT && p.use_spill) {
        sink.sp = &s_sp;
        sink.cta_flag = &s_spill;
    }
    sink.push_min = p.gq_push_min;
    sink.cooldown = p.gq_cooldown;
    sink.room_min = p.gq_room;
    if ((tid & 31) == 0) {
        sink.hc[0] = 0;
        sink.hc[1] = 0;
        if (sink.gq) atomicAdd(p.gq.ctl + 3, 1);  // busy: this warp may push to the warp tier
    }

    for (int i = tid & 31; i < hist_cells; i += 32) whist[i] = 0;
    ull acc = 0, visits = 0, tasks = 0, work = 0, bytes = 0;
    const bool directed = MODE == MODE_ORIENT || (MODE == MODE_EXTRACT && p.directed_out);
    const int t = p.t;
    long long pc_walk = 0;
    for (;;) {
        __syncthreads();
        if (p.prof && tid == 0 && pc_walk) {
            atomicAdd(&p.prof[kProfCtaWalk], ull(clock64() - pc_walk));
            pc_walk = 0;
        }
        if (tid == 0) {
            ull i = p.given_rows ? (blockIdx.x == 0 ? atomicAdd(p.task_counter, 1ull) : ~0ull)
                                 : atomicAdd(p.task_counter, 1ull);
            s_task = i < ull(p.n_tasks) ? int(i) : -1;
            s_next = 0;
            s_spill = 0;
        }
        if (sink.sp) sink.set_budget(p.spill_budget, tid & 31);
        __syncthreads();
        if (s_task < 0) break;
        int d;
        int it_s = 0, it_npv = 0;  // spill round: the item's depth and pivot count
        const long long pc0 = (p.prof && tid == 0) ? clock64() : 0;
        if (p.given_rows) {
            d = load_given<BLOCK>(p, rows);
        } else if (MODE == MODE_PIVOT && p.in_buf) {
            // spilled item (kind 0, more than kWarpD members): its set's ids
            // are the locals; the sub-graph induced by them is undirected
            const uint32_t *it = p.in_buf + p.in_off[s_task];
            d = int(it[1]);
            it_s = int(it[2]);
            it_npv = int(it[3]);
            for (int i = tid; i < d; i += BLOCK) l2g[i] = int32_t(it[4 + i]);
            __syncthreads();
            rows_from_locals<BLOCK>(p, l2g, d, rows, scratch, false, bytes);
        } else {
            const int32_t task = p.tasks[s_task];
            const bool need_rows = MODE == MODE_EXTRACT || MODE == MODE_PIVOT || t >= 2;
            d = build_task<BLOCK>(p, task, l2g, rows, scratch, need_rows, directed, &s_cnt, s_warp,
                                  bytes, p.task_w ? p.task_w[s_task] : -1);
        }
        if (MODE == MODE_EXTRACT) {
            const int W = (d + 31) >> 5, RS = row_stride(W);
            for (int i = tid; i < d; i += BLOCK) p.extract_l2g[i] = l2g[i];
            for (int i = tid; i < d * W; i += BLOCK) {
                int r = i / W, w = i - r * W;
                p.extract_rows[i] = rows[r * RS + w];
            }
            if (tid == 0) *p.extract_d = d;
            continue;
        }
        if (MODE == MODE_PIVOT && p.in_buf) {
            // an item is a node inside a counted task: no task, no visit here
            const ull wt0 = work;
            pivot_task<BLOCK, WPL>(p, rows, d, S0, P0, F, list, SS, sink, q, &s_next, &s_piv0,
                                   s_key, visits, work, it_s, it_npv);
            work = wt0 + (work - wt0) * ull((d + 31) >> 5);
            continue;
        }
        if (p.split) {
            // edge item (v,u) of a split vertex root v: u is a level-1 visit of
            // v's tree and the item walks u's subtree whatever its size
            if (tid == 0) ++visits;
            if (d == 0) continue;
        } else if (MODE == MODE_PIVOT && p.all_k) {
            if (d == 0) continue;  // scheduler.py:180-181
        } else if (d < t) {
            continue;  // scheduler.py:155-156
        }
        if (tid == 0) ++tasks;
        if (t <= 1 && !(MODE == MODE_PIVOT && p.all_k)) {
            // engine_orient.py:38-42 / engine_pivot.py:124-128
            if (tid == 0) acc += t == 0 ? 1ull : ull(d);
            continue;
        }
        const ull wt0 = work;  // units -> §8(d) word-ops of this task below
        const long long pc1 = (p.prof && tid == 0) ? clock64() : 0;
        if (MODE == MODE_ORIENT) {
            orient_task<BLOCK, WPL>(p, rows, d, F, list, cbuf, SS, &s_next, acc, visits, work);
        } else {
            pivot_task<BLOCK, WPL>(p, rows, d, S0, P0, F, list, SS, sink, q, &s_next, &s_piv0,
                                   s_key, visits, work);
        }
        work = wt0 + (work - wt0) * ull((d + 31) >> 5);
        if (p.prof && tid == 0) {
            atomicAdd(&p.prof[kProfCtaBuild], ull(pc1 - pc0));
            pc_walk = pc1;  // closed at the next task's opening barrier
        }
    }
    __syncthreads();
    if (MODE == MODE_PIVOT) sink.flush(tid & 31);
    if (sink.gq && (tid & 31) == 0) {
        atomicSub(p.gq.ctl + 3, 1);  // no longer busy (pushed items are drained by thieves)
    }
    if (MODE != MODE_EXTRACT) flush_block<BLOCK>(p, acc, visits, tasks, work, bytes, s_red);
}

// ---------------------------------------------------------------------------
// warp-per-task kernel for small tasks (d <= kWarpD): no CTA barriers, every
// warp fetches, extracts and walks its own tasks (PAPER.md:461-465 sub-block
// partitioning taken to one task per warp).  Tasks with d <= 32 run entirely
// in the S-tier (their rows already are one word).
// ---------------------------------------------------------------------------
constexpr int kWarpD = 128;
constexpr int kGqCap = 4096;  // GPU-wide subtree queue slots (pivot)
constexpr int kSplitD = 32;  // orientation/vertex: roots above this are split into edge items
constexpr int kAutoGroup = 8;  // orientation sub-warp group size for group_size = 0
constexpr int kPivotSplitD = 32;  // pivot: warp-tier tasks above this are split at the root


// warp-level bit matrix of the sub-graph induced by the sorted vertices l2g[0..d)
// (bitgraph.py:89-111: bit j of row i <=> arc l2g[i] -> l2g[j], or either arc)
__device__ void warp_rows(const CountParams &p, const int32_t *l2g, int d, uint32_t *rows,
                          bool directed, ull &bytes, const kct::SmallScratch &SS) {
    const int lane = threadIdx.x & 31;
    const int W = (d + 31) >> 5, RS = warp_row_stride(W, directed);
    for (int i = lane; i < d * RS; i += 32) rows[i] = 0u;
    kct::LocalMap map;
    map.key = reinterpret_cast<int32_t *>(SS.sstk);
    map.val = reinterpret_cast<uint8_t *>(SS.sstk + kct::kMapSlots);
    map.build(l2g, d, lane);  // ends with __syncwarp (rows zeroed too)
    const int32_t lo_id = l2g[0], hi_id = l2g[d - 1];
    for (int i = 0; i < d; ++i) {
        const int32_t gi = l2g[i];
        const int64_t beg = p.orow[gi], end = p.orow[gi + 1];
        if (lane == 0) bytes += 16 + 4ull * (end - beg);
        for (int64_t e = beg + lane; e < end; e += 32) {
            const int32_t x = p.ocol[e];
            if (x < lo_id || x > hi_id) continue;
            const int j = map.find(x);
            if (j >= 0) {
                atomicOr(&rows[i * RS + (j >> 5)], 1u << (j & 31));
                if (!directed) atomicOr(&rows[j * RS + (i >> 5)], 1u << (i & 31));
            }
        }
    }
    __syncwarp();
}

// warp-level K4: locals + bit matrix of one task (d <= kWarpD)
__device__ int warp_build(const CountParams &p, int32_t task, int32_t *l2g, uint32_t *rows,
                          bool need_rows, bool directed, ull &bytes, const kct::SmallScratch &SS,
                          int32_t w3 = -1) {
    const int lane = threadIdx.x & 31;
    int d;
    if (p.scheme == KC_SCHEME_VERTEX) {
        const int64_t beg = p.orow[task];
        d = int(p.orow[task + 1] - beg);
        for (int i = lane; i < d; i += 32) l2g[i] = p.ocol[beg + i];
        if (lane == 0) bytes += 4 + 16 + 4ull * d;
    } else {
        const int32_t u = p.ocoo[task], v = p.ocol[task];
        int64_t ab = p.orow[u], ae = p.orow[u + 1], bb = p.orow[v], be = p.orow[v + 1];
        if (ae - ab > be - bb) {
            int64_t t0 = ab, t1 = ae;
            ab = bb; ae = be; bb = t0; be = t1;
        }
        const int la = int(ae - ab), lb = int(be - bb);
        if (lane == 0) bytes += 4 + 8 + 32 + 4ull * la + 4ull * (lb < la ? lb : la) * 4;
        d = 0;
        for (int c = 0; c < la; c += 32) {
            const int i = c + lane;
            const int32_t x = i < la ? p.ocol[ab + i] : 0;
            bool f = i < la && gl_contains(p.ocol + bb, lb, x);
            if (w3 >= 0 && f)  // triple (v,u,w): also an out-neighbour of w
                f = gl_contains(p.ocol + p.orow[w3], int(p.orow[w3 + 1] - p.orow[w3]), x);
            const unsigned m = __ballot_sync(kct::FULL, f);
            const int at = d + __popc(m & ((1u << lane) - 1u));
            if (f && at < kWarpD) l2g[at] = x;
            d += __popc(m);
        }
    }
    __syncwarp();
    if (d > kWarpD) return d;  // caller defers the task to the CTA kernel
    if (!need_rows || d == 0) return d;
    warp_rows(p, l2g, d, rows, directed, bytes, SS);
    return d;
}

// register budget: the pivot walk keeps up to 128 registers (4 CTAs per SM,
// the shared-memory limit anyway); the orientation walk 56 (9 CTAs per SM)
template <int BLOCK, int MODE, bool GQ, int G = 32>
__global__ void __launch_bounds__(BLOCK, MODE == 1 ? 4 : 9) k_count_warp(CountParams p) {
    constexpr int NW = BLOCK / 32;
    constexpr int D = kWarpD, WPL = 1;
    constexpr int RSD = (D / 32) | 1;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ ull s_red[4 * NW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int hist_cells = MODE == MODE_PIVOT ? kct::kLeafCells : 0;
    const int node_words = MODE == MODE_PIVOT ? 2 * kct::kNodeCap : 0;
    // per warp: l2g[D] rows[D*RSD] list[D] S0[32] P0[32] cbuf[32] small leafhist
    // node stack frames
    const int per_warp = D + D * RSD + D + 32 * 3 + kct::kSmallWords + hist_cells + node_words +
                         p.nsm_frames * p.fw;
    uint32_t *base = reinterpret_cast<uint32_t *>(smem) + warp * per_warp;
    int32_t *l2g = reinterpret_cast<int32_t *>(base);
    uint32_t *rows = base + D;
    int *list = reinterpret_cast<int *>(rows + D * RSD);
    uint32_t *S0 = reinterpret_cast<uint32_t *>(list + D);
    uint32_t *P0 = S0 + 32;
    uint32_t *cbuf = P0 + 32;
    kct::SmallScratch SS;
    SS.srow = cbuf + 32;
    SS.sstk = SS.srow + 32;
    uint32_t *whist = SS.srow + kct::kSmallWords;
    if (MODE == MODE_PIVOT) {  // per-lane S-tier walks (kct::pivot_lanes)
        SS.nstk = reinterpret_cast<uint2 *>(whist + hist_cells);
        SS.ncap = kct::kNodeCap;
    }
    kct::Frames F;
    F.sm = whist + hist_cells + node_words;
    F.nsm = p.nsm_frames;
    F.fw = p.fw;
    F.gm = p.frames_global ? p.frames_global + (int64_t(blockIdx.x) * NW + warp) * p.frames_slot
                           : nullptr;
    __shared__ int s_hc[4 * NW];
    kct::PivotLeafSink sink;
    sink.whist = whist;
    sink.g_hist = p.hist;
    sink.L = p.hist_dim;
    __shared__ kct::GQueue s_gq;  // (see k_count: no address of a kernel parameter)
    __shared__ kct::Spill s_sp;
    if (tid == 0) {
        s_gq = p.gq;
        s_sp = p.spill;
    }
    __syncthreads();
    sink.gq = (GQ && MODE == MODE_PIVOT) ? &s_gq : nullptr;  // compile-time off when !GQ
    sink.eager = false;
    sink.l2g = l2g;
    sink.hc = s_hc + 4 * warp;
    if (MODE == MODE_PIVOT && p.use_spill) sink.sp = &s_sp;
    sink.push_min = p.gq_push_min;
    sink.cooldown = p.gq_cooldown;
    sink.room_min = p.gq_room;
    for (int i = lane; i < hist_cells; i += 32) whist[i] = 0;
    if (lane == 0) {
        sink.hc[0] = 0;
        sink.hc[1] = 0;
        if (sink.gq) atomicAdd(p.gq.ctl + 3, 1);  // busy: this warp may push
    }
    __syncwarp();

    ull acc = 0, visits = 0, tasks = 0, work = 0, bytes = 0;
    const int t = p.t;
    const bool allk = MODE == MODE_PIVOT && p.all_k;
    for (;;) {
        ull i = 0;
        if (lane == 0) i = atomicAdd(p.task_counter, 1ull);
        i = __shfl_sync(kct::FULL, i, 0);
        if (i >= ull(p.n_tasks)) break;
        if (sink.sp) sink.set_budget(p.spill_budget, lane);
        if (MODE == MODE_PIVOT && p.in_buf) {
            // spill round: walk item i (a node inside a counted task -- no
            // task, no visit of its own; engine_pivot.py:117-233 from there)
            const uint32_t *it = p.in_buf + p.in_off[i];
            const uint32_t kind = __ldg(it), n = __ldg(it + 1);
            if (kind == 2u) {  // S-tier universe + pending nodes
                SS.srow[lane] = __ldg(it + 4 + lane);
                for (int j = lane; j < int(n); j += 32)
                    SS.nstk[j] = make_uint2(__ldg(it + 36 + 2 * j), __ldg(it + 37 + 2 * j));
                __syncwarp();
                kct::pivot_lanes_run(SS.srow, int(n), t, allk, SS.nstk, SS.ncap, sink, lane,
                                     visits, work);
            } else {  // global ids of the set: rebuild its undirected sub-graph
                const int s0 = int(__ldg(it + 2)), npv0 = int(__ldg(it + 3));
                for (int j = lane; j < int(n); j += 32) l2g[j] = int32_t(__ldg(it + 4 + j));
                __syncwarp();
                warp_rows(p, l2g, int(n), rows, false, bytes, SS);
                const int W = (int(n) + 31) >> 5, RS = row_stride(W);
                const ull wt0 = work;
                if (W == 1) {
                    const uint32_t all = n >= 32 ? kct::FULL : ((1u << n) - 1u);
                    kct::pivot_lanes(rows, all, s0, npv0, t, allk, SS.nstk, SS.ncap, sink, lane,
                                     visits, work);
                } else {
                    kct::Set<WPL> A;
                    const int lo = lane << 5;
                    A.w[0] = lo >= int(n) ? 0u
                                          : (lo + 32 <= int(n) ? kct::FULL
                                                               : ((1u << (int(n) - lo)) - 1u));
                    kct::pivot_from<WPL>(rows, RS, W, t, allk, A, s0, npv0, F, list, SS, sink,
                                         nullptr, visits, work);
                }
                work = wt0 + (work - wt0) * ull(W);
            }
            __syncwarp();
            continue;
        }
        const int32_t task = p.tasks[i];
        const bool need_rows = MODE == MODE_PIVOT || t >= 2;
        const long long pc0 = (p.prof && lane == 0) ? clock64() : 0;
        const int d = warp_build(p, task, l2g, rows, need_rows, MODE == MODE_ORIENT, bytes, SS,
                                 p.task_w && !p.branch ? p.task_w[i] : -1);
        if (p.prof && lane == 0) {
            atomicAdd(&p.prof[kProfWarpBuild], ull(clock64() - pc0));
            if (d > D) atomicAdd(&p.prof[kProfOvfHist + min((d - 1) >> 5, 63)], 1ull);
        }
        const long long pc1 = (p.prof && lane == 0) ? clock64() : 0;
        if (d > D) {  // edge task larger than the warp tier: CTA kernel, next launch
            if (lane == 0) {
                const ull at = atomicAdd(p.overflow_n, 1ull);
                atomicMax(p.overflow_n + 6, ull(d));  // sizes the CTA launch (dcap)
                p.overflow[at] = task;
                if (p.task_w) p.overflow_w[at] = p.task_w[i];
            }
            continue;
        }
        if (p.split) {
            if (lane == 0) ++visits;  // see k_count
            if (d == 0) continue;
        } else if (allk) {
            if (d == 0) continue;
        } else if (d < t) {
            continue;
        }
        if (lane == 0 && !p.branch) ++tasks;  // a branch task is part of a counted task
        if (t <= 1 && !allk) {
            if (lane == 0) acc += t == 0 ? 1ull : ull(d);
            continue;
        }
        const int W = (d + 31) >> 5, RS = warp_row_stride(W, MODE == MODE_ORIENT);
        const uint32_t all = d >= 32 ? kct::FULL : ((1u << d) - 1u);
        const ull wt0 = work;  // units -> §8(d) word-ops of this task at the end
        if (MODE == MODE_ORIENT) {
            const int last = t - 2;
            if (last == 0) {
                for (int u = lane; u < d; u += 32) {
                    const uint32_t *ru = rows + u * RS;
                    int c = 0;
                    for (int w = 0; w < W; ++w) c += __popc(ru[w]);
                    acc += ull(c);
                    ++visits;
                    work += 1;
                }
            } else if (W == 1) {
                kct::orient_small<G>(rows, all, 0, last, SS.sstk, lane, acc, visits, work);
            } else {
                for (int u = 0; u < d; ++u) {
                    if (lane == 0) {
                        ++visits;
                        work += 1;
                    }
                    kct::orient_subtree<WPL, G>(rows, RS, W, last, u, F, list, cbuf, SS, acc, visits,
                                             work);
                }
            }
        } else {
            if (p.roots_only || p.branch) {
                // split pivot task (engine_pivot.py:133-136 root frame): the
                // roots pass stores S0's pivot and branch set P0; every
                // branch v of P0 is then walked as its own task (rebuilding
                // the task's bit matrix), spreading big trees over the GPU
                kct::Set<WPL> A;
                {
                    const int lo = lane << 5;
                    A.w[0] = lo >= d ? 0u : (lo + 32 <= d ? kct::FULL : ((1u << (d - lo)) - 1u));
                }
                if (p.roots_only) {
                    const int piv0 = kct::select_pivot<WPL>(rows, RS, A, list, lane, work, W);
                    const uint32_t rp = lane < W ? rows[piv0 * RS + lane] : 0u;
                    const uint32_t P = A.w[0] & ~rp;
                    if (lane < 4) p.root_P[4 * i + lane] = P;
                    const int c = kct::warp_count<WPL>(kct::Set<WPL>{{P}});
                    if (lane == 0) {
                        p.root_piv[i] = piv0;
                        p.root_cnt[i] = c;
                    }
                } else {
                    const int si = p.branch_si[i];
                    S0[lane] = A.w[0];
                    P0[lane] = lane < 4 ? p.root_P[4 * si + lane] : 0u;
                    __syncwarp();
                    kct::pivot_subtree<WPL>(rows, RS, W, t, allk, p.task_w[i], p.root_piv[si], S0,
                                            P0, F, list, SS, sink, visits, work);
                }
            } else if (W == 1) {
                kct::pivot_lanes(rows, all, 0, 0, t, allk, SS.nstk, SS.ncap, sink, lane, visits,
                                 work);
            } else {
                // root frame: S0 = all locals, pivot = argmax |row c| (lowest id on ties)
                kct::Set<WPL> A;
                {
                    const int lo = lane << 5;
                    A.w[0] = lo >= d ? 0u : (lo + 32 <= d ? kct::FULL : ((1u << (d - lo)) - 1u));
                }
                const int piv0 = kct::select_pivot<WPL>(rows, RS, A, list, lane, work, W);
                const uint32_t rp = lane < W ? rows[piv0 * RS + lane] : 0u;
                S0[lane] = A.w[0];
                P0[lane] = A.w[0] & ~rp;
                __syncwarp();
                for (int v = 0; v < d; ++v) {
                    if (!((P0[v >> 5] >> (v & 31)) & 1u)) continue;
                    kct::pivot_subtree<WPL>(rows, RS, W, t, allk, v, piv0, S0, P0, F, list, SS,
                                            sink, visits, work);
                }
            }
        }
        work = wt0 + (work - wt0) * ull(W);
        if (p.prof && lane == 0) atomicAdd(&p.prof[kProfWarpWalk], ull(clock64() - pc1));
        __syncwarp();
    }
    if (GQ && MODE == MODE_PIVOT) {
        // task queue drained: serve subtrees handed over by busy warps
        const kct::GQueue &q = s_gq;
        if (lane == 0) {  // busy -> hungry (atomics only: no lock storm at the tail)
            atomicAdd(q.ctl + 2, 1);
            atomicSub(q.ctl + 3, 1);
        }
        for (;;) {
            int slot = -1, done = 0;
            const long long pq0 = (p.prof && lane == 0) ? clock64() : 0;
            if (lane == 0) {
                // Poll without the lock; take it with a single try (no
                // spinning on it: a pusher must never queue behind hundreds
                // of hungry warps); exponential back-off between polls.
                const unsigned jitter = (blockIdx.x * 7 + warp * 13) & 127;
                unsigned backoff = 128;
                const unsigned long long t_start = kc_globaltimer();
                for (;;) {
                    const int sz = q.vol(1);
                    if (sz > 0) {
                        if (atomicCAS(q.ctl, 0, 1) == 0) {  // single try, never spin on it
                            __threadfence();
                            const int sz2 = q.vol(1);
                            if (sz2 > 0) {
                                slot = sz2 - 1;  // lock kept while the item is copied out
                                atomicSub(q.ctl + 2, 1);
                                atomicAdd(q.ctl + 3, 1);
                                break;
                            }
                            q.release();
                        }
                    } else if (q.vol(6)) {
                        // closed: nothing can be pushed any more, leave without the lock
                        atomicSub(q.ctl + 2, 1);
                        done = 1;
                        break;
                    } else if (q.vol(3) == 0) {
                        // nobody busy: the first warp to see it under the lock closes
                        // the queue (pushers refuse once closed), everyone else leaves
                        if (atomicCAS(q.ctl, 0, 1) == 0) {
                            __threadfence();
                            if (q.vol(1) == 0 && q.vol(3) == 0) q.set(6, 1);
                            q.release();
                        }
                    } else if (kc_globaltimer() - t_start > 20000000ull) {  // 20 ms idle
                        // give the SM back.  Under the lock: an item a pusher
                        // published since the poll above is taken, not left
                        // behind; otherwise `hungry` drops before any later
                        // pusher's check (reserve() re-reads it under the
                        // lock), so no item can be stranded
                        q.acquire();
                        const int sz2 = q.vol(1);
                        if (sz2 > 0) {
                            slot = sz2 - 1;  // lock kept while the item is copied out
                            atomicSub(q.ctl + 2, 1);
                            atomicAdd(q.ctl + 3, 1);
                            break;
                        }
                        atomicSub(q.ctl + 2, 1);
                        q.release();
                        done = 1;
                        break;
                    }
                    __nanosleep(backoff + jitter);
                    backoff = backoff < 8192 ? 2 * backoff : backoff;  // exponential back-off
                }
            }
            slot = __shfl_sync(kct::FULL, slot, 0);
            done = __shfl_sync(kct::FULL, done, 0);
            const long long pq1 = (p.prof && lane == 0) ? clock64() : 0;
            if (p.prof && lane == 0) atomicAdd(&p.prof[kProfGqIdle], ull(pq1 - pq0));
            if (done) break;
            // L2-coherent loads (__ldcg): this SM's L1 may hold an older item
            // of the same slot
            const uint32_t *it = q.items + int64_t(slot) * kct::kGItemWords;
            const uint32_t h0 = __ldcg(it);
            const int s0 = int(__ldcg(it + 1)), npv = int(__ldcg(it + 2));
            const uint32_t kind = __ldcg(it + 3);
            const int n = int(h0);
            if (kind == 1u) SS.srow[lane] = __ldcg(it + 4 + lane);
            else
                for (int i = lane; i < n; i += 32) l2g[i] = int32_t(__ldcg(it + 4 + i));
            __syncwarp();
            if (lane == 0) {
                q.set(1, slot);
                atomicAdd(q.ctl + 5, 1);  // pops (diagnostics)
                q.release();
            }
            if (p.prof && lane == 0) atomicAdd(&p.prof[kProfGqItems + (kind == 1u)], 1ull);
            if (kind == 1u) {  // compressed S-tier subtree: no rebuild
                kct::pivot_lanes(SS.srow, h0, s0, npv, t, allk, SS.nstk, SS.ncap, sink, lane,
                                 visits, work);
                if (p.prof && lane == 0) atomicAdd(&p.prof[kProfGqWalk], ull(clock64() - pq1));
                if (lane == 0) {
                    atomicAdd(q.ctl + 2, 1);
                    atomicSub(q.ctl + 3, 1);
                }
                __syncwarp();
                continue;
            }
            // the subtree of X depends only on the sub-graph induced by X
            warp_rows(p, l2g, n, rows, false, bytes, SS);
            const int W = (n + 31) >> 5, RS = row_stride(W);
            const ull wt0 = work;
            if (W == 1) {
                const uint32_t all = n >= 32 ? kct::FULL : ((1u << n) - 1u);
                kct::pivot_lanes(rows, all, s0, npv, t, allk, SS.nstk, SS.ncap, sink, lane, visits,
                                 work);
            } else {
                kct::Set<WPL> A;
                {
                    const int lo = lane << 5;
                    A.w[0] = lo >= n ? 0u : (lo + 32 <= n ? kct::FULL : ((1u << (n - lo)) - 1u));
                }
                kct::pivot_from<WPL>(rows, RS, W, t, allk, A, s0, npv, F, list, SS, sink, nullptr,
                                     visits, work);
            }
            work = wt0 + (work - wt0) * ull(W);
            if (p.prof && lane == 0) atomicAdd(&p.prof[kProfGqWalk], ull(clock64() - pq1));
            if (lane == 0) {
                atomicAdd(q.ctl + 2, 1);
                atomicSub(q.ctl + 3, 1);
            }
            __syncwarp();
        }
    }
    if (MODE == MODE_PIVOT) sink.flush(lane);
    __syncthreads();
    flush_block<BLOCK>(p, acc, visits, tasks, work, bytes, s_red);
}

// ---------------------------------------------------------------------------
// task lists
// ---------------------------------------------------------------------------
__global__ void k_vertex_flags(const int64_t *__restrict__ orow, int64_t n, int32_t *__restrict__ f) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x)
        f[v] = orow[v + 1] - orow[v] > 0 ? 1 : 0;
}

// keep vertex v if its make_tasks index is in [lo, hi) and out-degree >= min_d;
// key = out-degree (descending sort => largest first)
__global__ void k_vertex_select(const int64_t *__restrict__ orow, const int32_t *__restrict__ pos,
                                int64_t n, int64_t lo, int64_t hi, int min_d,
                                uint8_t *__restrict__ keep, uint32_t *__restrict__ key) {
    for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
         v += int64_t(gridDim.x) * blockDim.x) {
        int64_t d = orow[v + 1] - orow[v];
        keep[v] = d > 0 && d >= min_d && pos[v] >= lo && pos[v] < hi;
        key[v] = uint32_t(d);
    }
}

__global__ void k_edge_select(const int64_t *__restrict__ orow, const int32_t *__restrict__ ocoo,
                              const int32_t *__restrict__ ocol, int64_t m, int64_t lo, int64_t hi,
                              int min_d, const uint8_t *__restrict__ vsel,
                              const int32_t *__restrict__ esize, uint8_t *__restrict__ keep,
                              uint32_t *__restrict__ key) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
         e += int64_t(gridDim.x) * blockDim.x) {
        int32_t u = ocoo[e], v = ocol[e];
        int64_t du = orow[u + 1] - orow[u], dv = orow[v + 1] - orow[v];
        // exact |N+(u) n N+(v)| when known, else its bound min(du, dv)
        int64_t b = esize ? int64_t(esize[e]) : (du < dv ? du : dv);
        keep[e] = e >= lo && e < hi && b >= min_d && (!vsel || vsel[u]);
        key[e] = uint32_t(b);  // bound on the task's locals: routes it to the warp/CTA kernel
    }
}

// sorted-descending keys: number of keys > thr (first index with key <= thr)
__global__ void k_split_point(const uint32_t *__restrict__ keys, int64_t n, uint32_t thr,
                              int32_t *__restrict__ out) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] > thr) lo = mid + 1;
        else hi = mid;
    }
    *out = int32_t(lo);
}

// exact edge-task sizes |N+(u) n N+(v)| (bitgraph.py:67-86 locals count):
// warp per edge, lanes over the shorter out-list, binary search in the longer
__global__ void k_edge_sizes(const int64_t *__restrict__ orow, const int32_t *__restrict__ ocol,
                             const int32_t *__restrict__ ocoo, int64_t m,
                             int32_t *__restrict__ esize) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t e = warp; e < m; e += nwarps) {
        const int32_t u = ocoo[e], v = ocol[e];
        int64_t ab = orow[u], ae = orow[u + 1], bb = orow[v], be = orow[v + 1];
        if (ae - ab > be - bb) {
            int64_t t0 = ab, t1 = ae;
            ab = bb; ae = be; bb = t0; be = t1;
        }
        const int la = int(ae - ab), lb = int(be - bb);
        int c = 0;
        for (int i = lane; i < la; i += 32) c += gl_contains(ocol + bb, lb, ocol[ab + i]) ? 1 : 0;
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) esize[e] = c;
    }
}

__global__ void k_gather_sizes(const int32_t *__restrict__ items, int64_t n,
                               const int32_t *__restrict__ esize, int32_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        out[i] = esize[items[i]];
}

// triples (e, w) for every w in N+(u) n N+(v) of each big edge item e = (u,v):
// the level-1 subtrees of the item's tree (warp per item, ascending w)
__global__ void k_make_triples(const int64_t *__restrict__ orow, const int32_t *__restrict__ ocol,
                               const int32_t *__restrict__ ocoo, const int32_t *__restrict__ items,
                               int64_t n, const int32_t *__restrict__ offs,
                               int32_t *__restrict__ tri_e, int32_t *__restrict__ tri_w) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t it = warp; it < n; it += nwarps) {
        const int32_t e = items[it];
        const int32_t u = ocoo[e], v = ocol[e];
        int64_t ab = orow[u], ae = orow[u + 1], bb = orow[v], be = orow[v + 1];
        if (ae - ab > be - bb) {
            int64_t t0 = ab, t1 = ae;
            ab = bb; ae = be; bb = t0; be = t1;
        }
        const int la = int(ae - ab), lb = int(be - bb);
        int at = offs[it];
        for (int c = 0; c < la; c += 32) {
            const int i = c + lane;
            const int32_t x = i < la ? ocol[ab + i] : 0;
            const bool f = i < la && gl_contains(ocol + bb, lb, x);
            const unsigned m = __ballot_sync(0xffffffffu, f);
            if (f) {
                const int k = at + __popc(m & ((1u << lane) - 1u));
                tri_e[k] = e;
                tri_w[k] = x;
            }
            at += __popc(m);
        }
    }
}

// branch tasks of the split pivot tasks: (task, v) for every v of P0, in
// task order (the biggest tasks' branches first)
__global__ void k_branch_list(const int32_t *__restrict__ cnt, const int32_t *__restrict__ off,
                              const uint32_t *__restrict__ rootP, int64_t n,
                              const int32_t *__restrict__ tasks, int32_t *__restrict__ btask,
                              int32_t *__restrict__ bv, int32_t *__restrict__ bsi) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        if (!cnt[i]) continue;
        int at = off[i];
        for (int w = 0; w < 4; ++w) {
            uint32_t m = rootP[4 * i + w];
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1u;
                btask[at] = tasks[i];
                bv[at] = (w << 5) + b;
                bsi[at] = int32_t(i);
                ++at;
            }
        }
    }
}

__global__ void k_mark_roots(const int32_t *__restrict__ roots, int64_t n,
                             uint8_t *__restrict__ vsel) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        vsel[roots[i]] = 1;
}

__global__ void k_iota(int32_t *__restrict__ a, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        a[i] = int32_t(i);
}

inline int grid_1d(int64_t n, int sms) {
    int64_t b = (n + 255) / 256;
    if (b > int64_t(sms) * 16) b = int64_t(sms) * 16;
    return int(b < 1 ? 1 : b);
}

// stream of the current library call: DevBuf allocations are stream-ordered on it
thread_local cudaStream_t tl_stream = nullptr;
thread_local int tl_launches = 0;  // counting-kernel launches of the current call
// KC_TIMING=1: device time of every counting launch (events on its stream),
// printed to stderr at the end of kc_count -- a launch list without ncu
struct LaunchTimer {
    const char *what;
    int64_t n_tasks;
    int grid;
    cudaEvent_t a, b;
};
thread_local std::vector<LaunchTimer> tl_timers;
inline bool timing_on() {
    static const bool on = [] {
        const char *e = getenv("KC_TIMING");
        return e && e[0] == '1';
    }();
    return on;
}
inline cudaEvent_t timer_begin(cudaStream_t s) {
    if (!timing_on()) return nullptr;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    return e;
}
inline void timer_end(cudaEvent_t a, cudaStream_t s, const char *what, int64_t n, int grid) {
    if (!a) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    tl_timers.push_back({what, n, grid, a, e});
}
struct StreamScope {
    cudaStream_t prev;
    explicit StreamScope(cudaStream_t s) : prev(tl_stream) { tl_stream = s; }
    ~StreamScope() { tl_stream = prev; }
};

struct DevBuf {
    void *p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    explicit DevBuf(size_t bytes) : s(tl_stream) { p = kc_alloc<uint8_t>(bytes, s); }
    // stream-ordered on `st`: the buffer of a kernel launched on st (freed on st)
    DevBuf(size_t bytes, cudaStream_t st) : s(st) { p = kc_alloc<uint8_t>(bytes, s); }
    ~DevBuf() { kc_free(p, s); }
    template <typename T>
    T *as() const {
        return reinterpret_cast<T *>(p);
    }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
};

// Builds the device task list: ids of the tasks in [lo, hi) of make_tasks
// order with enough locals, sorted by descending cost (largest first keeps the
// persistent queue balanced).  Returns the count.
int64_t build_tasks(kc_graph *g, int scheme, int64_t lo, int64_t hi, int min_d, DevBuf &out,
                    uint32_t big_thr, int64_t *n_big, const uint8_t *vsel = nullptr,
                    uint32_t mid_thr = 0, int64_t *n_mid = nullptr, uint32_t *max_key = nullptr) {
    if (n_mid) *n_mid = 0;
    if (max_key) *max_key = 0;
    const int64_t N = scheme == KC_SCHEME_EDGE ? g->m_dir : g->n;
    *n_big = 0;
    if (N == 0) return 0;
    DevBuf keep(N), key(4 * N), key2(4 * N), ids(4 * N), ids2(4 * N), cnt(16);
    if (scheme == KC_SCHEME_VERTEX) {
        DevBuf flag(4 * N), pos(4 * N);
        k_vertex_flags<<<grid_1d(N, g->num_sms), 256, 0, g->stream>>>(g->orow_ptr, N,
                                                                       flag.as<int32_t>());
        size_t bytes = 0;
        KC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flag.as<int32_t>(),
                                              pos.as<int32_t>(), int(N), g->stream));
        void *tmp = kc_tmp(g, bytes);
        KC_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, flag.as<int32_t>(), pos.as<int32_t>(),
                                              int(N), g->stream));
        k_vertex_select<<<grid_1d(N, g->num_sms), 256, 0, g->stream>>>(
            g->orow_ptr, pos.as<int32_t>(), N, lo, hi, min_d, keep.as<uint8_t>(),
            key.as<uint32_t>());
    } else {
        k_edge_select<<<grid_1d(N, g->num_sms), 256, 0, g->stream>>>(
            g->orow_ptr, g->ocoo, g->ocol, N, lo, hi, min_d, vsel, g->esize, keep.as<uint8_t>(),
            key.as<uint32_t>());
    }
    k_iota<<<grid_1d(N, g->num_sms), 256, 0, g->stream>>>(ids.as<int32_t>(), N);
    KC_CUDA(cudaGetLastError());
    // compact (ids, keys) by keep
    size_t bytes = 0;
    KC_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, ids.as<int32_t>(), keep.as<uint8_t>(),
                                       ids2.as<int32_t>(), cnt.as<int32_t>(), int(N), g->stream));
    void *tmp = kc_tmp(g, bytes);
    KC_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, ids.as<int32_t>(), keep.as<uint8_t>(),
                                       ids2.as<int32_t>(), cnt.as<int32_t>(), int(N), g->stream));
    KC_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, key.as<uint32_t>(), keep.as<uint8_t>(),
                                       key2.as<uint32_t>(), cnt.as<int32_t>(), int(N), g->stream));
    int32_t h = 0;
    KC_CUDA(cudaMemcpyAsync(&h, cnt.p, 4, cudaMemcpyDeviceToHost, g->stream));
    KC_CUDA(cudaStreamSynchronize(g->stream));
    const int64_t n_sel = h;
    out.~DevBuf();
    new (&out) DevBuf(4 * (n_sel > 0 ? n_sel : 1));
    if (n_sel > 0) {
        bytes = 0;
        KC_CUDA(cub::DeviceRadixSort::SortPairsDescending(
            nullptr, bytes, key2.as<uint32_t>(), key.as<uint32_t>(), ids2.as<int32_t>(),
            out.as<int32_t>(), int(n_sel), 0, 32, g->stream));
        tmp = kc_tmp(g, bytes);
        KC_CUDA(cub::DeviceRadixSort::SortPairsDescending(
            tmp, bytes, key2.as<uint32_t>(), key.as<uint32_t>(), ids2.as<int32_t>(),
            out.as<int32_t>(), int(n_sel), 0, 32, g->stream));
        k_split_point<<<1, 1, 0, g->stream>>>(key.as<uint32_t>(), n_sel, big_thr,
                                              cnt.as<int32_t>() + 1);
        if (n_mid)
            k_split_point<<<1, 1, 0, g->stream>>>(key.as<uint32_t>(), n_sel, mid_thr,
                                                  cnt.as<int32_t>() + 2);
        int32_t nb[2] = {0, 0};
        KC_CUDA(cudaMemcpyAsync(nb, cnt.as<int32_t>() + 1, 8, cudaMemcpyDeviceToHost,
                                g->stream));
        if (max_key)  // keys sorted descending: the largest task's locals (bound)
            KC_CUDA(cudaMemcpyAsync(max_key, key.p, 4, cudaMemcpyDeviceToHost, g->stream));
        KC_CUDA(cudaStreamSynchronize(g->stream));
        *n_big = nb[0];
        if (n_mid) *n_mid = nb[1];
    }
    return n_sel;
}

constexpr int kBlock = 128;
constexpr int kSmidSlots = 1024;  // %smid can exceed the SM count
// kc_do_count's counter block `outs` (u64 words): [0] task counter, [1..4]
// limbs, [5] visits, [6] tasks run, [7] warp-tier counter, [8, 8+kSmidSlots)
// visits per SM, then word_ops, extract bytes, four more task counters and
// the overflow count, then the subtree queue's control words (8 ints)
constexpr int kOutGq = 8 + kSmidSlots + 12;
constexpr int kOutWords = kOutGq + 4;
constexpr int kSmemMax = 225 * 1024;  // of 227 KB per block (static smem < 2 KB)
constexpr int kSmemTarget = 100 * 1024;  // aim for >= 2 resident CTAs per SM

// DFS frames a warp can touch: orient frames 1..t-3 (frame t-2 is scored in
// registers), pivot frames 1..d (+1 guard)
int frames_needed(int mode, int t, int dcap) {
    if (mode == MODE_ORIENT) return std::max(1, std::min(t - 2, dcap + 1));
    return dcap + 2;
}

typedef std::vector<std::unique_ptr<DevBuf>> Keep;

// Buffers of a kernel are allocated stream-ordered on the stream it is
// launched on (DevBuf(bytes, stream)), so a kernel on the aux stream never
// waits for, nor races with, the graph stream's allocations and frees.

// shared-memory plan of the CTA-tier kernel for one block size
struct CtaPlan {
    size_t smem = 0;
    int nsm = 0, rows_in_smem = 0, per_sm = 0;
    const void *kern = nullptr;
};

template <int MODE, int WPL, int BLOCK>
CtaPlan plan_cta(const CountParams &p) {
    constexpr int NW = BLOCK / 32;
    CtaPlan pl;
    const size_t hist_words = MODE == MODE_PIVOT ? kct::kLeafCells : 0;
    const size_t dpad = size_t((p.dcap + 3) & ~3);
    const size_t l2g_bytes = 4 * dpad;
    const size_t rows_words = (size_t(p.dcap) * row_stride(p.wcap) + 3) & ~size_t(3);
    const int need = frames_needed(MODE, p.t, p.dcap);
    auto area_words = [&](int nsm) {
        size_t w = (MODE == MODE_PIVOT ? 64 * WPL + kStealCap * (32 * WPL + 4) : 0) +
                   size_t(NW) * (dpad + 32 * WPL + kCtaSmallWords + hist_words +
                                 (MODE == MODE_ORIENT && p.t >= 4 ? kct::mid_words(WPL, p.mid_max)
                                                                  : 0) +
                                 (MODE == MODE_PIVOT ? 2 * kct::kNodeCap : 0) +
                                 size_t(nsm) * p.fw);
        if (p.scheme == KC_SCHEME_EDGE) w = std::max(w, dpad);
        if (MODE != MODE_PIVOT) {
            size_t hs = 2;  // build_task's hash table: H >= 2 dcap slots, 1.5 words each
            while (hs < 2 * size_t(p.dcap)) hs <<= 1;
            w = std::max(w, hs + hs / 2);
        }
        return w;
    };
    // as many shared frames as fit the target budget (at least 4, at most need)
    int nsm = std::min(need, 64);
    auto total = [&](int ns, bool rows_smem) {
        return l2g_bytes + 4 * area_words(ns) + (rows_smem ? 4 * rows_words : 0) + 64;
    };
    pl.rows_in_smem = total(std::min(nsm, 4), true) <= size_t(kSmemMax);
    while (nsm > 4 && total(nsm, pl.rows_in_smem) > size_t(kSmemTarget)) nsm >>= 1;
    while (nsm > 1 && total(nsm, pl.rows_in_smem) > size_t(kSmemMax)) --nsm;
    pl.nsm = nsm;
    pl.smem = total(nsm, pl.rows_in_smem);
    if (pl.smem > size_t(kSmemMax)) return pl;  // per_sm = 0: not launchable
    auto kern = (MODE == MODE_PIVOT && p.use_gq) ? k_count<BLOCK, MODE, WPL, true>
                                                 : k_count<BLOCK, MODE, WPL, false>;
    KC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(pl.smem)));
    KC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pl.per_sm, kern, BLOCK, pl.smem));
    pl.kern = reinterpret_cast<const void *>(kern);
    return pl;
}

template <int MODE, int WPL, int BLOCK>
void launch_cta(kc_graph *g, CountParams &p, const CtaPlan &pl, int grid_override, Keep &keep,
                cudaStream_t stream) {
    constexpr int NW = BLOCK / 32;
    KC_REQUIRE(pl.smem <= size_t(kSmemMax), KC_ENOMEM, "per-task scratch exceeds shared memory");
    KC_REQUIRE(pl.per_sm > 0, KC_ECUDA, "count kernel cannot be resident");
    const size_t rows_words = (size_t(p.dcap) * row_stride(p.wcap) + 3) & ~size_t(3);
    const int need = frames_needed(MODE, p.t, p.dcap);
    p.rows_in_smem = pl.rows_in_smem;
    p.nsm_frames = pl.nsm;
    int grid = grid_override > 0 ? grid_override : pl.per_sm * g->num_sms;
    if (p.n_tasks > 0 && int64_t(grid) > p.n_tasks && !grid_override) grid = int(p.n_tasks);
    if (grid < 1) grid = 1;
    if (!p.rows_in_smem) {
        p.rows_slot = int64_t(rows_words);
        keep.emplace_back(new DevBuf(4 * rows_words * size_t(grid), stream));
        p.rows_global = keep.back()->as<uint32_t>();
    }
    p.frames_global = nullptr;
    p.frames_slot = 0;
    if (MODE != MODE_EXTRACT && need > pl.nsm) {
        p.frames_slot = int64_t(need - pl.nsm) * p.fw;
        keep.emplace_back(new DevBuf(4 * size_t(p.frames_slot) * size_t(grid) * NW, stream));
        p.frames_global = keep.back()->as<uint32_t>();
    }
    auto kern = (MODE == MODE_PIVOT && p.use_gq) ? k_count<BLOCK, MODE, WPL, true>
                                                 : k_count<BLOCK, MODE, WPL, false>;
    cudaEvent_t t0 = timer_begin(stream);
    kern<<<grid, BLOCK, pl.smem, stream>>>(p);
    KC_CUDA(cudaGetLastError());
    timer_end(t0, stream,
              MODE == MODE_PIVOT ? "cta/pivot"
                                 : (BLOCK == 128 ? "cta/orient" : BLOCK == 256 ? "cta/orient-256"
                                                                               : "cta/orient-512"),
              p.n_tasks, grid);
    ++tl_launches;
}

// CTA tier.  Orientation with one word per lane (d <= 1024): the block size
// (4, 8 or 16 warps sharing one task's bit matrix) that keeps the most warps
// resident per SM -- with big matrices (RMAT-22: 964 locals, 119 KB) a
// 4-warp CTA leaves the SM at one CTA, 4 warps.
template <int MODE, int WPL>
void launch_wpl(kc_graph *g, CountParams &p, int grid_override, Keep &keep,
                cudaStream_t stream) {
    p.fw = MODE == MODE_PIVOT ? 64 * WPL + 4 : 32 * WPL + 4;
    const CtaPlan p128 = plan_cta<MODE, WPL, 128>(p);
    if constexpr (MODE == MODE_ORIENT && WPL == 1) {
        if (grid_override <= 0 && p.n_tasks > int64_t(g->num_sms)) {
            const CtaPlan p256 = plan_cta<MODE, WPL, 256>(p);
            const CtaPlan p512 = plan_cta<MODE, WPL, 512>(p);
            const int w128 = p128.per_sm * 4, w256 = p256.per_sm * 8, w512 = p512.per_sm * 16;
            if (w512 > w256 && w512 > w128) {
                launch_cta<MODE, WPL, 512>(g, p, p512, grid_override, keep, stream);
                return;
            }
            if (w256 > w128) {
                launch_cta<MODE, WPL, 256>(g, p, p256, grid_override, keep, stream);
                return;
            }
        }
    }
    launch_cta<MODE, WPL, 128>(g, p, p128, grid_override, keep, stream);
}

// warp-per-task kernel for tasks with at most kWarpD locals
template <int MODE>
void launch_warp(kc_graph *g, CountParams &p, Keep &keep, cudaStream_t stream) {
    constexpr int NW = kBlock / 32;
    constexpr int D = kWarpD, RSD = (kWarpD / 32) | 1;
    const size_t hist_words = MODE == MODE_PIVOT ? kct::kLeafCells : 0;
    p.fw = MODE == MODE_PIVOT ? 64 + 4 : 32 + 4;
    const int need = std::max(1, std::min(frames_needed(MODE, p.t, D), D + 2));
    const size_t fixed = size_t(D) + D * RSD + D + 96 + kct::kSmallWords + hist_words +
                         (MODE == MODE_PIVOT ? 2 * kct::kNodeCap : 0);
    int nsm = std::min(need, 8);
    p.nsm_frames = nsm;
    const size_t smem = 4 * size_t(NW) * (fixed + size_t(nsm) * p.fw) + 64;
    auto kern = (MODE == MODE_PIVOT && p.use_gq) ? k_count_warp<kBlock, MODE, true>
                                                 : k_count_warp<kBlock, MODE, false>;
    if constexpr (MODE == MODE_ORIENT) {
        // orientation: sub-warp group size; the pivot
        // engine scores candidates one lane each (group size 1 in the
        // paper's terms, its favourable setting per PAPER.md:720)
        switch (p.group_size) {
            case 1: kern = k_count_warp<kBlock, MODE, false, 1>; break;
            case 2: kern = k_count_warp<kBlock, MODE, false, 2>; break;
            case 4: kern = k_count_warp<kBlock, MODE, false, 4>; break;
            case 8: kern = k_count_warp<kBlock, MODE, false, 8>; break;
            case 16: kern = k_count_warp<kBlock, MODE, false, 16>; break;
            default: kern = k_count_warp<kBlock, MODE, false, 32>; break;
        }
    }
    KC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    KC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem));
    KC_REQUIRE(per_sm > 0, KC_ECUDA, "warp count kernel cannot be resident");
    int grid = per_sm * g->num_sms;
    const int64_t want = (p.n_tasks + NW - 1) / NW;
    if (want < grid) grid = int(want < 1 ? 1 : want);
    p.frames_global = nullptr;
    p.frames_slot = 0;
    if (need > nsm) {
        p.frames_slot = int64_t(need - nsm) * p.fw;
        keep.emplace_back(new DevBuf(4 * size_t(p.frames_slot) * size_t(grid) * NW, stream));
        p.frames_global = keep.back()->as<uint32_t>();
    }
    cudaEvent_t t0 = timer_begin(stream);
    kern<<<grid, kBlock, smem, stream>>>(p);
    KC_CUDA(cudaGetLastError());
    timer_end(t0, stream,
              MODE == MODE_PIVOT ? (p.roots_only ? "warp/pivot-roots"
                                    : p.branch   ? "warp/pivot-branches"
                                                 : "warp/pivot")
                                 : (p.task_w ? "warp/orient-triples"
                                    : p.split ? "warp/orient-items"
                                              : "warp/orient"),
              p.n_tasks, grid);
    ++tl_launches;
}

template <int MODE>
void launch(kc_graph *g, CountParams &p, int grid_override, Keep &keep, cudaStream_t stream) {
    const int wpl = (p.wcap + 31) / 32;
    KC_REQUIRE(wpl <= 4, KC_EINVAL,
               "oriented max out-degree above 4096 locals is not supported by the bitmap engine");
    if (MODE == MODE_EXTRACT || wpl <= 1) launch_wpl<MODE, 1>(g, p, grid_override, keep, stream);
    else if (wpl == 2) launch_wpl<MODE, 2>(g, p, grid_override, keep, stream);
    else launch_wpl<MODE, 4>(g, p, grid_override, keep, stream);
}

// launch + wait (single-shot debug entry points)
template <int MODE>
void launch_sync(kc_graph *g, CountParams &p, int grid_override) {
    Keep keep;
    launch<MODE>(g, p, grid_override, keep, g->stream);
    KC_CUDA(cudaStreamSynchronize(g->stream));
}

}  // namespace

// Two item buffers for the pivot spill rounds (round r reads one, writes the
// other).  Capacities: 1G words (4 GB) and 16M items per list per buffer;
// a full buffer only makes walkers keep their work (kct::Spill).
constexpr int kSpillBudget = 1 << 16;  // branches per bounded walk (KC_SPILL_BUDGET)
struct SpillBufs {
    ull cap_words = 0;
    uint32_t cap_small = 0, cap_big = 0;
    std::unique_ptr<DevBuf> words[2], offs[2], ctls;
    void alloc(kc_graph *g) {
        size_t free_b = 0, total_b = 0;
        KC_CUDA(cudaMemGetInfo(&free_b, &total_b));
        cap_words = std::min<ull>(ull(1) << 30, ull(free_b / 8) / 4);  // <= 1/8 of free HBM
        cap_small = cap_big = 1u << 24;
        for (int i = 0; i < 2; ++i) {
            words[i].reset(new DevBuf(4 * size_t(cap_words), g->stream));
            offs[i].reset(new DevBuf(4 * (size_t(cap_small) + cap_big), g->stream));
        }
        ctls.reset(new DevBuf(2 * 8 * 8, g->stream));
        KC_CUDA(cudaMemsetAsync(ctls->p, 0, 2 * 8 * 8, g->stream));
    }
    ull *ctl(int i) const { return ctls->as<ull>() + 8 * i; }
    uint32_t *buf(int i) const { return words[i]->as<uint32_t>(); }
    uint32_t *small_off(int i) const { return offs[i]->as<uint32_t>(); }
    uint32_t *big_off(int i) const { return offs[i]->as<uint32_t>() + cap_small; }
    kct::Spill at(int i) const {
        kct::Spill sp;
        sp.buf = buf(i);
        sp.ctl = ctl(i);
        sp.small_off = small_off(i);
        sp.big_off = big_off(i);
        sp.cap_words = cap_words;
        sp.cap_small = cap_small;
        sp.cap_big = cap_big;
        sp.big_thr = kWarpD;
        return sp;
    }
};

// ---------------------------------------------------------------------------
void kc_do_count(kc_graph *g, const kc_count_args *a, kc_count_raw *raw, uint64_t *hist,
                 int64_t hist_cap, uint64_t *visits_per_sm, int32_t n_sm) {
    KC_REQUIRE(g->oriented, KC_EINVAL, "graph is not oriented (call kc_orient first)");
    KC_REQUIRE(a->k >= 3, KC_EINVAL, "kc_count needs k >= 3 (k = 1, 2 are closed forms)");
    KC_REQUIRE(a->algorithm == KC_ALGO_ORIENT || a->algorithm == KC_ALGO_PIVOT, KC_EINVAL,
               "unknown algorithm");
    KC_REQUIRE(a->scheme == KC_SCHEME_VERTEX || a->scheme == KC_SCHEME_EDGE, KC_EINVAL,
               "unknown scheme");
    KC_REQUIRE(!a->all_k || a->algorithm == KC_ALGO_PIVOT, KC_EINVAL,
               "all-k reporting requires the pivot algorithm");
    const int gs = a->group_size;
    KC_REQUIRE(gs == 0 || gs == 1 || gs == 2 || gs == 4 || gs == 8 || gs == 16 || gs == 32,
               KC_EINVAL, "group_size must be 0 (auto) or a power of two <= 32");
    const bool pivot = a->algorithm == KC_ALGO_PIVOT;
    const int t = a->scheme == KC_SCHEME_VERTEX ? a->k - 1 : a->k - 2;
    const int64_t L = pivot ? g->d_max + 2 : 0;
    memset(raw, 0, sizeof(*raw));
    raw->hist_dim = L;
    if (pivot) {
        KC_REQUIRE(hist && hist_cap >= L * L, KC_EINVAL, "histogram buffer too small");
        memset(hist, 0, sizeof(uint64_t) * size_t(L * L));
    }
    if (visits_per_sm) memset(visits_per_sm, 0, sizeof(uint64_t) * size_t(n_sm));
    kc_device_guard guard(g->device);
    StreamScope scope(g->stream);
    tl_launches = 0;
    tl_timers.clear();

    int64_t all = kc_task_count(g, a->scheme);
    int64_t lo = a->task_lo < 0 ? 0 : a->task_lo;
    int64_t hi = a->task_hi < 0 || a->task_hi > all ? all : a->task_hi;
    if (lo > hi) lo = hi;
    const int min_d = a->all_k ? 1 : (t > 1 ? t : 1);
    // Orientation, vertex scheme, t >= 4: roots with more than kSplitD locals
    // are split into their out-edge items (v,u) -- the level-1 subtrees of v's
    // tree -- so a hub's tree spreads over the whole GPU instead of one CTA.
    // Item (v,u) walks u's subtree over N+(v) n N+(u) with target t-1 (the
    // edge scheme's sub-graph) and counts u's own visit, so counts and
    // visits are exactly the vertex scheme's (engine_orient.py:32-79).
    const bool split = !pivot && a->scheme == KC_SCHEME_VERTEX && t >= 4;
    if ((split || a->scheme == KC_SCHEME_EDGE) && !g->esize && g->m_dir > 0) {
        g->esize = kc_alloc<int32_t>(g->m_dir, g->stream);
        k_edge_sizes<<<g->num_sms * 16, 256, 0, g->stream>>>(g->orow_ptr, g->ocol, g->ocoo,
                                                             g->m_dir, g->esize);
        KC_CUDA(cudaGetLastError());
    }
    DevBuf tasks;
    int64_t n_big = 0, n_mid = 0;
    uint32_t max_task_d = 0;  // largest task's locals (exact for vertex and edge keys)
    // pivot: warp-tier tasks above kPivotSplitD locals are split at the root
    static const int pivot_split_d = [] {
        const char *e = getenv("KC_PIVOT_SPLIT");
        return e && *e ? atoi(e) : kPivotSplitD;  // 0 / >= 128: off
    }();
    const bool psplit = pivot && (a->all_k || t >= 2) && pivot_split_d > 0 &&
                        pivot_split_d < kWarpD;
    const int64_t n_tasks =
        build_tasks(g, a->scheme, lo, hi, min_d, tasks, split ? kSplitD : kWarpD, &n_big, nullptr,
                    uint32_t(pivot_split_d), psplit ? &n_mid : nullptr, &max_task_d);
    const int64_t n_split = psplit ? std::max<int64_t>(n_mid - n_big, 0) : 0;
    DevBuf items;
    int64_t n_items = 0, n_items_big = 0;
    uint32_t max_item_d = 0;
    if (split && n_big > 0) {
        DevBuf vsel(size_t(g->n > 0 ? g->n : 1));
        KC_CUDA(cudaMemsetAsync(vsel.p, 0, size_t(g->n > 0 ? g->n : 1), g->stream));
        k_mark_roots<<<grid_1d(n_big, g->num_sms), 256, 0, g->stream>>>(tasks.as<int32_t>(), n_big,
                                                                        vsel.as<uint8_t>());
        KC_CUDA(cudaGetLastError());
        n_items = build_tasks(g, KC_SCHEME_EDGE, 0, g->m_dir, 0, items, kWarpD, &n_items_big,
                              vsel.as<uint8_t>(), 0, nullptr, &max_item_d);
    }

    DevBuf outs(8 * size_t(kOutWords));
    KC_CUDA(cudaMemsetAsync(outs.p, 0, 8 * size_t(kOutWords), g->stream));
    DevBuf dhist(L ? 8 * size_t(L * L) : 8);
    if (L) KC_CUDA(cudaMemsetAsync(dhist.p, 0, 8 * size_t(L * L), g->stream));

    CountParams p;
    memset(&p, 0, sizeof(p));
    p.orow = g->orow_ptr;
    p.ocol = g->ocol;
    p.ocoo = g->ocoo;
    p.tasks = tasks.as<int32_t>();
    p.n_tasks = n_tasks;
    p.scheme = a->scheme;
    p.t = t;
    p.all_k = a->all_k;
    p.dcap = int(std::max<int64_t>(g->d_max, 1));
    p.wcap = (p.dcap + 31) / 32;
    p.group_size = gs == 0 ? kAutoGroup : gs;
    p.hist_dim = int(L);
    p.hist = dhist.as<ull>();
    p.sh_hl = int(std::min<int64_t>(L, 48));
    ull *o = outs.as<ull>();
    p.task_counter = o;
    p.limbs = o + 1;
    p.visits_total = o + 5;
    p.tasks_run = o + 6;
    p.visits_per_sm = o + 8;
    p.word_ops = o + 8 + kSmidSlots;
    p.ext_bytes = o + 9 + kSmidSlots;
    DevBuf prof(timing_on() ? 8 * size_t(kProfWords) : 8);
    if (timing_on()) {
        KC_CUDA(cudaMemsetAsync(prof.p, 0, 8 * size_t(kProfWords), g->stream));
        p.prof = prof.as<ull>();
    }

    cudaEvent_t e0, e1, e_fork, e_join;
    KC_CUDA(cudaEventCreate(&e0));
    KC_CUDA(cudaEventCreate(&e1));
    KC_CUDA(cudaEventCreateWithFlags(&e_fork, cudaEventDisableTiming));
    KC_CUDA(cudaEventCreateWithFlags(&e_join, cudaEventDisableTiming));
    KC_CUDA(cudaEventRecord(e0, g->stream));
    DevBuf gq_items(pivot ? 4 * size_t(kGqCap) * kct::kGItemWords : 4);
    p.gq.items = gq_items.as<uint32_t>();
    // queue control words live in `outs` (zeroed above) so the final copy
    // brings them back with the counters: the host checks the queue drained
    p.gq.ctl = reinterpret_cast<int *>(o + kOutGq);
    p.gq.cap = kGqCap;
    // GPU-wide subtree hand-over for the pivot engine (KC_GQ=0 turns it off)
    static const bool gq_on = [] {
        const char *e = getenv("KC_GQ");
        return !(e && e[0] == '0');  // on unless KC_GQ=0
    }();
    p.use_gq = pivot && gq_on ? 1 : 0;
    auto env_int = [](const char *name, int dflt) {
        const char *e = getenv(name);
        return e && *e ? atoi(e) : dflt;
    };
    p.gq_push_min = env_int("KC_GQ_PUSHMIN", kct::kPushMin);
    p.gq_cooldown = env_int("KC_GQ_COOLDOWN", kct::kPushCooldown);
    p.gq_room = env_int("KC_GQ_ROOM", kct::kPushRoom);
    // Pivot bounded walks + spill rounds (KC_SPILL=0 turns them off and
    // leaves the subtree queue in charge of the balance)
    static const bool spill_on = [] {
        const char *e = getenv("KC_SPILL");
        return !(e && e[0] == '0');
    }();
    p.use_spill = pivot && spill_on ? 1 : 0;
    p.spill_budget = env_int("KC_SPILL_BUDGET", kSpillBudget);
    // 256: 8-word rows for 129..256-member pair levels (9 KB per warp);
    // 128: 2.3 KB per warp, more warps per SM, bigger sets uncompressed
    p.mid_max = env_int("KC_MID_MAX", 256) <= 128 ? 128 : 256;
    SpillBufs spb;
    if (p.use_spill) {
        spb.alloc(g);
        p.spill = spb.at(0);
        p.use_gq = 0;  // the spill rounds replace the subtree queue
    }
    Keep keep;
    // Edge tasks (and split items) all go to the warp-per-task kernel; the few
    // whose intersection exceeds kWarpD locals are appended to an overflow
    // list and run by the CTA-cooperative kernel afterwards.  Vertex tasks
    // are routed exactly by out-degree: big ones to the CTA kernel on the
    // graph stream, concurrently with the warp kernel on the aux stream.
    const bool edge_like = split || a->scheme == KC_SCHEME_EDGE;
    const int64_t n_tri_max = n_items_big * std::max<int64_t>(g->d_max, 1);  // triples bound
    DevBuf ovf(4 * size_t(std::max<int64_t>(split ? std::max(n_items, n_tri_max) : n_tasks, 1)));
    DevBuf ovf_w(4 * size_t(std::max<int64_t>(split ? std::max(n_items, n_tri_max) : 1, 1)));
    p.overflow = ovf.as<int32_t>();
    p.overflow_w = ovf_w.as<int32_t>();
    p.overflow_n = o + 8 + kSmidSlots + 3;
    if (!g->aux) KC_CUDA(cudaStreamCreateWithFlags(&g->aux, cudaStreamNonBlocking));
    KC_CUDA(cudaEventRecord(e_fork, g->stream));
    KC_CUDA(cudaStreamWaitEvent(g->aux, e_fork, 0));
    DevBuf tri_e, tri_w;
    int64_t n_tri = 0;
    if (split) {
        // items with more than kWarpD locals are split once more into triples
        // (v,u,w), w in N+(v) n N+(u): the level-1 subtrees of item (v,u),
        // walked with target t-2 after counting w's own visit; u's visit is
        // added on the host (raw->visits += n_items_big)
        // triples re-intersect their item's lists once per w: worth it only
        // for deep trees (t >= 6, i.e. k >= 7); shallower runs keep big
        // items in the CTA-cooperative kernel
        if (n_items_big > 0 && t < 6) {
            CountParams b = p;
            b.scheme = KC_SCHEME_EDGE;
            b.t = t - 1;
            b.split = 1;
            b.tasks = items.as<int32_t>();
            b.n_tasks = n_items_big;
            b.dcap = int(std::max<uint32_t>(std::min<uint32_t>(max_item_d, uint32_t(p.dcap)), 1u));
            b.wcap = (b.dcap + 31) / 32;
            b.task_counter = o + 8 + kSmidSlots + 6;
            launch<MODE_ORIENT>(g, b, 0, keep, g->stream);
        }
        if (n_items_big > 0 && t >= 6) {
            DevBuf sizes(4 * size_t(n_items_big)), offs(4 * size_t(n_items_big));
            k_gather_sizes<<<grid_1d(n_items_big, g->num_sms), 256, 0, g->stream>>>(
                items.as<int32_t>(), n_items_big, g->esize, sizes.as<int32_t>());
            size_t bytes = 0;
            KC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, sizes.as<int32_t>(),
                                                  offs.as<int32_t>(), int(n_items_big),
                                                  g->stream));
            void *tmp = kc_tmp(g, bytes);
            KC_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, sizes.as<int32_t>(),
                                                  offs.as<int32_t>(), int(n_items_big),
                                                  g->stream));
            int32_t last[2] = {0, 0};
            KC_CUDA(cudaMemcpyAsync(&last[0], offs.as<int32_t>() + n_items_big - 1, 4,
                                    cudaMemcpyDeviceToHost, g->stream));
            KC_CUDA(cudaMemcpyAsync(&last[1], sizes.as<int32_t>() + n_items_big - 1, 4,
                                    cudaMemcpyDeviceToHost, g->stream));
            KC_CUDA(cudaStreamSynchronize(g->stream));
            n_tri = int64_t(last[0]) + last[1];
            new (&tri_e) DevBuf(4 * size_t(std::max<int64_t>(n_tri, 1)));
            new (&tri_w) DevBuf(4 * size_t(std::max<int64_t>(n_tri, 1)));
            if (n_tri > 0) {
                k_make_triples<<<g->num_sms * 16, 256, 0, g->stream>>>(
                    g->orow_ptr, g->ocol, g->ocoo, items.as<int32_t>(), n_items_big,
                    offs.as<int32_t>(), tri_e.as<int32_t>(), tri_w.as<int32_t>());
                KC_CUDA(cudaGetLastError());
            }
        }
        if (n_tri > 0) {
            CountParams q = p;
            q.scheme = KC_SCHEME_EDGE;
            q.t = t - 2;
            q.split = 1;
            q.tasks = tri_e.as<int32_t>();
            q.task_w = tri_w.as<int32_t>();
            q.n_tasks = n_tri;
            q.task_counter = o + 8 + kSmidSlots + 5;
            launch_warp<MODE_ORIENT>(g, q, keep, g->stream);
        }
        if (n_items - n_items_big > 0) {
            CountParams q = p;
            q.scheme = KC_SCHEME_EDGE;
            q.t = t - 1;
            q.split = 1;
            q.tasks = items.as<int32_t>() + n_items_big;
            q.n_tasks = n_items - n_items_big;
            q.task_counter = o + 8 + kSmidSlots + 2;
            launch_warp<MODE_ORIENT>(g, q, keep, g->aux);
        }
        if (n_tasks - n_big > 0) {
            CountParams q = p;
            q.tasks = tasks.as<int32_t>() + n_big;
            q.n_tasks = n_tasks - n_big;
            launch_warp<MODE_ORIENT>(g, q, keep, g->aux);
        }
    } else {
        if (n_big > 0) {
            CountParams b = p;
            b.n_tasks = n_big;
            b.dcap = int(std::max<uint32_t>(std::min<uint32_t>(max_task_d, uint32_t(p.dcap)), 1u));
            b.wcap = (b.dcap + 31) / 32;
            if (pivot) launch<MODE_PIVOT>(g, b, 0, keep, g->stream);
            else launch<MODE_ORIENT>(g, b, 0, keep, g->stream);
        }
        int64_t first = n_big;  // warp-tier tasks not yet launched
        if (pivot && n_split > 0) {
            // pivot root split: the warp-tier tasks with more than
            // kPivotSplitD locals become one task per root branch
            keep.emplace_back(new DevBuf(4 * size_t(n_split), g->aux));
            int32_t *root_piv = keep.back()->as<int32_t>();
            keep.emplace_back(new DevBuf(16 * size_t(n_split), g->aux));
            uint32_t *root_P = keep.back()->as<uint32_t>();
            keep.emplace_back(new DevBuf(4 * size_t(n_split), g->aux));
            int32_t *root_cnt = keep.back()->as<int32_t>();
            keep.emplace_back(new DevBuf(4 * size_t(n_split), g->aux));
            int32_t *boff = keep.back()->as<int32_t>();
            KC_CUDA(cudaMemsetAsync(root_cnt, 0, 4 * size_t(n_split), g->aux));
            CountParams r = p;
            r.tasks = tasks.as<int32_t>() + n_big;
            r.n_tasks = n_split;
            r.roots_only = 1;
            r.use_gq = 0;
            r.root_piv = root_piv;
            r.root_P = root_P;
            r.root_cnt = root_cnt;
            r.task_counter = o + 8 + kSmidSlots + 7;
            launch_warp<MODE_PIVOT>(g, r, keep, g->aux);
            size_t bytes = 0;
            KC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, root_cnt, boff, int(n_split),
                                                  g->aux));
            keep.emplace_back(new DevBuf(bytes > 0 ? bytes : 1, g->aux));
            void *tmp = keep.back()->p;
            KC_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, root_cnt, boff, int(n_split),
                                                  g->aux));
            int32_t hl[2] = {0, 0};
            KC_CUDA(cudaMemcpyAsync(&hl[0], boff + n_split - 1, 4, cudaMemcpyDeviceToHost, g->aux));
            KC_CUDA(cudaMemcpyAsync(&hl[1], root_cnt + n_split - 1, 4, cudaMemcpyDeviceToHost,
                                    g->aux));
            KC_CUDA(cudaStreamSynchronize(g->aux));
            const int64_t nb = int64_t(hl[0]) + hl[1];
            if (nb > 0) {
                keep.emplace_back(new DevBuf(12 * size_t(nb), g->aux));
                int32_t *bt = keep.back()->as<int32_t>();
                k_branch_list<<<grid_1d(n_split, g->num_sms), 256, 0, g->aux>>>(
                    root_cnt, boff, root_P, n_split, tasks.as<int32_t>() + n_big, bt, bt + nb,
                    bt + 2 * nb);
                KC_CUDA(cudaGetLastError());
                CountParams b = p;
                b.branch = 1;
                b.tasks = bt;
                b.task_w = bt + nb;
                b.branch_si = bt + 2 * nb;
                b.root_piv = root_piv;
                b.root_P = root_P;
                b.n_tasks = nb;
                b.task_counter = o + 8 + kSmidSlots + 8;
                launch_warp<MODE_PIVOT>(g, b, keep, g->aux);
            }
            first = n_big + n_split;
        }
        if (n_tasks - first > 0) {
            CountParams q = p;
            q.tasks = tasks.as<int32_t>() + first;
            q.n_tasks = n_tasks - first;
            q.task_counter = o + 7;
            if (pivot) launch_warp<MODE_PIVOT>(g, q, keep, g->aux);
            else launch_warp<MODE_ORIENT>(g, q, keep, g->aux);
        }
    }
    if (edge_like) {
        ull ovf_hdr[7] = {0, 0, 0, 0, 0, 0, 0};
        KC_CUDA(cudaMemcpyAsync(ovf_hdr, p.overflow_n, sizeof(ovf_hdr), cudaMemcpyDeviceToHost,
                                g->stream));
        KC_CUDA(cudaStreamSynchronize(g->stream));
        const ull n_ovf = ovf_hdr[0];
        if (n_ovf > 0) {
            // in split mode only triples can overflow (items and roots are
            // routed by exact size); elsewhere only plain edge tasks
            CountParams b = p;
            b.scheme = KC_SCHEME_EDGE;
            b.t = split ? t - 2 : t;
            b.split = split ? 1 : 0;
            b.task_w = split ? ovf_w.as<int32_t>() : nullptr;
            b.tasks = ovf.as<int32_t>();
            b.n_tasks = int64_t(n_ovf);
            // shared memory sized for the largest overflow task, not d_max:
            // RMAT-22 k=7 overflow triples have <= 416 locals against d_max 964
            b.dcap = int(std::max<ull>(std::min<ull>(ovf_hdr[6], ull(p.dcap)), 1ull));
            b.wcap = (b.dcap + 31) / 32;
            b.task_counter = o + 8 + kSmidSlots + 4;
            if (pivot) launch<MODE_PIVOT>(g, b, 0, keep, g->stream);
            else launch<MODE_ORIENT>(g, b, 0, keep, g->stream);
        }
    }
    if (p.use_spill) {
        // spill rounds: walk the items the previous round handed over (bounded
        // again), big sets on the CTA tier, the rest on the warp tier, until a
        // round hands nothing over
        KC_CUDA(cudaStreamSynchronize(g->aux));
        KC_CUDA(cudaStreamSynchronize(g->stream));
        int cur = 0;
        for (int round = 1;; ++round) {
            ull hdr[5];
            KC_CUDA(cudaMemcpy(hdr, spb.ctl(cur), sizeof(hdr), cudaMemcpyDeviceToHost));
            const int64_t n_small = int64_t(std::min<ull>(hdr[1], spb.cap_small));
            const int64_t n_big = int64_t(std::min<ull>(hdr[2], spb.cap_big));
            if (timing_on())
                fprintf(stderr, "[kc_timing] spill round %d: small %lld big %lld words %llu "
                        "failed %llu\n", round, (long long)n_small, (long long)n_big,
                        hdr[0], hdr[3]), fflush(stderr);
            if (n_small == 0 && n_big == 0) break;
            // budget of this round: small while few items are in flight (the
            // tail, where one long walk would idle the GPU), larger when the
            // items far outnumber the warps -- fewer, bigger spills keep the
            // item count (and the per-item rebuild cost) bounded
            const int64_t warps = int64_t(g->num_sms) * 16;
            const int64_t scale = std::max<int64_t>(1, (n_small + n_big) / (4 * warps));
            const int round_budget =
                int(std::min<int64_t>(int64_t(p.spill_budget) * std::min<int64_t>(scale, 64),
                                      int64_t(1) << 30));
            const int nxt = cur ^ 1;
            KC_CUDA(cudaMemsetAsync(spb.ctl(nxt), 0, 8 * 8, g->stream));
            keep.emplace_back(new DevBuf(16, g->stream));
            ull *ctr = keep.back()->as<ull>();
            KC_CUDA(cudaMemsetAsync(ctr, 0, 16, g->stream));
            KC_CUDA(cudaEventRecord(e_fork, g->stream));
            KC_CUDA(cudaStreamWaitEvent(g->aux, e_fork, 0));
            if (n_big > 0) {
                CountParams b = p;
                b.spill = spb.at(nxt);
                b.spill_budget = round_budget;
                b.in_buf = spb.buf(cur);
                b.in_off = spb.big_off(cur);
                b.n_tasks = n_big;
                b.tasks = nullptr;
                b.task_w = nullptr;
                b.split = 0;
                b.task_counter = ctr;
                b.dcap = int(std::max<ull>(std::min<ull>(hdr[4], ull(p.dcap)), 1ull));
                b.wcap = (b.dcap + 31) / 32;
                launch<MODE_PIVOT>(g, b, 0, keep, g->stream);
            }
            if (n_small > 0) {
                CountParams q = p;
                q.spill = spb.at(nxt);
                q.spill_budget = round_budget;
                q.in_buf = spb.buf(cur);
                q.in_off = spb.small_off(cur);
                q.n_tasks = n_small;
                q.tasks = nullptr;
                q.task_w = nullptr;
                q.split = 0;
                q.branch = 0;
                q.roots_only = 0;
                q.task_counter = ctr + 1;
                launch_warp<MODE_PIVOT>(g, q, keep, g->aux);
            }
            KC_CUDA(cudaStreamSynchronize(g->aux));
            KC_CUDA(cudaStreamSynchronize(g->stream));
            cur = nxt;
            KC_REQUIRE(round < 100000, KC_ECUDA, "spill rounds do not terminate");
        }
    }
    KC_CUDA(cudaEventRecord(e_join, g->aux));
    KC_CUDA(cudaStreamWaitEvent(g->stream, e_join, 0));
    KC_CUDA(cudaEventRecord(e1, g->stream));
    KC_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    KC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    for (auto &lt : tl_timers) {
        float lms = 0;
        cudaEventElapsedTime(&lms, lt.a, lt.b);
        fprintf(stderr, "[kc_timing] %-22s tasks=%-10lld grid=%-5d %10.3f ms\n", lt.what,
                (long long)lt.n_tasks, lt.grid, lms);
        cudaEventDestroy(lt.a);
        cudaEventDestroy(lt.b);
    }
    if (!tl_timers.empty()) {
        fprintf(stderr, "[kc_timing] count phase %10.3f ms\n", ms);
        std::vector<ull> hp(kProfWords);
        KC_CUDA(cudaMemcpy(hp.data(), prof.p, 8 * hp.size(), cudaMemcpyDeviceToHost));
        fprintf(stderr,
                "[kc_timing] cycles: cta build %.3e walk %.3e (per CTA, thread 0); warp build "
                "%.3e walk %.3e (summed over warps)\n",
                double(hp[kProfCtaBuild]), double(hp[kProfCtaWalk]), double(hp[kProfWarpBuild]),
                double(hp[kProfWarpWalk]));
        fprintf(stderr,
                "[kc_timing] subtree queue: idle %.3e walk %.3e cycles (summed over warps), "
                "items id-list %llu compressed %llu\n",
                double(hp[kProfGqIdle]), double(hp[kProfGqWalk]), hp[kProfGqItems],
                hp[kProfGqItems + 1]);
        fprintf(stderr, "[kc_timing] overflow sizes (32-local buckets):");
        for (int b = 0; b < 64; ++b)
            if (hp[kProfOvfHist + b]) fprintf(stderr, " %d:%llu", (b + 1) * 32, hp[kProfOvfHist + b]);
        fprintf(stderr, "\n");
    }
    tl_timers.clear();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e_fork);
    cudaEventDestroy(e_join);

    std::vector<ull> h(kOutWords);
    KC_CUDA(cudaMemcpyAsync(h.data(), outs.p, 8 * h.size(), cudaMemcpyDeviceToHost, g->stream));
    if (L)
        KC_CUDA(cudaMemcpyAsync(hist, dhist.p, 8 * size_t(L * L), cudaMemcpyDeviceToHost,
                                g->stream));
    KC_CUDA(cudaStreamSynchronize(g->stream));
    int gq_ctl[8];
    memcpy(gq_ctl, &h[kOutGq], sizeof(gq_ctl));
    // every handed-over subtree must have been walked (its leaves are in hist)
    KC_REQUIRE(gq_ctl[1] == 0, KC_ECUDA, "subtree queue not drained at kernel exit");
    raw->word_ops = h[8 + kSmidSlots];
    raw->extract_bytes = h[9 + kSmidSlots];
    for (int i = 0; i < 4; ++i) raw->limbs[i] = h[1 + i];
    const ull tri_items = (split && t >= 6) ? ull(n_items_big) : 0ull;
    raw->visits = h[5] + tri_items;  // u's visit of every item split into triples
    if (p.use_gq && getenv("KC_GQ_DEBUG"))
        fprintf(stderr, "[kc_gq] pushes=%d pops=%d size=%d hungry=%d busy=%d\n", gq_ctl[4],
                gq_ctl[5], gq_ctl[1], gq_ctl[2], gq_ctl[3]);
    raw->tasks_run = h[6];
    raw->count_ms = ms;
    raw->group_size = pivot ? 1 : p.group_size;
    raw->launches = tl_launches;
    if (visits_per_sm) {
        for (int i = 0; i < n_sm && i < kSmidSlots; ++i) visits_per_sm[i] = h[8 + i];
        if (n_sm > 0) visits_per_sm[0] += tri_items;  // see raw->visits
    }
}

namespace {
// per-task cost estimate for shard balancing, make_tasks order (scheduler.py:89-95)
//   vertex tasks, orientation t >= 4 (hub roots split into out-edge items):
//       sum over out-edges e of (1 + |N+(u) n N+(v)|)^2     (the split items' cost)
//   other vertex tasks: d+(v)^2;   edge tasks: (1 + |N+(u) n N+(v)|)^2
__global__ void k_vertex_cost(const int64_t *__restrict__ orow, const int32_t *__restrict__ esize,
                              int64_t n, int64_t *__restrict__ cost) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t v = warp; v < n; v += nw) {
        const int64_t b = orow[v], e = orow[v + 1];
        int64_t c = 0;
        if (esize) {
            for (int64_t i = b + lane; i < e; i += 32) {
                const int64_t x = 1 + esize[i];
                c += x * x;
            }
            for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        } else {
            c = (e - b) * (e - b);
        }
        if (lane == 0) cost[v] = c;
    }
}

__global__ void k_edge_cost(const int32_t *__restrict__ esize, int64_t m, int64_t *__restrict__ cost) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t x = 1 + esize[i];
        cost[i] = x * x;
    }
}

// cuts[r] = 1 + first i with cum[i] >= total * r / world (shard.balanced_ranges)
__global__ void k_cuts(const int64_t *__restrict__ cum, int64_t n, int world, int64_t *cuts) {
    const double total = double(cum[n - 1]);
    for (int r = threadIdx.x + 1; r < world; r += blockDim.x) {
        const double target = total * double(r) / double(world);
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (double(cum[mid]) < target) lo = mid + 1;
            else hi = mid;
        }
        cuts[r] = lo + 1;
    }
}
}  // namespace

// device task costs in make_tasks order; returns the task count, costs in *out
static int64_t device_task_costs(kc_graph *g, const kc_count_args *a, DevBuf &out) {
    const bool pivot = a->algorithm == KC_ALGO_PIVOT;
    const int t = a->scheme == KC_SCHEME_VERTEX ? a->k - 1 : a->k - 2;
    const bool split = !pivot && a->scheme == KC_SCHEME_VERTEX && t >= 4;
    if ((split || a->scheme == KC_SCHEME_EDGE) && !g->esize && g->m_dir > 0) {
        g->esize = kc_alloc<int32_t>(g->m_dir, g->stream);
        k_edge_sizes<<<g->num_sms * 16, 256, 0, g->stream>>>(g->orow_ptr, g->ocol, g->ocoo,
                                                             g->m_dir, g->esize);
        KC_CUDA(cudaGetLastError());
    }
    if (a->scheme == KC_SCHEME_EDGE) {
        new (&out) DevBuf(8 * size_t(std::max<int64_t>(g->m_dir, 1)));
        if (g->m_dir)
            k_edge_cost<<<grid_1d(g->m_dir, g->num_sms), 256, 0, g->stream>>>(
                g->esize, g->m_dir, out.as<int64_t>());
        KC_CUDA(cudaGetLastError());
        return g->m_dir;
    }
    const int64_t n = g->n;
    if (n == 0) {
        new (&out) DevBuf(8);
        return 0;
    }
    DevBuf cost(8 * size_t(n)), flag(4 * size_t(n)), cnt(8);
    k_vertex_cost<<<g->num_sms * 16, 256, 0, g->stream>>>(g->orow_ptr, split ? g->esize : nullptr,
                                                          n, cost.as<int64_t>());
    k_vertex_flags<<<grid_1d(n, g->num_sms), 256, 0, g->stream>>>(g->orow_ptr, n,
                                                                   flag.as<int32_t>());
    new (&out) DevBuf(8 * size_t(n));
    size_t bytes = 0;
    KC_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, cost.as<int64_t>(), flag.as<int32_t>(),
                                       out.as<int64_t>(), cnt.as<int32_t>(), int(n), g->stream));
    void *tmp = kc_tmp(g, bytes);
    KC_CUDA(cub::DeviceSelect::Flagged(tmp, bytes, cost.as<int64_t>(), flag.as<int32_t>(),
                                       out.as<int64_t>(), cnt.as<int32_t>(), int(n), g->stream));
    int32_t h = 0;
    KC_CUDA(cudaMemcpyAsync(&h, cnt.p, 4, cudaMemcpyDeviceToHost, g->stream));
    KC_CUDA(cudaStreamSynchronize(g->stream));
    return h;
}

void kc_do_task_costs(kc_graph *g, const kc_count_args *a, int64_t *costs, int64_t n_tasks) {
    KC_REQUIRE(g->oriented, KC_EINVAL, "graph is not oriented");
    kc_device_guard guard(g->device);
    StreamScope scope(g->stream);
    DevBuf out;
    const int64_t n = device_task_costs(g, a, out);
    KC_REQUIRE(n == n_tasks, KC_EINVAL, "n_tasks does not match make_tasks");
    if (n)
        KC_CUDA(cudaMemcpyAsync(costs, out.p, 8 * size_t(n), cudaMemcpyDeviceToHost, g->stream));
    KC_CUDA(cudaStreamSynchronize(g->stream));
}

void kc_do_shard_ranges(kc_graph *g, const kc_count_args *a, int world, int64_t *cuts) {
    KC_REQUIRE(g->oriented, KC_EINVAL, "graph is not oriented");
    KC_REQUIRE(world >= 1, KC_EINVAL, "world must be >= 1");
    kc_device_guard guard(g->device);
    StreamScope scope(g->stream);
    DevBuf cost;
    const int64_t n = device_task_costs(g, a, cost);
    std::vector<int64_t> h(size_t(world) + 1, 0);
    h[world] = n;
    if (world > 1 && n > 0) {
        DevBuf cum(8 * size_t(n)), dc(8 * (size_t(world) + 1));
        size_t bytes = 0;
        KC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, cost.as<int64_t>(),
                                              cum.as<int64_t>(), int(n), g->stream));
        void *tmp = kc_tmp(g, bytes);
        KC_CUDA(cub::DeviceScan::InclusiveSum(tmp, bytes, cost.as<int64_t>(), cum.as<int64_t>(),
                                              int(n), g->stream));
        k_cuts<<<1, 128, 0, g->stream>>>(cum.as<int64_t>(), n, world, dc.as<int64_t>());
        KC_CUDA(cudaGetLastError());
        KC_CUDA(cudaMemcpyAsync(h.data() + 1, dc.as<int64_t>() + 1, 8 * size_t(world - 1),
                                cudaMemcpyDeviceToHost, g->stream));
        KC_CUDA(cudaStreamSynchronize(g->stream));
    } else if (world > 1) {
        for (int r = 1; r < world; ++r) h[r] = 0;
    }
    for (int r = 0; r <= world; ++r) {  // clip + monotone, as shard.balanced_ranges
        h[r] = std::min(std::max<int64_t>(h[r], 0), n);
        if (r > 0) h[r] = std::max(h[r], h[r - 1]);
    }
    h[world] = n;
    memcpy(cuts, h.data(), 8 * (size_t(world) + 1));
}

void kc_do_extract(kc_graph *g, int scheme, int64_t task, int directed, int64_t *l2g,
                   uint64_t *words, int64_t cap, int64_t wpr_cap, int64_t *d_out) {
    KC_REQUIRE(g->oriented, KC_EINVAL, "graph is not oriented");
    const int64_t N = scheme == KC_SCHEME_EDGE ? g->m_dir : g->n;
    KC_REQUIRE(task >= 0 && task < N, KC_EINVAL, "task out of range");
    kc_device_guard guard(g->device);
    StreamScope scope(g->stream);
    const int dcap = int(std::max<int64_t>(g->d_max, 1));
    const int wcap = (dcap + 31) / 32;
    DevBuf tk(4), rows(4 * size_t(dcap) * wcap), l(4 * size_t(dcap)), dd(4), outs(64);
    int32_t t32 = int32_t(task);
    KC_CUDA(cudaMemcpyAsync(tk.p, &t32, 4, cudaMemcpyHostToDevice, g->stream));
    KC_CUDA(cudaMemsetAsync(outs.p, 0, 64, g->stream));
    CountParams p;
    memset(&p, 0, sizeof(p));
    p.orow = g->orow_ptr;
    p.ocol = g->ocol;
    p.ocoo = g->ocoo;
    p.tasks = tk.as<int32_t>();
    p.n_tasks = 1;
    p.scheme = scheme;
    p.t = 2;
    p.dcap = dcap;
    p.wcap = wcap;
    p.directed_out = directed;
    p.extract_rows = rows.as<uint32_t>();
    p.extract_l2g = l.as<int32_t>();
    p.extract_d = dd.as<int>();
    p.task_counter = outs.as<ull>();
    launch_sync<MODE_EXTRACT>(g, p, 1);
    int d = 0;
    KC_CUDA(cudaMemcpyAsync(&d, dd.p, 4, cudaMemcpyDeviceToHost, g->stream));
    KC_CUDA(cudaStreamSynchronize(g->stream));
    KC_REQUIRE(d <= cap, KC_EINVAL, "scratch BitGraph too small for this task");
    const int W = (d + 31) / 32;
    const int64_t wpr = (d + 63) / 64;
    KC_REQUIRE(wpr <= wpr_cap || d == 0, KC_EINVAL, "words_per_row capacity too small");
    std::vector<int32_t> hl(d > 0 ? d : 1);
    std::vector<uint32_t> hr(size_t(d) * W + 1);
    if (d) {
        KC_CUDA(cudaMemcpyAsync(hl.data(), l.p, 4 * size_t(d), cudaMemcpyDeviceToHost, g->stream));
        KC_CUDA(cudaMemcpyAsync(hr.data(), rows.p, 4 * size_t(d) * W, cudaMemcpyDeviceToHost,
                                g->stream));
        KC_CUDA(cudaStreamSynchronize(g->stream));
    }
    for (int i = 0; i < d; ++i) {
        l2g[i] = hl[i];
        for (int64_t w = 0; w < wpr_cap; ++w) {
            uint64_t lo = 2 * w < W ? hr[size_t(i) * W + 2 * w] : 0;
            uint64_t hi = 2 * w + 1 < W ? hr[size_t(i) * W + 2 * w + 1] : 0;
            words[i * wpr_cap + w] = lo | (hi << 32);
        }
    }
    *d_out = d;
}

// one host-provided matrix through the same device traversal
void kc_do_count_bitgraph(int device, const uint64_t *rows64, int64_t d64, int t, int algorithm,
                          int all_t, uint64_t *out4, uint64_t *slots_lo, uint64_t *slots_hi) {
    KC_REQUIRE(d64 >= 0 && d64 < (1 << 20), KC_EINVAL, "bad local count");
    KC_REQUIRE(t >= 0, KC_EINVAL, "t must be non-negative");
    const int d = int(d64);
    memset(out4, 0, 4 * sizeof(uint64_t));
    const bool pivot = algorithm == KC_ALGO_PIVOT;
    if (!(pivot && all_t) && t <= 1) {
        out4[0] = t == 0 ? 1 : uint64_t(d);
        return;
    }
    if (pivot && all_t && d == 0) {
        slots_lo[0] = 1;
        slots_hi[0] = 0;
        return;
    }
    if (d == 0) return;
    kc_device_guard guard(device);
    kc_graph tmpg;
    tmpg.device = device;
    KC_CUDA(cudaDeviceGetAttribute(&tmpg.num_sms, cudaDevAttrMultiProcessorCount, device));
    tmpg.stream = nullptr;  // legacy stream: host copies below are ordered with it
    StreamScope scope(nullptr);
    const int W = (d + 31) / 32;
    const int64_t wpr = (d + 63) / 64;
    std::vector<uint32_t> r32(size_t(d) * W);
    for (int i = 0; i < d; ++i)
        for (int w = 0; w < W; ++w) {
            uint64_t x = rows64[i * wpr + (w >> 1)];
            r32[size_t(i) * W + w] = uint32_t(w & 1 ? x >> 32 : x);
        }
    DevBuf dr(4 * r32.size()), outs(8 * (8 + size_t(kSmidSlots)));
    const int64_t L = d + 2;
    DevBuf dh(8 * size_t(L * L));
    KC_CUDA(cudaMemcpy(dr.p, r32.data(), 4 * r32.size(), cudaMemcpyHostToDevice));
    KC_CUDA(cudaMemset(outs.p, 0, 8 * (8 + size_t(kSmidSlots))));
    KC_CUDA(cudaMemset(dh.p, 0, 8 * size_t(L * L)));
    CountParams p;
    memset(&p, 0, sizeof(p));
    p.n_tasks = 1;
    p.scheme = KC_SCHEME_VERTEX;
    p.t = t;
    p.all_k = pivot && all_t;
    p.dcap = d;
    p.wcap = W;
    p.given_rows = dr.as<uint32_t>();
    p.given_d = d;
    p.hist_dim = int(L);
    p.hist = dh.as<ull>();
    p.sh_hl = int(std::min<int64_t>(L, 48));
    ull *o = outs.as<ull>();
    p.task_counter = o;
    p.limbs = o + 1;
    p.visits_total = o + 5;
    p.tasks_run = o + 6;
    p.visits_per_sm = o + 8;
    try {
        if (pivot) {
            launch_sync<MODE_PIVOT>(&tmpg, p, 1);
        } else {
            launch_sync<MODE_ORIENT>(&tmpg, p, 1);
        }
    } catch (...) {
        throw;
    }
    std::vector<ull> h(8);
    KC_CUDA(cudaMemcpy(h.data(), outs.p, 64, cudaMemcpyDeviceToHost));
    typedef unsigned __int128 u128;
    if (!pivot) {
        u128 c = u128(h[1]) + (u128(h[2]) << 32);
        out4[0] = uint64_t(c);
        out4[1] = uint64_t(c >> 64);
        out4[2] = h[5];
        return;
    }
    std::vector<ull> hh(size_t(L * L));
    KC_CUDA(cudaMemcpy(hh.data(), dh.p, 8 * hh.size(), cudaMemcpyDeviceToHost));
    // exact binomials by Pascal's rule with a saturation flag (engine_pivot.py:57-65)
    std::vector<u128> C(size_t(L * L), 0);
    std::vector<uint8_t> big(size_t(L * L), 0);
    for (int n = 0; n < L; ++n)
        for (int r = 0; r <= n; ++r) {
            size_t i = size_t(n) * L + r;
            if (r == 0 || r == n) C[i] = 1;
            else {
                size_t a = size_t(n - 1) * L + r - 1, b = size_t(n - 1) * L + r;
                u128 s = C[a] + C[b];
                big[i] = big[a] || big[b] || s < C[a];
                C[i] = big[i] ? 0 : s;
            }
        }
    bool over = false;
    out4[2] = h[5];
    if (all_t) {
        std::vector<u128> slot(size_t(d) + 2, 0);
        for (int len = 0; len < L; ++len)
            for (int np = 0; np <= len && np < L; ++np) {
                ull cnt = hh[size_t(len) * L + np];
                if (!cnt) continue;
                for (int r = 0; r <= np; ++r) {
                    size_t i = size_t(np) * L + r;
                    if (big[i]) { over = true; continue; }
                    u128 prod;
                    if (__builtin_mul_overflow(C[i], u128(cnt), &prod)) { over = true; continue; }
                    u128 &s = slot[len - r];
                    if (s + prod < s) over = true;
                    s += prod;
                }
            }
        for (int i = 0; i <= d; ++i) {
            slots_lo[i] = uint64_t(slot[i]);
            slots_hi[i] = uint64_t(slot[i] >> 64);
        }
    } else {
        u128 total = 0;
        for (int len = t; len < L; ++len)
            for (int np = 0; np <= len && np < L; ++np) {
                ull cnt = hh[size_t(len) * L + np];
                if (!cnt) continue;
                size_t i = size_t(np) * L + (len - t);
                if (len - t > np) continue;
                if (big[i]) { over = true; continue; }
                u128 prod;
                if (__builtin_mul_overflow(C[i], u128(cnt), &prod)) { over = true; continue; }
                if (total + prod < total) over = true;
                total += prod;
            }
        out4[0] = uint64_t(total);
        out4[1] = uint64_t(total >> 64);
    }
    out4[3] = over ? 1 : 0;
}

namespace {
template <int WPL>
__global__ void k_find_pivot(const uint32_t *rows, int d, const uint32_t *cand, int *out) {
    __shared__ int list[4096];
    const int W = (d + 31) >> 5, lane = threadIdx.x & 31;
    kct::Set<WPL> C;
#pragma unroll
    for (int p = 0; p < WPL; ++p) C.w[p] = p * 32 + lane < W ? cand[p * 32 + lane] : 0u;
    ull work = 0;
    const int pv = kct::select_pivot<WPL>(rows, W, C, list, lane, work, W);
    if (threadIdx.x == 0) out[0] = pv;
}
}  // namespace

void kc_do_find_pivot(int device, const uint64_t *rows64, int64_t d64, const uint64_t *cand64,
                      int64_t *pivot, uint64_t *pruned) {
    KC_REQUIRE(d64 > 0 && d64 <= 4096, KC_EINVAL, "find_pivot supports 1..4096 locals");
    const int d = int(d64);
    const int W = (d + 31) / 32;
    const int64_t wpr = (d + 63) / 64;
    bool any = false;
    for (int64_t w = 0; w < wpr; ++w) any |= cand64[w] != 0;
    KC_REQUIRE(any, KC_EINVAL, "candidate set is empty");
    kc_device_guard guard(device);
    StreamScope scope(nullptr);
    std::vector<uint32_t> r32(size_t(d) * W), c32(W);
    for (int i = 0; i < d; ++i)
        for (int w = 0; w < W; ++w) {
            uint64_t x = rows64[i * wpr + (w >> 1)];
            r32[size_t(i) * W + w] = uint32_t(w & 1 ? x >> 32 : x);
        }
    for (int w = 0; w < W; ++w) c32[w] = uint32_t(w & 1 ? cand64[w >> 1] >> 32 : cand64[w >> 1]);
    DevBuf dr(4 * r32.size()), dc(4 * size_t(W)), dout(4);
    KC_CUDA(cudaMemcpy(dr.p, r32.data(), 4 * r32.size(), cudaMemcpyHostToDevice));
    KC_CUDA(cudaMemcpy(dc.p, c32.data(), 4 * c32.size(), cudaMemcpyHostToDevice));
    if (W <= 32) k_find_pivot<1><<<1, 32>>>(dr.as<uint32_t>(), d, dc.as<uint32_t>(), dout.as<int>());
    else if (W <= 64) k_find_pivot<2><<<1, 32>>>(dr.as<uint32_t>(), d, dc.as<uint32_t>(), dout.as<int>());
    else k_find_pivot<4><<<1, 32>>>(dr.as<uint32_t>(), d, dc.as<uint32_t>(), dout.as<int>());
    KC_CUDA(cudaGetLastError());
    int pv = 0;
    KC_CUDA(cudaMemcpy(&pv, dout.p, 4, cudaMemcpyDeviceToHost));
    *pivot = pv;
    for (int64_t w = 0; w < wpr; ++w) pruned[w] = cand64[w] & ~rows64[pv * wpr + w];
}
