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
#include <vector>

#include "kc_internal.cuh"

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
    int dcap;          // max locals per task
    int wcap;          // ceil(dcap / 32)
    int group_size;    // orient: 0 = auto per task
    int rows_in_smem;  // rows in shared memory, else in rows_global slot
    uint32_t *rows_global;
    int64_t rows_slot;   // u32 words per CTA slot
    int stack_words;     // orient: smem words for group stacks
    int pv_smem_frames;  // pivot: frames per warp held in smem
    uint32_t *pv_global; // pivot: deep frames, per-warp slots
    int64_t pv_slot;     // u32 words per warp slot
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
};

__host__ __device__ __forceinline__ int row_stride(int W) { return W | 1; }

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

// Returns d (number of locals); fills l2g and (when t >= 2 or pivot) rows.
// scratch must hold >= dcap int32 (used for the edge scheme's second list).
template <int BLOCK>
__device__ int build_task(const CountParams &p, int32_t task, int32_t *l2g, uint32_t *rows,
                          int32_t *scratch, bool need_rows, bool directed, int *s_cnt,
                          int *s_warp, ull &bytes) {
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
            block_append<BLOCK>(f, x, l2g, s_cnt, s_warp);
        }
        d = *s_cnt;
    }
    __syncthreads();
    if (!need_rows || d == 0) return d;
    const int W = (d + 31) >> 5, RS = row_stride(W);
    for (int i = tid; i < d * RS; i += BLOCK) rows[i] = 0u;
    __syncthreads();
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
            const int j = smem_find(l2g, d, x);
            if (j >= 0) {
                atomicOr(&rows[i * RS + (j >> 5)], 1u << (j & 31));
                if (!directed) atomicOr(&rows[j * RS + (i >> 5)], 1u << (i & 31));
            }
        }
    }
    __syncthreads();
    return d;
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
// K5: orient traversal with sub-warp groups
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int auto_group(int W) {
    int g = 1;
    while (g < W && g < 32) g <<= 1;
    return g;
}

// group stack stride in words: 2 rows (cand, rem) per frame plus a cursor
// word per frame; stride == G (mod 32) keeps the lanes of a warp on distinct banks
__host__ __device__ __forceinline__ int group_stride(int frames, int W, int G) {
    int need = frames * (2 * W + 1);
    need = (need + 31) & ~31;
    return need + (G & 31);
}

template <int BLOCK>
__device__ void orient_task(const CountParams &p, const uint32_t *rows, int d, uint32_t *stack,
                            int *s_next, ull &acc, ull &visits, ull &work) {
    const int t = p.t;
    const int tid = threadIdx.x, lane = tid & 31;
    const int W = (d + 31) >> 5, RS = row_stride(W);
    int G = p.group_size > 0 ? p.group_size : auto_group(W);
    const int frames = t - 2 > 0 ? t - 2 : 0;  // frames 1..t-2 are materialized
    const int GS = group_stride(frames, W, G);
    int NG = BLOCK / G;
    if (frames > 0 && NG * GS > p.stack_words) NG = p.stack_words / GS;
    const int gid = tid / G, gl = tid & (G - 1);
    if (gid >= NG) return;
    const int gbase = lane & ~(G - 1);
    const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << gbase);
    const int last = t - 2;
    const int nchunks = (W + G - 1) / G;
    uint32_t *st = stack + gid * GS;
    // frame f (1..frames): cand at (f-1)*(2W+1), rem at +W, cursor at +2W
    auto cand = [&](int f) { return st + (f - 1) * (2 * W + 1); };
    auto rem = [&](int f) { return st + (f - 1) * (2 * W + 1) + W; };
    auto cur = [&](int f) { return st + (f - 1) * (2 * W + 1) + 2 * W; };

    for (;;) {
        int u = 0;
        if (gl == 0) u = atomicAdd(s_next, 1);
        u = __shfl_sync(gmask, u, 0, G);
        if (u >= d) break;
        // frame 0 expands u (engine_orient.py:58-62); S0 = all locals
        if (gl == 0) {
            ++visits;
            work += W;
        }
        const uint32_t *ru = rows + u * RS;
        if (last == 0) {
            for (int w = gl; w < W; w += G) acc += __popc(ru[w]);
            continue;
        }
        uint32_t nz = 0;
        for (int w = gl; w < W; w += G) {
            uint32_t x = ru[w];
            cand(1)[w] = x;
            rem(1)[w] = x;
            nz |= x;
        }
        if (!(__ballot_sync(gmask, nz != 0) & gmask)) continue;
        int s = 1;
        if (gl == 0) *cur(1) = 0;
        __syncwarp(gmask);
        while (s >= 1) {
            int v = -1;
            int c = *cur(s);
            for (; c < nchunks; ++c) {
                const int w = c * G + gl;
                uint32_t x = w < W ? rem(s)[w] : 0u;
                unsigned b = __ballot_sync(gmask, x != 0) & gmask;
                if (b) {
                    const int src = __ffs(b) - 1;
                    const uint32_t wx = __shfl_sync(gmask, x, src);
                    v = ((c * G + src - gbase) << 5) + __ffs(wx) - 1;
                    if (lane == src) rem(s)[w] = x & (x - 1u);
                    break;
                }
            }
            __syncwarp(gmask);
            if (gl == 0) *cur(s) = c;
            __syncwarp(gmask);
            if (v < 0) {
                --s;
                continue;
            }
            if (gl == 0) {
                ++visits;
                work += W;
            }
            const uint32_t *rv = rows + v * RS;
            const uint32_t *cs = cand(s);
            if (s == last) {
                for (int w = gl; w < W; w += G) acc += __popc(cs[w] & rv[w]);
            } else {
                uint32_t *cn = cand(s + 1), *rn = rem(s + 1);
                uint32_t nz2 = 0;
                for (int w = gl; w < W; w += G) {
                    uint32_t y = cs[w] & rv[w];
                    cn[w] = y;
                    rn[w] = y;
                    nz2 |= y;
                }
                if (__ballot_sync(gmask, nz2 != 0) & gmask) {
                    ++s;
                    if (gl == 0) *cur(s) = 0;
                    __syncwarp(gmask);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K6/K7: pivot traversal (warp groups)
// ---------------------------------------------------------------------------
// frame layout (words): cand[W] pruned[W] rem[W] piv npv cur
__host__ __device__ __forceinline__ int pv_frame_words(int W) { return 3 * W + 3; }

struct PivotFrames {
    uint32_t *sm;  // first pv_smem_frames frames
    uint32_t *gm;  // deeper frames
    int nsm;
    int fw;
    __device__ __forceinline__ uint32_t *f(int s) const {
        return s < nsm ? sm + s * fw : gm + (s - nsm) * fw;
    }
};

// argmax_{c in cand} |cand & row(c)|, lowest c on ties (engine_pivot.py:82-101).
// Whole warp; candidates compacted into `list`, scored lane-parallel.
__device__ int warp_select_pivot(const uint32_t *rows, int RS, int W, const uint32_t *cand,
                                 int *list, ull &work) {
    const int lane = threadIdx.x & 31;
    int n_c = 0;
    for (int c0 = 0; c0 < W; c0 += 32) {
        const int w = c0 + lane;
        uint32_t x = w < W ? cand[w] : 0u;
        int cnt = __popc(x), incl = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        int off = n_c + incl - cnt;
        while (x) {
            list[off++] = (w << 5) + __ffs(x) - 1;
            x &= x - 1u;
        }
        n_c += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    if (lane == 0) work += ull(n_c) * W;
    ull best = 0;
    for (int i = lane; i < n_c; i += 32) {
        const int c = list[i];
        const uint32_t *rc = rows + c * RS;
        int cov = 0;
        for (int w = 0; w < W; ++w) cov += __popc(cand[w] & rc[w]);
        ull key = (ull(cov + 1) << 32) | ull(0xffffffffu - uint32_t(c));
        best = key > best ? key : best;
    }
    for (int o = 16; o; o >>= 1) {
        ull y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y > best ? y : best;
    }
    __syncwarp();
    return int(0xffffffffu - uint32_t(best & 0xffffffffull));
}

__device__ __forceinline__ void hist_add(const CountParams &p, ull *s_hist, int len, int np) {
    if (len < p.sh_hl) atomicAdd(&s_hist[len * (len + 1) / 2 + np], 1ull);
    else atomicAdd(&p.hist[int64_t(len) * p.hist_dim + np], 1ull);
}

// DFS of one root branch v0 (already expanded at frame 0 into frame 1 = child)
__device__ void pivot_dfs(const CountParams &p, const uint32_t *rows, int RS, int W,
                          const PivotFrames &F, int *list, ull *s_hist, ull &visits,
                          ull &work) {
    const int lane = threadIdx.x & 31;
    const int t = p.t;
    const bool allk = p.all_k != 0;
    int s = 1;
    while (s >= 1) {
        uint32_t *fr = F.f(s);
        uint32_t *C = fr, *P = fr + W, *R = fr + 2 * W;
        const int piv = int(fr[3 * W]);
        const int npv = int(fr[3 * W + 1]);
        int c = int(fr[3 * W + 2]);
        int v = -1;
        for (; c * 32 < W; ++c) {
            const int w = c * 32 + lane;
            uint32_t x = w < W ? R[w] : 0u;
            unsigned b = __ballot_sync(0xffffffffu, x != 0);
            if (b) {
                const int src = __ffs(b) - 1;
                const uint32_t wx = __shfl_sync(0xffffffffu, x, src);
                v = ((c * 32 + src) << 5) + __ffs(wx) - 1;
                if (lane == src) R[w] = x & (x - 1u);
                break;
            }
        }
        __syncwarp();
        if (lane == 0) fr[3 * W + 2] = uint32_t(c);
        __syncwarp();
        if (v < 0) {
            --s;
            continue;
        }
        const int np2 = npv + (v == piv ? 1 : 0);
        if (!allk && s + 1 - t > np2) continue;  // engine_pivot.py:152-153
        if (lane == 0) {
            ++visits;
            work += W;
        }
        const uint32_t *rv = rows + v * RS;
        uint32_t *fn = F.f(s + 1);
        uint32_t *Cn = fn;
        const int vq = v >> 5;
        const uint32_t below = (1u << (v & 31)) - 1u;
        uint32_t nz = 0;
        for (int w = lane; w < W; w += 32) {
            uint32_t x = C[w] & rv[w];
            // engine_pivot.py:158-166 drop already-branched pruned bits below v
            if (w < vq) x &= ~P[w];
            else if (w == vq) x &= ~(P[w] & below);
            Cn[w] = x;
            nz |= x;
        }
        const bool any = __ballot_sync(0xffffffffu, nz != 0) != 0;
        __syncwarp();
        if (any) {
            const int pv = warp_select_pivot(rows, RS, W, Cn, list, work);
            const uint32_t *rp = rows + pv * RS;
            for (int w = lane; w < W; w += 32) {
                uint32_t y = Cn[w] & ~rp[w];
                fn[W + w] = y;
                fn[2 * W + w] = y;
            }
            if (lane == 0) {
                fn[3 * W] = uint32_t(pv);
                fn[3 * W + 1] = uint32_t(np2);
                fn[3 * W + 2] = 0u;
            }
            __syncwarp();
            ++s;
        } else if (allk || s + 1 >= t) {
            if (lane == 0) hist_add(p, s_hist, s + 1, np2);
        }
    }
}

template <int BLOCK>
__device__ void pivot_task(const CountParams &p, const uint32_t *rows, int d, uint32_t *pv_area,
                           int *lists, ull *s_hist, int *s_next, int *s_piv0, ull *s_key,
                           ull &visits, ull &work) {
    constexpr int NW = BLOCK / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = (d + 31) >> 5, RS = row_stride(W);
    const int t = p.t;
    const bool allk = p.all_k != 0;
    const int fw = pv_frame_words(W);
    // frame 0 (shared by the block): cand = all locals, pivot by block argmax
    uint32_t *root = pv_area;  // W words cand, W words pruned
    for (int w = tid; w < W; w += BLOCK) {
        const int lo = w << 5;
        root[w] = lo + 32 <= d ? 0xffffffffu : ((1u << (d - lo)) - 1u);
    }
    ull best = 0;
    for (int c = tid; c < d; c += BLOCK) {
        const uint32_t *rc = rows + c * RS;
        int cov = 0;
        for (int w = 0; w < W; ++w) cov += __popc(rc[w]);
        ull key = (ull(cov + 1) << 32) | ull(0xffffffffu - uint32_t(c));
        best = key > best ? key : best;
    }
    for (int o = 16; o; o >>= 1) {
        ull y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y > best ? y : best;
    }
    if (lane == 0) s_key[warp] = best;
    if (tid == 0) *s_next = 0;  // next branch
    __syncthreads();
    if (tid == 0) {
        ull b = 0;
        for (int w = 0; w < NW; ++w) b = s_key[w] > b ? s_key[w] : b;
        *s_piv0 = int(0xffffffffu - uint32_t(b & 0xffffffffull));
    }
    __syncthreads();
    const int piv0 = *s_piv0;
    const uint32_t *rp0 = rows + piv0 * RS;
    for (int w = tid; w < W; w += BLOCK) root[W + w] = root[w] & ~rp0[w];
    __syncthreads();

    // warps take branch vertices v in pruned(0) ascending
    PivotFrames F;
    F.fw = fw;
    F.nsm = p.pv_smem_frames;
    F.sm = root + 2 * W + warp * (p.pv_smem_frames * fw);
    F.gm = p.pv_global + (int64_t(blockIdx.x) * NW + warp) * p.pv_slot;
    int *list = lists + warp * p.dcap;
    const uint32_t *P0 = root + W;
    for (;;) {
        int v = 0;
        if (lane == 0) v = atomicAdd(s_next, 1);
        v = __shfl_sync(0xffffffffu, v, 0);
        if (v >= d) break;
        if (!((P0[v >> 5] >> (v & 31)) & 1u)) continue;
        const int np2 = v == piv0 ? 1 : 0;
        if (!allk && 1 - t > np2) continue;
        if (lane == 0) {
            ++visits;
            work += W;
        }
        const uint32_t *rv = rows + v * RS;
        uint32_t *f1 = F.f(1);
        const int vq = v >> 5;
        const uint32_t below = (1u << (v & 31)) - 1u;
        uint32_t nz = 0;
        for (int w = lane; w < W; w += 32) {
            uint32_t x = root[w] & rv[w];
            if (w < vq) x &= ~P0[w];
            else if (w == vq) x &= ~(P0[w] & below);
            f1[w] = x;
            nz |= x;
        }
        const bool any = __ballot_sync(0xffffffffu, nz != 0) != 0;
        __syncwarp();
        if (!any) {
            if ((allk || 1 >= t) && lane == 0) hist_add(p, s_hist, 1, np2);
            continue;
        }
        const int pv = warp_select_pivot(rows, RS, W, f1, list, work);
        const uint32_t *rp = rows + pv * RS;
        for (int w = lane; w < W; w += 32) {
            uint32_t y = f1[w] & ~rp[w];
            f1[W + w] = y;
            f1[2 * W + w] = y;
        }
        if (lane == 0) {
            f1[3 * W] = uint32_t(pv);
            f1[3 * W + 1] = uint32_t(np2);
            f1[3 * W + 2] = 0u;
        }
        __syncwarp();
        pivot_dfs(p, rows, RS, W, F, list, s_hist, visits, work);
    }
}

// ---------------------------------------------------------------------------
// the persistent kernel
// ---------------------------------------------------------------------------
enum Mode { MODE_ORIENT = 0, MODE_PIVOT = 1, MODE_EXTRACT = 2 };

template <int BLOCK, int MODE>
__global__ void __launch_bounds__(BLOCK) k_count(CountParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_next, s_piv0, s_cnt, s_task;
    __shared__ int s_warp[BLOCK / 32];
    __shared__ ull s_key[BLOCK / 32];
    __shared__ ull s_red[4 * (BLOCK / 32)];
    const int tid = threadIdx.x;
    // layout: [hist u64][l2g i32 dcap][rows u32][work area]
    int hist_cells = MODE == MODE_PIVOT ? p.sh_hl * (p.sh_hl + 1) / 2 : 0;
    ull *s_hist = reinterpret_cast<ull *>(smem);
    int32_t *l2g = reinterpret_cast<int32_t *>(smem + 8 * hist_cells);
    uint32_t *area = reinterpret_cast<uint32_t *>(l2g + p.dcap);
    uint32_t *rows;
    if (p.rows_in_smem) {
        rows = area;
        area += int64_t(p.dcap) * row_stride(p.wcap);
    } else {
        rows = p.rows_global + int64_t(blockIdx.x) * p.rows_slot;
    }
    for (int i = tid; i < hist_cells; i += BLOCK) s_hist[i] = 0;
    ull acc = 0, visits = 0, tasks = 0, work = 0, bytes = 0;
    const bool directed = MODE == MODE_ORIENT || (MODE == MODE_EXTRACT && p.directed_out);
    const int t = p.t;
    for (;;) {
        __syncthreads();
        if (tid == 0) {
            ull i = p.given_rows ? (blockIdx.x == 0 ? atomicAdd(p.task_counter, 1ull) : ~0ull)
                                 : atomicAdd(p.task_counter, 1ull);
            s_task = i < ull(p.n_tasks) ? int(i) : -1;
            s_next = 0;
        }
        __syncthreads();
        if (s_task < 0) break;
        int d;
        if (p.given_rows) {
            d = load_given<BLOCK>(p, rows);
        } else {
            const int32_t task = p.tasks[s_task];
            // int32 scratch for the edge scheme lives in the work area
            const bool need_rows = MODE == MODE_EXTRACT || MODE == MODE_PIVOT || t >= 2;
            d = build_task<BLOCK>(p, task, l2g, rows, reinterpret_cast<int32_t *>(area), need_rows,
                                  directed, &s_cnt, s_warp, bytes);
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
        if (MODE == MODE_PIVOT && p.all_k) {
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
        if (MODE == MODE_ORIENT) {
            orient_task<BLOCK>(p, rows, d, area, &s_next, acc, visits, work);
        } else {
            pivot_task<BLOCK>(p, rows, d, area, reinterpret_cast<int *>(
                                  area + 2 * ((d + 31) >> 5) +
                                  (BLOCK / 32) * p.pv_smem_frames * pv_frame_words((d + 31) >> 5)),
                              s_hist, &s_next, &s_piv0, s_key, visits, work);
        }
    }
    __syncthreads();
    if (MODE == MODE_PIVOT) {
        for (int i = tid; i < hist_cells; i += BLOCK) {
            ull x = s_hist[i];
            if (x) {
                // triangular index -> (len, np)
                int len = int((sqrtf(8.0f * i + 1.0f) - 1.0f) * 0.5f);
                while (len * (len + 1) / 2 > i) --len;
                while ((len + 1) * (len + 2) / 2 <= i) ++len;
                int np = i - len * (len + 1) / 2;
                atomicAdd(&p.hist[int64_t(len) * p.hist_dim + np], x);
            }
        }
    }
    if (MODE != MODE_EXTRACT) flush_block<BLOCK>(p, acc, visits, tasks, work, bytes, s_red);
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
                              int min_d, uint8_t *__restrict__ keep, uint32_t *__restrict__ key) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
         e += int64_t(gridDim.x) * blockDim.x) {
        int32_t u = ocoo[e], v = ocol[e];
        int64_t du = orow[u + 1] - orow[u], dv = orow[v + 1] - orow[v];
        int64_t b = du < dv ? du : dv;  // |N+(u) ∩ N+(v)| <= min
        keep[e] = e >= lo && e < hi && b >= min_d;
        key[e] = uint32_t(du * dv > 0xffffffffll ? 0xffffffffll : du * dv);
    }
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

struct DevBuf {
    void *p = nullptr;
    DevBuf() = default;
    explicit DevBuf(size_t bytes) { p = kc_alloc<uint8_t>(bytes); }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
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
int64_t build_tasks(kc_graph *g, int scheme, int64_t lo, int64_t hi, int min_d, DevBuf &out) {
    const int64_t N = scheme == KC_SCHEME_EDGE ? g->m_dir : g->n;
    if (N == 0) return 0;
    DevBuf keep(N), key(4 * N), key2(4 * N), ids(4 * N), ids2(4 * N), cnt(8);
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
            g->orow_ptr, g->ocoo, g->ocol, N, lo, hi, min_d, keep.as<uint8_t>(),
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
    }
    KC_CUDA(cudaStreamSynchronize(g->stream));
    return n_sel;
}

constexpr int kBlock = 256;
constexpr int kSmidSlots = 1024;  // %smid can exceed the SM count
constexpr int kSmemMax = 220 * 1024;

struct Plan {
    size_t smem = 0;
    int blocks = 0;
};

size_t orient_stack_words(int t, int wcap, int group_size) {
    const int frames = t - 2 > 0 ? t - 2 : 0;
    if (frames == 0) return 32;
    size_t best = 0;
    for (int W = 1; W <= wcap; ++W) {
        int G = group_size > 0 ? group_size : auto_group(W);
        size_t need = size_t(kBlock / G) * group_stride(frames, W, G);
        best = need > best ? need : best;
    }
    return best;
}

template <int MODE>
void launch(kc_graph *g, CountParams &p, int grid_override = 0) {
    const int NW = kBlock / 32;
    size_t hist_bytes = MODE == MODE_PIVOT ? 8 * size_t(p.sh_hl) * (p.sh_hl + 1) / 2 : 0;
    size_t l2g_bytes = 4 * size_t(p.dcap > 0 ? p.dcap : 1);
    size_t rows_words = size_t(p.dcap) * row_stride(p.wcap);
    size_t work_words = 0;
    if (MODE == MODE_ORIENT) {
        work_words = orient_stack_words(p.t, p.wcap, p.group_size);
    } else if (MODE == MODE_PIVOT) {
        const int fw = pv_frame_words(p.wcap);
        // root (2W) + per-warp frames + per-warp candidate lists
        work_words = 2 * p.wcap + size_t(NW) * p.pv_smem_frames * fw + size_t(NW) * p.dcap;
    }
    if (p.scheme == KC_SCHEME_EDGE) work_words = std::max(work_words, size_t(p.dcap));
    size_t base = hist_bytes + l2g_bytes + 4 * work_words + 64;
    p.rows_in_smem = base + 4 * rows_words <= size_t(kSmemMax);
    size_t smem = base + (p.rows_in_smem ? 4 * rows_words : 0);
    KC_REQUIRE(smem <= size_t(kSmemMax), KC_ENOMEM, "per-task scratch exceeds shared memory");
    auto kern = k_count<kBlock, MODE>;
    KC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int per_sm = 0;
    KC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem));
    KC_REQUIRE(per_sm > 0, KC_ECUDA, "count kernel cannot be resident");
    int grid = grid_override > 0 ? grid_override : per_sm * g->num_sms;
    if (p.n_tasks > 0 && int64_t(grid) > p.n_tasks && !grid_override) grid = int(p.n_tasks);
    if (grid < 1) grid = 1;
    DevBuf rows_g, pv_g;
    if (!p.rows_in_smem) {
        p.rows_slot = int64_t(rows_words);
        new (&rows_g) DevBuf(4 * rows_words * size_t(grid));
        p.rows_global = rows_g.as<uint32_t>();
    }
    if (MODE == MODE_PIVOT) {
        const int fw = pv_frame_words(p.wcap);
        int64_t deep = int64_t(p.dcap) + 2 - p.pv_smem_frames;
        if (deep < 1) deep = 1;
        p.pv_slot = deep * fw;
        new (&pv_g) DevBuf(4 * size_t(p.pv_slot) * size_t(grid) * NW);
        p.pv_global = pv_g.as<uint32_t>();
    }
    kern<<<grid, kBlock, smem, g->stream>>>(p);
    KC_CUDA(cudaGetLastError());
    KC_CUDA(cudaStreamSynchronize(g->stream));
}

}  // namespace

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
    const int64_t L = g->d_max + 2;
    memset(raw, 0, sizeof(*raw));
    raw->hist_dim = pivot ? L : 0;
    if (pivot) {
        KC_REQUIRE(hist && hist_cap >= L * L, KC_EINVAL, "histogram buffer too small");
        memset(hist, 0, sizeof(uint64_t) * size_t(L * L));
    }
    if (visits_per_sm) memset(visits_per_sm, 0, sizeof(uint64_t) * size_t(n_sm));
    kc_device_guard guard(g->device);

    int64_t all = kc_task_count(g, a->scheme);
    int64_t lo = a->task_lo < 0 ? 0 : a->task_lo;
    int64_t hi = a->task_hi < 0 || a->task_hi > all ? all : a->task_hi;
    if (lo > hi) lo = hi;
    const int min_d = a->all_k ? 1 : (t > 1 ? t : 1);
    DevBuf tasks;
    const int64_t n_tasks = build_tasks(g, a->scheme, lo, hi, min_d, tasks);

    DevBuf outs(8 * (10 + size_t(kSmidSlots)));
    KC_CUDA(cudaMemsetAsync(outs.p, 0, 8 * (10 + size_t(kSmidSlots)), g->stream));
    DevBuf dhist(pivot ? 8 * size_t(L * L) : 8);
    if (pivot) KC_CUDA(cudaMemsetAsync(dhist.p, 0, 8 * size_t(L * L), g->stream));

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
    p.group_size = gs;
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

    cudaEvent_t e0, e1;
    KC_CUDA(cudaEventCreate(&e0));
    KC_CUDA(cudaEventCreate(&e1));
    KC_CUDA(cudaEventRecord(e0, g->stream));
    if (n_tasks > 0) {
        if (pivot) {
            p.pv_smem_frames = 8;
            launch<MODE_PIVOT>(g, p);
        } else {
            p.stack_words = int(orient_stack_words(t, p.wcap, gs));
            launch<MODE_ORIENT>(g, p);
        }
    }
    KC_CUDA(cudaEventRecord(e1, g->stream));
    KC_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    KC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);

    std::vector<ull> h(10 + size_t(kSmidSlots));
    KC_CUDA(cudaMemcpy(h.data(), outs.p, 8 * h.size(), cudaMemcpyDeviceToHost));
    raw->word_ops = h[8 + kSmidSlots];
    raw->extract_bytes = h[9 + kSmidSlots];
    for (int i = 0; i < 4; ++i) raw->limbs[i] = h[1 + i];
    raw->visits = h[5];
    raw->tasks_run = h[6];
    raw->count_ms = ms;
    if (visits_per_sm)
        for (int i = 0; i < n_sm && i < kSmidSlots; ++i) visits_per_sm[i] = h[8 + i];
    if (pivot) KC_CUDA(cudaMemcpy(hist, dhist.p, 8 * size_t(L * L), cudaMemcpyDeviceToHost));
}

void kc_do_extract(kc_graph *g, int scheme, int64_t task, int directed, int64_t *l2g,
                   uint64_t *words, int64_t cap, int64_t wpr_cap, int64_t *d_out) {
    KC_REQUIRE(g->oriented, KC_EINVAL, "graph is not oriented");
    const int64_t N = scheme == KC_SCHEME_EDGE ? g->m_dir : g->n;
    KC_REQUIRE(task >= 0 && task < N, KC_EINVAL, "task out of range");
    kc_device_guard guard(g->device);
    const int dcap = int(std::max<int64_t>(g->d_max, 1));
    const int wcap = (dcap + 31) / 32;
    DevBuf tk(4), rows(4 * size_t(dcap) * wcap), l(4 * size_t(dcap)), dd(4), outs(64);
    int32_t t32 = int32_t(task);
    KC_CUDA(cudaMemcpy(tk.p, &t32, 4, cudaMemcpyHostToDevice));
    KC_CUDA(cudaMemset(outs.p, 0, 64));
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
    launch<MODE_EXTRACT>(g, p, 1);
    int d = 0;
    KC_CUDA(cudaMemcpy(&d, dd.p, 4, cudaMemcpyDeviceToHost));
    KC_REQUIRE(d <= cap, KC_EINVAL, "scratch BitGraph too small for this task");
    const int W = (d + 31) / 32;
    const int64_t wpr = (d + 63) / 64;
    KC_REQUIRE(wpr <= wpr_cap || d == 0, KC_EINVAL, "words_per_row capacity too small");
    std::vector<int32_t> hl(d > 0 ? d : 1);
    std::vector<uint32_t> hr(size_t(d) * W + 1);
    if (d) {
        KC_CUDA(cudaMemcpy(hl.data(), l.p, 4 * size_t(d), cudaMemcpyDeviceToHost));
        KC_CUDA(cudaMemcpy(hr.data(), rows.p, 4 * size_t(d) * W, cudaMemcpyDeviceToHost));
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
    KC_CUDA(cudaStreamCreateWithFlags(&tmpg.stream, cudaStreamNonBlocking));
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
            p.pv_smem_frames = 8;
            launch<MODE_PIVOT>(&tmpg, p, 1);
        } else {
            p.stack_words = int(orient_stack_words(t, W, 0));
            launch<MODE_ORIENT>(&tmpg, p, 1);
        }
    } catch (...) {
        cudaStreamDestroy(tmpg.stream);
        throw;
    }
    std::vector<ull> h(8);
    KC_CUDA(cudaMemcpy(h.data(), outs.p, 64, cudaMemcpyDeviceToHost));
    cudaStreamDestroy(tmpg.stream);
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
__global__ void k_find_pivot(const uint32_t *rows, int d, const uint32_t *cand, int *out) {
    __shared__ int list[4096];
    const int W = (d + 31) >> 5;
    ull work = 0;
    int pv = warp_select_pivot(rows, W, W, cand, list, work);
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
    k_find_pivot<<<1, 32>>>(dr.as<uint32_t>(), d, dc.as<uint32_t>(), dout.as<int>());
    KC_CUDA(cudaGetLastError());
    int pv = 0;
    KC_CUDA(cudaMemcpy(&pv, dout.p, 4, cudaMemcpyDeviceToHost));
    *pivot = pv;
    for (int64_t w = 0; w < wpr; ++w) pruned[w] = cand64[w] & ~rows64[pv * wpr + w];
}
