/*
 * kc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, CPU restatement of the reference k-clique counting path
 * (arxiv/paper_2104_13209, package `kcliques` 0.1.0 under /root/reference/pkg).
 * It is the parity checker for the CUDA product in paper_2104_13209_b200/ and
 * the CPU baseline leg of bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline / --impl reference) may load it.  The product path
 * never links or calls it.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/pkg/src/kcliques/).
 *
 * Pinning: tests/test_oracle_golden.py checks this file against
 *   - the known answers in the reference's own tests (closed forms, K75 k=37,
 *     K140 overflow, C(131,65)/C(132,66), zero cases), and
 *   - tests/golden/*.json, produced by tests/golden/make_golden.py which runs
 *     the reference package itself (counts, visits, ranks, d_max, bit matrices).
 *
 * Word layout is the reference's: uint64 words, LSB-first
 * (_bitops.py:1-5), local index i at bit i%64 of word i/64.
 */
#define _POSIX_C_SOURCE 200809L
#include <pthread.h>
#include <time.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef uint64_t u64;

#define OC_OK 0
#define OC_EINVAL 1
#define OC_EOVERFLOW 3
#define OC_ENOMEM 5

/* ------------------------------------------------------------------ */
/* word primitives  (_bitops.py:20-73, :116-126)                       */
/* ------------------------------------------------------------------ */
static inline u64 popcount64(u64 x) { return (u64)__builtin_popcountll(x); }
static inline u64 ctz64(u64 x) { return x ? (u64)__builtin_ctzll(x) : 64; }

/* _bitops.py:61-73 binary search in the sorted slice col[lo:hi] */
static inline int csr_contains(const int32_t *col, int64_t lo, int64_t hi, int64_t x) {
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        int64_t c = col[mid];
        if (c < x) lo = mid + 1;
        else if (c > x) hi = mid;
        else return 1;
    }
    return 0;
}

/* _bitops.py:76-86 : u64 amount into a 128-bit accumulator + overflow flag */
static inline void acc_add(u64 *out, u64 add_lo) {
    u64 lo = out[0] + add_lo;
    if (lo < out[0]) {
        u64 hi = out[1] + 1;
        if (hi == 0) out[3] = 1;
        out[1] = hi;
    }
    out[0] = lo;
}

/* _bitops.py:89-99 */
static inline void acc_add128(u64 *out, u64 add_lo, u64 add_hi) {
    u64 lo = out[0] + add_lo;
    u64 carry = lo < out[0] ? 1 : 0;
    u64 mid = out[1] + add_hi;
    int wrapped = mid < out[1];
    u64 hi = mid + carry;
    if (wrapped || hi < mid) out[3] = 1;
    out[0] = lo;
    out[1] = hi;
}

/* _bitops.py:102-113 */
static inline void slot_add128(u64 *lo_arr, u64 *hi_arr, int64_t i, u64 add_lo, u64 add_hi,
                               u64 *meta) {
    u64 lo = lo_arr[i] + add_lo;
    u64 carry = lo < lo_arr[i] ? 1 : 0;
    u64 mid = hi_arr[i] + add_hi;
    int wrapped = mid < hi_arr[i];
    u64 hi = mid + carry;
    if (wrapped || hi < mid) meta[1] = 1;
    lo_arr[i] = lo;
    hi_arr[i] = hi;
}

/* _bitops.py:116-126 */
static inline void fill_all_ones(u64 *row, int64_t count, int64_t wpr) {
    for (int64_t w = 0; w < wpr; w++) {
        int64_t lo_bit = w << 6;
        if (lo_bit + 64 <= count) row[w] = ~(u64)0;
        else if (lo_bit < count) row[w] = (((u64)1) << (count - lo_bit)) - 1;
        else row[w] = 0;
    }
}

/* ------------------------------------------------------------------ */
/* CSR builder  (graph.py:162-200)                                     */
/* ------------------------------------------------------------------ */
static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}
static int cmp_u64(const void *a, const void *b) {
    u64 x = *(const u64 *)a, y = *(const u64 *)b;
    return (x > y) - (x < y);
}

/* graph.py:93-109 (load_edge_list, after parsing): drop self-loops (tally them,
 * keep their ids unique ascending), orient each pair (min, max), lexsort,
 * drop repeats (tally them).  pairs_out: int64[2*m_raw]; loop_ids: int64[m_raw];
 * counts[4] = {m_out, n_loop_ids, n_self_loops, n_duplicates}. */
static int cmp_pair(const void *a, const void *b) {
    const int64_t *x = (const int64_t *)a, *y = (const int64_t *)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    return (x[1] > y[1]) - (x[1] < y[1]);
}

int oc_normalize_edges(const int64_t *raw, int64_t m_raw, int64_t *pairs_out, int64_t *loop_ids,
                       int64_t *counts) {
    int64_t n_self = 0, n_rest = 0;
    for (int64_t i = 0; i < m_raw; ++i) {
        int64_t u = raw[2 * i], v = raw[2 * i + 1];
        if (u == v) { /* loops = u == v; loop_ids = unique(u[loops])   :96-98 */
            loop_ids[n_self++] = u;
            continue;
        }
        pairs_out[2 * n_rest] = u < v ? u : v; /* lo = minimum, hi = maximum :99-100 */
        pairs_out[2 * n_rest + 1] = u < v ? v : u;
        ++n_rest;
    }
    qsort(loop_ids, (size_t)n_self, sizeof(int64_t), cmp_i64);
    int64_t n_loop_u = 0;
    for (int64_t i = 0; i < n_self; ++i)
        if (i == 0 || loop_ids[i] != loop_ids[i - 1]) loop_ids[n_loop_u++] = loop_ids[i];
    qsort(pairs_out, (size_t)n_rest, 2 * sizeof(int64_t), cmp_pair); /* lexsort :101-102 */
    int64_t n_keep = 0;
    for (int64_t i = 0; i < n_rest; ++i) { /* keep[1:] = differs from previous :103-105 */
        if (i && pairs_out[2 * i] == pairs_out[2 * i - 2] &&
            pairs_out[2 * i + 1] == pairs_out[2 * i - 1])
            continue;
        pairs_out[2 * n_keep] = pairs_out[2 * i];
        pairs_out[2 * n_keep + 1] = pairs_out[2 * i + 1];
        ++n_keep;
    }
    counts[0] = n_keep;
    counts[1] = n_loop_u;
    counts[2] = n_self;
    counts[3] = n_rest - n_keep;
    return 0;
}

/* graph.py:177-181: ids = union1d(pairs.ravel(), extra) (sorted unique).
 * ids_out must hold 2*m + n_extra entries. */
int oc_compact_ids(const int64_t *pairs, int64_t m, const int64_t *extra, int64_t n_extra,
                   int64_t *ids_out, int64_t *n_out) {
    int64_t tot = 2 * m + n_extra;
    for (int64_t i = 0; i < 2 * m; i++) ids_out[i] = pairs[i];
    for (int64_t i = 0; i < n_extra; i++) ids_out[2 * m + i] = extra[i];
    qsort(ids_out, (size_t)tot, sizeof(int64_t), cmp_i64);
    int64_t n = 0;
    for (int64_t i = 0; i < tot; i++)
        if (n == 0 || ids_out[n - 1] != ids_out[i]) ids_out[n++] = ids_out[i];
    *n_out = n;
    return OC_OK;
}

static int64_t lower_bound_i64(const int64_t *a, int64_t n, int64_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* graph.py:190-200: searchsorted ids, symmetrize, lexsort (src,dst),
 * bincount+cumsum row_ptr.  row_ptr int64[n+1], col/coo_src int32[2m]. */
int oc_build_csr(const int64_t *pairs, int64_t m, const int64_t *ids, int64_t n,
                 int64_t *row_ptr, int32_t *col, int32_t *coo_src) {
    u64 *keys = (u64 *)malloc(sizeof(u64) * (size_t)(2 * m + 1));
    if (!keys) return OC_ENOMEM;
    for (int64_t e = 0; e < m; e++) {
        u64 cu = (u64)lower_bound_i64(ids, n, pairs[2 * e]);
        u64 cv = (u64)lower_bound_i64(ids, n, pairs[2 * e + 1]);
        keys[e] = (cu << 32) | cv;
        keys[m + e] = (cv << 32) | cu;
    }
    qsort(keys, (size_t)(2 * m), sizeof(u64), cmp_u64);
    for (int64_t v = 0; v <= n; v++) row_ptr[v] = 0;
    for (int64_t i = 0; i < 2 * m; i++) {
        coo_src[i] = (int32_t)(keys[i] >> 32);
        col[i] = (int32_t)(keys[i] & 0xffffffffu);
        row_ptr[coo_src[i] + 1]++;
    }
    for (int64_t v = 0; v < n; v++) row_ptr[v + 1] += row_ptr[v];
    free(keys);
    return OC_OK;
}

/* ------------------------------------------------------------------ */
/* Ranking  (orientation.py:48-135)                                    */
/* ------------------------------------------------------------------ */

/* orientation.py:124-128: lexsort((arange(n), degrees)); rank = position */
int oc_rank_degree(const int64_t *row_ptr, int64_t n, int32_t *rank) {
    u64 *keys = (u64 *)malloc(sizeof(u64) * (size_t)(n + 1));
    if (!keys) return OC_ENOMEM;
    for (int64_t v = 0; v < n; v++) keys[v] = ((u64)(row_ptr[v + 1] - row_ptr[v]) << 32) | (u64)v;
    qsort(keys, (size_t)n, sizeof(u64), cmp_u64);
    for (int64_t i = 0; i < n; i++) rank[keys[i] & 0xffffffffu] = (int32_t)i;
    free(keys);
    return OC_OK;
}

/* orientation.py:51-78 lazy-deletion binary min-heap */
static inline int64_t heap_push(u64 *heap, int64_t size, u64 key) {
    heap[size] = key;
    int64_t i = size;
    while (i > 0) {
        int64_t parent = (i - 1) >> 1;
        if (heap[parent] <= heap[i]) break;
        u64 tmp = heap[parent]; heap[parent] = heap[i]; heap[i] = tmp;
        i = parent;
    }
    return size + 1;
}
static inline int64_t heap_pop(u64 *heap, int64_t size) {
    size -= 1;
    heap[0] = heap[size];
    int64_t i = 0;
    for (;;) {
        int64_t left = 2 * i + 1;
        if (left >= size) break;
        int64_t small = left, right = left + 1;
        if (right < size && heap[right] < heap[left]) small = right;
        if (heap[i] <= heap[small]) break;
        u64 tmp = heap[i]; heap[i] = heap[small]; heap[small] = tmp;
        i = small;
    }
    return size;
}

/* orientation.py:81-113 (_peel) + :129-135: sequential min-residual-degree
 * removal, ties by lower id; rank = removal position. */
int oc_rank_degeneracy(const int64_t *row_ptr, const int32_t *col, int64_t n, int32_t *rank,
                       int64_t *degeneracy_out) {
    if (n == 0) { *degeneracy_out = 0; return OC_OK; }
    int64_t *deg = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    u64 *heap = (u64 *)malloc(sizeof(u64) * (size_t)(n + row_ptr[n] + 1));
    unsigned char *removed = (unsigned char *)calloc((size_t)n, 1);
    if (!deg || !heap || !removed) { free(deg); free(heap); free(removed); return OC_ENOMEM; }
    int64_t size = 0;
    for (int64_t v = 0; v < n; v++) {
        deg[v] = row_ptr[v + 1] - row_ptr[v];
        size = heap_push(heap, size, ((u64)deg[v] << 32) | (u64)v);
    }
    int64_t degeneracy = 0;
    for (int64_t pos = 0; pos < n; pos++) {
        int64_t v;
        for (;;) {
            u64 key = heap[0];
            v = (int64_t)(key & 0xffffffffu);
            int64_t key_deg = (int64_t)(key >> 32);
            size = heap_pop(heap, size);
            if (!removed[v] && key_deg == deg[v]) break;
        }
        removed[v] = 1;
        rank[v] = (int32_t)pos;
        if (deg[v] > degeneracy) degeneracy = deg[v];
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; e++) {
            int64_t w = col[e];
            if (!removed[w]) {
                deg[w] -= 1;
                size = heap_push(heap, size, ((u64)deg[w] << 32) | (u64)w);
            }
        }
    }
    *degeneracy_out = degeneracy;
    free(deg); free(heap); free(removed);
    return OC_OK;
}

/* orientation.py:139-153: keep e iff rank[src] < rank[dst]; segments keep
 * compact-id order.  Outputs sized by the caller: orow_ptr[n+1], ocol/ocoo[m]. */
int oc_orient(const int64_t *row_ptr, const int32_t *col, const int32_t *coo_src, int64_t n,
              const int32_t *rank, int64_t *orow_ptr, int32_t *ocol, int32_t *ocoo_src,
              int64_t *m_dir_out, int64_t *d_max_out) {
    int64_t two_m = row_ptr[n];
    int64_t k = 0;
    for (int64_t v = 0; v <= n; v++) orow_ptr[v] = 0;
    for (int64_t e = 0; e < two_m; e++) {
        if (rank[coo_src[e]] < rank[col[e]]) {
            ocol[k] = col[e];
            ocoo_src[k] = coo_src[e];
            orow_ptr[coo_src[e] + 1]++;
            k++;
        }
    }
    int64_t d_max = 0;
    for (int64_t v = 0; v < n; v++) {
        if (orow_ptr[v + 1] > d_max) d_max = orow_ptr[v + 1];
        orow_ptr[v + 1] += orow_ptr[v];
    }
    *m_dir_out = k;
    *d_max_out = d_max;
    return OC_OK;
}

/* ------------------------------------------------------------------ */
/* induced sub-graph  (bitgraph.py:59-111)                             */
/* ------------------------------------------------------------------ */

/* bitgraph.py:59-64 */
static int64_t locals_vertex(const int64_t *row_ptr, const int32_t *col, int64_t v, int64_t *l2g) {
    int64_t lo = row_ptr[v], d = row_ptr[v + 1] - lo;
    for (int64_t i = 0; i < d; i++) l2g[i] = col[lo + i];
    return d;
}

/* bitgraph.py:67-86: merge intersection of two ascending slices */
static int64_t locals_edge(const int64_t *row_ptr, const int32_t *col, int64_t u, int64_t v,
                           int64_t *l2g) {
    int64_t a = row_ptr[u], a_end = row_ptr[u + 1];
    int64_t b = row_ptr[v], b_end = row_ptr[v + 1];
    int64_t d = 0;
    while (a < a_end && b < b_end) {
        int32_t x = col[a], y = col[b];
        if (x == y) { l2g[d++] = x; a++; b++; }
        else if (x < y) a++;
        else b++;
    }
    return d;
}

/* bitgraph.py:89-111: one binary search per unordered local pair in the
 * rank-lower endpoint's out-slice. words is [d][wpr_stride]. */
static void fill_adjacency(const int64_t *row_ptr, const int32_t *col, const int32_t *rank,
                           const int64_t *l2g, int64_t d, u64 *words, int64_t wpr,
                           int64_t stride, int directed) {
    for (int64_t i = 0; i < d; i++)
        for (int64_t w = 0; w < wpr; w++) words[i * stride + w] = 0;
    for (int64_t i = 0; i < d; i++) {
        int64_t gi = l2g[i];
        for (int64_t j = i + 1; j < d; j++) {
            int64_t gj = l2g[j];
            if (rank[gi] < rank[gj]) {
                if (csr_contains(col, row_ptr[gi], row_ptr[gi + 1], gj)) {
                    words[i * stride + (j >> 6)] |= ((u64)1) << (j & 63);
                    if (!directed) words[j * stride + (i >> 6)] |= ((u64)1) << (i & 63);
                }
            } else {
                if (csr_contains(col, row_ptr[gj], row_ptr[gj + 1], gi)) {
                    words[j * stride + (i >> 6)] |= ((u64)1) << (i & 63);
                    if (!directed) words[i * stride + (j >> 6)] |= ((u64)1) << (j & 63);
                }
            }
        }
    }
}

/* bitgraph.py:125-152 single-task extraction (for the K4 parity tests).
 * scheme 0 = vertex (task = vertex id), 1 = edge (task = oriented edge id).
 * l2g int64[cap], words uint64[cap][ceil(cap/64)] with stride wpr_cap. */
int oc_extract(const int64_t *orow_ptr, const int32_t *ocol, const int32_t *ocoo_src,
               const int32_t *rank, int scheme, int64_t task, int directed, int64_t *l2g,
               u64 *words, int64_t wpr_cap, int64_t *d_out) {
    int64_t d = scheme == 0 ? locals_vertex(orow_ptr, ocol, task, l2g)
                            : locals_edge(orow_ptr, ocol, ocoo_src[task], ocol[task], l2g);
    int64_t wpr = (d + 63) >> 6;
    fill_adjacency(orow_ptr, ocol, rank, l2g, d, words, wpr, wpr_cap, directed);
    *d_out = d;
    return OC_OK;
}

/* ------------------------------------------------------------------ */
/* orient engine  (engine_orient.py:32-79)                             */
/* ------------------------------------------------------------------ */
/* stk is [depth][stride]; out = {lo, hi, visits, overflow} */
static void orient_count_into(const u64 *rows, int64_t stride, int64_t wpr, int64_t d, int64_t t,
                              u64 *stk, int64_t *cw, u64 *cb, u64 *out) {
    if (t <= 1) {
        if (t == 0) acc_add(out, 1);
        else if (t == 1) acc_add(out, (u64)d);
        return;
    }
    if (d == 0) return;
    fill_all_ones(stk, d, wpr);
    int64_t last = t - 2, s = 0;
    cw[0] = 0;
    cb[0] = stk[0];
    while (s >= 0) {
        u64 b = cb[s];
        if (b == 0) {
            int64_t w = cw[s] + 1;
            while (w < wpr && stk[s * stride + w] == 0) w++;
            if (w >= wpr) { s--; continue; }
            cw[s] = w;
            b = stk[s * stride + w];
        }
        int64_t v = (cw[s] << 6) + (int64_t)ctz64(b);
        cb[s] = b & (b - 1);
        out[2] += 1;
        const u64 *rv = rows + v * stride;
        if (s == last) {
            u64 c = 0;
            for (int64_t w = 0; w < wpr; w++) c += popcount64(stk[s * stride + w] & rv[w]);
            acc_add(out, c);
        } else {
            u64 nz = 0;
            for (int64_t w = 0; w < wpr; w++) {
                u64 x = stk[s * stride + w] & rv[w];
                stk[(s + 1) * stride + w] = x;
                nz |= x;
            }
            if (nz != 0) {
                s++;
                cw[s] = 0;
                cb[s] = stk[s * stride];
            }
        }
    }
}

/* ------------------------------------------------------------------ */
/* binomial table  (engine_pivot.py:41-65)                             */
/* ------------------------------------------------------------------ */
/* (N+1)x(N+1) tables; too_big where C(n,r) >= 2^128.  Pascal's rule with a
 * saturating flag is exact: C(n,r) >= both summands. */
int oc_binomial_table(int64_t n_max, u64 *lo, u64 *hi, unsigned char *too_big) {
    int64_t size = n_max + 1;
    u128 *prev = (u128 *)calloc((size_t)size + 1, sizeof(u128));
    u128 *cur = (u128 *)calloc((size_t)size + 1, sizeof(u128));
    unsigned char *pbig = (unsigned char *)calloc((size_t)size + 1, 1);
    unsigned char *cbig = (unsigned char *)calloc((size_t)size + 1, 1);
    if (!prev || !cur || !pbig || !cbig) { free(prev); free(cur); free(pbig); free(cbig); return OC_ENOMEM; }
    memset(lo, 0, sizeof(u64) * (size_t)(size * size));
    memset(hi, 0, sizeof(u64) * (size_t)(size * size));
    memset(too_big, 0, (size_t)(size * size));
    for (int64_t n = 0; n < size; n++) {
        for (int64_t r = 0; r <= n; r++) {
            if (r == 0 || r == n) { cur[r] = 1; cbig[r] = 0; }
            else {
                u128 a = prev[r - 1], b = prev[r];
                u128 s = a + b;
                cbig[r] = pbig[r - 1] || pbig[r] || s < a;
                cur[r] = cbig[r] ? 0 : s;
            }
            if (cbig[r]) too_big[n * size + r] = 1;
            else { lo[n * size + r] = (u64)cur[r]; hi[n * size + r] = (u64)(cur[r] >> 64); }
        }
        u128 *tp = prev; prev = cur; cur = tp;
        unsigned char *tb = pbig; pbig = cbig; cbig = tb;
    }
    free(prev); free(cur); free(pbig); free(cbig);
    return OC_OK;
}

/* ------------------------------------------------------------------ */
/* pivot engine  (engine_pivot.py:82-233)                              */
/* ------------------------------------------------------------------ */
/* engine_pivot.py:82-101: argmax |cand & row(v)|, lowest id wins ties */
static int64_t select_pivot(const u64 *rows, int64_t stride, int64_t wpr, const u64 *cand,
                            u64 *pruned) {
    int64_t best = -1, best_cov = -1;
    for (int64_t w0 = 0; w0 < wpr; w0++) {
        u64 b = cand[w0];
        while (b) {
            int64_t v = (w0 << 6) + (int64_t)ctz64(b);
            b &= b - 1;
            int64_t cov = 0;
            for (int64_t w = 0; w < wpr; w++) cov += (int64_t)popcount64(cand[w] & rows[v * stride + w]);
            if (cov > best_cov) { best_cov = cov; best = v; }
        }
    }
    for (int64_t w = 0; w < wpr; w++) pruned[w] = cand[w] & ~rows[best * stride + w];
    return best;
}

int oc_find_pivot(const u64 *rows, int64_t stride, int64_t wpr, const u64 *cand, u64 *pruned,
                  int64_t *pivot_out) {
    *pivot_out = select_pivot(rows, stride, wpr, cand, pruned);
    return OC_OK;
}

typedef struct {
    u64 *cand, *pruned;  /* [depth][stride] */
    int64_t *piv, *npv, *cw;
    u64 *cb;
} pivot_scratch;

/* engine_pivot.py:117-178 (per-t) and :181-233 (all-t).  all_t selects the
 * variant; tb = table (size x size).  out = {lo,hi,visits,overflow};
 * all-t: slot_lo/slot_hi[d+2], meta = {visits, overflow}. */
static void pivot_walk(const u64 *rows, int64_t stride, int64_t wpr, int64_t d, int64_t t,
                       int all_t, pivot_scratch *sc, const u64 *blo, const u64 *bhi,
                       const unsigned char *bbig, int64_t bsize, u64 *out, u64 *slot_lo,
                       u64 *slot_hi, u64 *meta) {
    if (!all_t && t <= 1) {
        if (t == 0) acc_add(out, 1);
        else if (t == 1) acc_add(out, (u64)d);
        return;
    }
    if (d == 0) return;
    u64 *C = sc->cand, *P = sc->pruned;
    fill_all_ones(C, d, wpr);
    sc->piv[0] = select_pivot(rows, stride, wpr, C, P);
    sc->npv[0] = 0;
    int64_t s = 0;
    sc->cw[0] = 0;
    sc->cb[0] = P[0];
    while (s >= 0) {
        u64 b = sc->cb[s];
        if (b == 0) {
            int64_t w = sc->cw[s] + 1;
            while (w < wpr && P[s * stride + w] == 0) w++;
            if (w >= wpr) { s--; continue; }
            sc->cw[s] = w;
            b = P[s * stride + w];
        }
        int64_t v = (sc->cw[s] << 6) + (int64_t)ctz64(b);
        sc->cb[s] = b & (b - 1);
        int64_t np2 = sc->npv[s] + (v == sc->piv[s] ? 1 : 0);
        if (!all_t) {
            if (s + 1 - t > np2) continue;
            out[2] += 1;
        } else {
            meta[0] += 1;
        }
        int64_t vq = v >> 6;
        u64 vr = (u64)(v & 63);
        u64 nz = 0;
        for (int64_t w = 0; w < wpr; w++) {
            u64 x = C[s * stride + w] & rows[v * stride + w];
            if (w < vq) x &= ~P[s * stride + w];
            else if (w == vq) x &= ~(P[s * stride + w] & ((((u64)1) << vr) - 1));
            C[(s + 1) * stride + w] = x;
            nz |= x;
        }
        if (nz != 0) {
            s++;
            sc->npv[s] = np2;
            sc->piv[s] = select_pivot(rows, stride, wpr, C + s * stride, P + s * stride);
            sc->cw[s] = 0;
            sc->cb[s] = P[s * stride];
        } else if (!all_t) {
            if (s + 1 >= t) {
                int64_t r = s + 1 - t;
                if (bbig[np2 * bsize + r]) out[3] = 1;
                else acc_add128(out, blo[np2 * bsize + r], bhi[np2 * bsize + r]);
            }
        } else {
            for (int64_t r = 0; r <= np2; r++) {
                int64_t tt = s + 1 - r;
                if (bbig[np2 * bsize + r]) meta[1] = 1;
                else slot_add128(slot_lo, slot_hi, tt, blo[np2 * bsize + r], bhi[np2 * bsize + r], meta);
            }
        }
    }
}

/* ------------------------------------------------------------------ */
/* single bit-matrix engines (engine_orient.py:91-114, engine_pivot.py:248-308) */
/* ------------------------------------------------------------------ */
/* rows: [d][stride] u64.  algo 0 = orient, 1 = pivot, 2 = pivot all-t.
 * out4 = {lo, hi, visits, overflow}; for all-t, slot_lo/hi[d+2]. */
int oc_count_bitgraph(const u64 *rows, int64_t stride, int64_t d, int64_t t, int algo,
                      u64 *out4, u64 *slot_lo, u64 *slot_hi) {
    int64_t wpr = (d + 63) >> 6;
    int64_t wcap = stride > 0 ? stride : 1;
    memset(out4, 0, 4 * sizeof(u64));
    if (algo == 0) {
        int64_t depth = t < 2 ? 1 : (t - 1 < d + 1 ? t - 1 : d + 1);
        if (depth < 1) depth = 1;
        u64 *stk = (u64 *)calloc((size_t)(depth * wcap), sizeof(u64));
        int64_t *cw = (int64_t *)calloc((size_t)depth, sizeof(int64_t));
        u64 *cb = (u64 *)calloc((size_t)depth, sizeof(u64));
        orient_count_into(rows, wcap, wpr, d, t, stk, cw, cb, out4);
        free(stk); free(cw); free(cb);
        return out4[3] ? OC_EOVERFLOW : OC_OK;
    }
    int64_t bsize = (d > 1 ? d : 1) + 1;
    u64 *blo = (u64 *)malloc(sizeof(u64) * (size_t)(bsize * bsize));
    u64 *bhi = (u64 *)malloc(sizeof(u64) * (size_t)(bsize * bsize));
    unsigned char *bbig = (unsigned char *)malloc((size_t)(bsize * bsize));
    oc_binomial_table(bsize - 1, blo, bhi, bbig);
    int64_t depth = d + 1;
    pivot_scratch sc;
    sc.cand = (u64 *)calloc((size_t)(depth * wcap), sizeof(u64));
    sc.pruned = (u64 *)calloc((size_t)(depth * wcap), sizeof(u64));
    sc.piv = (int64_t *)calloc((size_t)depth, sizeof(int64_t));
    sc.npv = (int64_t *)calloc((size_t)depth, sizeof(int64_t));
    sc.cw = (int64_t *)calloc((size_t)depth, sizeof(int64_t));
    sc.cb = (u64 *)calloc((size_t)depth, sizeof(u64));
    u64 meta[2] = {0, 0};
    if (algo == 1) {
        pivot_walk(rows, wcap, wpr, d, t, 0, &sc, blo, bhi, bbig, bsize, out4, NULL, NULL, NULL);
    } else {
        memset(slot_lo, 0, sizeof(u64) * (size_t)(d + 2));
        memset(slot_hi, 0, sizeof(u64) * (size_t)(d + 2));
        pivot_walk(rows, wcap, wpr, d, 0, 1, &sc, blo, bhi, bbig, bsize, NULL, slot_lo, slot_hi, meta);
        out4[2] = meta[0];
        out4[3] = meta[1];
        if (d == 0) slot_lo[0] = 1; /* engine_pivot.py:306-307 */
    }
    free(sc.cand); free(sc.pruned); free(sc.piv); free(sc.npv); free(sc.cw); free(sc.cb);
    free(blo); free(bhi); free(bbig);
    return out4[3] ? OC_EOVERFLOW : OC_OK;
}

/* ------------------------------------------------------------------ */
/* worker pool  (scheduler.py:141-185, :211-293)                       */
/* ------------------------------------------------------------------ */
typedef struct {
    const int64_t *row_ptr;
    const int32_t *col, *rank, *coo_src;
    const int64_t *tasks;
    int64_t n_tasks, d_max, t;
    int edge, algo, all_k;
    const u64 *blo, *bhi;
    const unsigned char *bbig;
    int64_t bsize;
    int64_t *cursor;
    /* per worker */
    u64 out[4];
    u64 *slot_lo, *slot_hi;
    u64 meta[2];
    double busy_s; /* this thread's CPU time */
} worker_arg;

static void *worker_loop(void *p) {
    worker_arg *a = (worker_arg *)p;
    {
        struct timespec ts;
        clock_gettime(CLOCK_THREAD_CPUTIME_ID, &ts);
        a->busy_s = (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
    }
    int64_t cap = a->d_max > 1 ? a->d_max : 1;
    int64_t wcap = (cap + 63) >> 6;
    int64_t *l2g = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
    u64 *words = (u64 *)calloc((size_t)(cap * wcap), sizeof(u64));
    int pivot = a->algo != 0;
    int64_t depth = pivot ? cap + 1 : (a->t < 2 ? 1 : (a->t - 1 < cap + 1 ? a->t - 1 : cap + 1));
    if (depth < 1) depth = 1;
    u64 *stk = (u64 *)calloc((size_t)(depth * wcap), sizeof(u64));
    int64_t *cw = (int64_t *)calloc((size_t)depth, sizeof(int64_t));
    u64 *cb = (u64 *)calloc((size_t)depth, sizeof(u64));
    pivot_scratch sc = {0};
    if (pivot) {
        sc.cand = stk;
        sc.pruned = (u64 *)calloc((size_t)(depth * wcap), sizeof(u64));
        sc.piv = (int64_t *)calloc((size_t)depth, sizeof(int64_t));
        sc.npv = (int64_t *)calloc((size_t)depth, sizeof(int64_t));
        sc.cw = cw;
        sc.cb = cb;
    }
    for (;;) {
        int64_t i = __atomic_fetch_add(a->cursor, 1, __ATOMIC_RELAXED); /* scheduler.py:147 */
        if (i >= a->n_tasks) break;
        int64_t task = a->tasks[i];
        int64_t d = a->edge ? locals_edge(a->row_ptr, a->col, a->coo_src[task], a->col[task], l2g)
                            : locals_vertex(a->row_ptr, a->col, task, l2g);
        if (a->all_k) {
            if (d == 0) continue; /* scheduler.py:180-181 */
        } else if (d < a->t) {
            continue; /* scheduler.py:155-156 */
        }
        int64_t wpr = (d + 63) >> 6;
        fill_adjacency(a->row_ptr, a->col, a->rank, l2g, d, words, wpr, wcap, !pivot);
        if (a->all_k)
            pivot_walk(words, wcap, wpr, d, 0, 1, &sc, a->blo, a->bhi, a->bbig, a->bsize, NULL,
                       a->slot_lo, a->slot_hi, a->meta);
        else if (pivot)
            pivot_walk(words, wcap, wpr, d, a->t, 0, &sc, a->blo, a->bhi, a->bbig, a->bsize,
                       a->out, NULL, NULL, NULL);
        else
            orient_count_into(words, wcap, wpr, d, a->t, stk, cw, cb, a->out);
    }
    free(l2g); free(words); free(stk); free(cw); free(cb);
    if (pivot) { free(sc.pruned); free(sc.piv); free(sc.npv); }
    struct timespec ts;
    clock_gettime(CLOCK_THREAD_CPUTIME_ID, &ts);
    a->busy_s = (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec - a->busy_s;
    return NULL;
}

/*
 * scheduler.py:211-293 over an oriented graph.
 *   algo: 0 orient, 1 pivot; edge: 0 vertex, 1 edge scheme; all_k needs pivot.
 *   t: target inside each task (k-1 vertex, k-2 edge); ignored for all_k.
 *   tasks: make_tasks (scheduler.py:89-95) order; [task_lo, task_hi) is the
 *   slice this call runs (the multi-rank shard).
 * Results:
 *   count_out[2] = 128-bit total (lo, hi); visits_per_worker[workers];
 *   flags_out[0] = any worker's 128-bit accumulator/binomial overflowed;
 *   flags_out[1] = the cross-worker sum itself exceeded 128 bits.
 *   all_k: slots_lo/hi[d_max+2] (sum over workers, same flags).
 */
static int run_list(const int64_t *orow_ptr, const int32_t *ocol, const int32_t *ocoo_src,
                    const int32_t *rank, int64_t d_max, int algo, int edge, int all_k, int64_t t,
                    const int64_t *tasks, int64_t n_list, int workers, u64 *count_out,
                    u64 *visits_per_worker, u64 *flags_out, u64 *slots_lo, u64 *slots_hi,
                    double *busy_s);

int oc_run_tasks(const int64_t *orow_ptr, const int32_t *ocol, const int32_t *ocoo_src,
                 const int32_t *rank, int64_t n, int64_t m_dir, int64_t d_max, int algo, int edge,
                 int all_k, int64_t t, int64_t task_lo, int64_t task_hi, int workers,
                 u64 *count_out, u64 *visits_per_worker, u64 *flags_out, u64 *slots_lo,
                 u64 *slots_hi) {
    if (workers < 1) return OC_EINVAL;
    int64_t n_all = 0;
    int64_t *tasks = (int64_t *)malloc(sizeof(int64_t) * (size_t)((edge ? m_dir : n) + 1));
    if (!tasks) return OC_ENOMEM;
    if (edge) {
        for (int64_t e = 0; e < m_dir; e++) tasks[n_all++] = e;
    } else {
        for (int64_t v = 0; v < n; v++)
            if (orow_ptr[v + 1] - orow_ptr[v] > 0) tasks[n_all++] = v;
    }
    if (task_lo < 0) task_lo = 0;
    if (task_hi > n_all || task_hi < 0) task_hi = n_all;
    if (task_lo > task_hi) task_lo = task_hi;
    int rc = run_list(orow_ptr, ocol, ocoo_src, rank, d_max, algo, edge, all_k, t,
                      tasks + task_lo, task_hi - task_lo, workers, count_out, visits_per_worker,
                      flags_out, slots_lo, slots_hi, NULL);
    free(tasks);
    return rc;
}

/* The same pool over an explicit list of task ids (vertex ids or oriented
 * edge ids) -- the CPU baseline's stratified sample.  busy_s (optional,
 * [workers]) receives each worker thread's CPU time. */
int oc_run_task_list(const int64_t *orow_ptr, const int32_t *ocol, const int32_t *ocoo_src,
                     const int32_t *rank, int64_t d_max, int algo, int edge, int all_k, int64_t t,
                     const int64_t *tasks, int64_t n_list, int workers, u64 *count_out,
                     u64 *visits_per_worker, u64 *flags_out, u64 *slots_lo, u64 *slots_hi,
                     double *busy_s) {
    if (workers < 1) return OC_EINVAL;
    return run_list(orow_ptr, ocol, ocoo_src, rank, d_max, algo, edge, all_k, t, tasks, n_list,
                    workers, count_out, visits_per_worker, flags_out, slots_lo, slots_hi, busy_s);
}

static int run_list(const int64_t *orow_ptr, const int32_t *ocol, const int32_t *ocoo_src,
                    const int32_t *rank, int64_t d_max, int algo, int edge, int all_k, int64_t t,
                    const int64_t *tasks, int64_t n_list, int workers, u64 *count_out,
                    u64 *visits_per_worker, u64 *flags_out, u64 *slots_lo, u64 *slots_hi,
                    double *busy_s) {
    int pivot = algo != 0 || all_k;
    int64_t bsize = 1;
    u64 *blo = NULL, *bhi = NULL;
    unsigned char *bbig = NULL;
    if (pivot) {
        bsize = d_max + 2; /* BinomialTable(og.d_max + 1), scheduler.py:216-218 */
        blo = (u64 *)malloc(sizeof(u64) * (size_t)(bsize * bsize));
        bhi = (u64 *)malloc(sizeof(u64) * (size_t)(bsize * bsize));
        bbig = (unsigned char *)malloc((size_t)(bsize * bsize));
        oc_binomial_table(bsize - 1, blo, bhi, bbig);
    }
    int64_t n_slots = (d_max > 1 ? d_max : 1) + 2;
    int64_t cursor = 0;
    worker_arg *args = (worker_arg *)calloc((size_t)workers, sizeof(worker_arg));
    pthread_t *th = (pthread_t *)calloc((size_t)workers, sizeof(pthread_t));
    for (int w = 0; w < workers; w++) {
        worker_arg *a = &args[w];
        a->row_ptr = orow_ptr; a->col = ocol; a->rank = rank; a->coo_src = ocoo_src;
        a->tasks = tasks; a->n_tasks = n_list;
        a->d_max = d_max; a->t = t; a->edge = edge; a->algo = pivot ? 1 : 0; a->all_k = all_k;
        a->blo = blo; a->bhi = bhi; a->bbig = bbig; a->bsize = bsize;
        a->cursor = &cursor;
        if (all_k) {
            a->slot_lo = (u64 *)calloc((size_t)n_slots, sizeof(u64));
            a->slot_hi = (u64 *)calloc((size_t)n_slots, sizeof(u64));
        }
    }
    if (workers == 1) worker_loop(&args[0]);
    else {
        for (int w = 0; w < workers; w++) pthread_create(&th[w], NULL, worker_loop, &args[w]);
        for (int w = 0; w < workers; w++) pthread_join(th[w], NULL);
    }
    u128 total = 0;
    int any_over = 0, sum_over = 0;
    if (all_k) {
        for (int64_t s = 0; s < n_slots; s++) {
            u128 acc = 0;
            for (int w = 0; w < workers; w++) {
                u128 x = ((u128)args[w].slot_hi[s] << 64) | args[w].slot_lo[s];
                u128 y = acc + x;
                if (y < acc) sum_over = 1;
                acc = y;
            }
            slots_lo[s] = (u64)acc;
            slots_hi[s] = (u64)(acc >> 64);
        }
        for (int w = 0; w < workers; w++) {
            visits_per_worker[w] = args[w].meta[0];
            if (args[w].meta[1]) any_over = 1;
        }
    } else {
        for (int w = 0; w < workers; w++) {
            u128 x = ((u128)args[w].out[1] << 64) | args[w].out[0];
            u128 y = total + x;
            if (y < total) sum_over = 1;
            total = y;
            visits_per_worker[w] = args[w].out[2];
            if (args[w].out[3]) any_over = 1;
        }
    }
    count_out[0] = (u64)total;
    count_out[1] = (u64)(total >> 64);
    flags_out[0] = (u64)any_over;
    flags_out[1] = (u64)sum_over;
    if (busy_s)
        for (int w = 0; w < workers; w++) busy_s[w] = args[w].busy_s;
    for (int w = 0; w < workers; w++) { free(args[w].slot_lo); free(args[w].slot_hi); }
    free(args); free(th); free(blo); free(bhi); free(bbig);
    return any_over ? OC_EOVERFLOW : OC_OK;
}

/* number of make_tasks entries (scheduler.py:89-95) */
int64_t oc_num_tasks(const int64_t *orow_ptr, int64_t n, int64_t m_dir, int edge) {
    if (edge) return m_dir;
    int64_t c = 0;
    for (int64_t v = 0; v < n; v++) c += orow_ptr[v + 1] - orow_ptr[v] > 0;
    return c;
}
