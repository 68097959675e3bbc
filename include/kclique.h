/*
 * kclique.h -- C ABI of the B200-native k-clique counter (libkc.so).
 *
 * This is the drop-in boundary for the reference's counting hot path
 * (arxiv/paper_2104_13209, package `kcliques`, paths relative to
 * /root/reference/pkg/src/kcliques/).  Plain C types only: pointers, sizes,
 * status codes.  Every device buffer is owned by the opaque kc_graph handle.
 *
 * Reference interfaces replaced (see INTEGRATION.md for the ctypes binding):
 *   kc_normalize_edges    <- graph.py:93-109       load_edge_list's normal form (loops, dedup)
 *   kc_graph_from_edges   <- graph.py:162-200      from_edges(edges) -> Graph
 *   kc_graph_from_raw_edges <- graph.py:203-209    read_graph: from_edges(load_edge_list(..)) after parsing
 *   kc_graph_from_csr     <- graph.py:112-131      Graph(n, m, row_ptr, col, coo_src, orig_ids)
 *   kc_orient             <- orientation.py:116-153 compute_rank(g, criterion) + orient(g, ranking)
 *   kc_count              <- scheduler.py:141-185  _worker_loop / _worker_loop_all + the
 *                            thread pool and reduction of scheduler.py:211-293
 *   kc_num_tasks, kc_task_costs, kc_shard_ranges <- scheduler.py:89-95 make_tasks (+ costs and
 *                            balanced root ranges for the multi-GPU shards)
 *   kc_extract            <- bitgraph.py:125-152   extract_vertex_induced / extract_edge_induced
 *   kc_count_bitgraph     <- engine_orient.py:91-114, engine_pivot.py:248-308
 *                            count_tcliques_orient / count_tcliques_pivot / ..._all_t
 *   kc_find_pivot         <- engine_pivot.py:104-114 find_pivot
 *
 * Status codes mirror the reference's exception classes:
 *   KC_OK 0, KC_EINVAL 1 (ValueError), KC_EOVERFLOW 3 (OverflowError),
 *   KC_ECUDA 4 (RuntimeError; message via kc_last_error()), KC_ENOMEM 5.
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry point returns KC_ECUDA.
 */
#ifndef KCLIQUE_H
#define KCLIQUE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KC_OK 0
#define KC_EINVAL 1
#define KC_EOVERFLOW 3
#define KC_ECUDA 4
#define KC_ENOMEM 5

#define KC_ABI_VERSION 2

/* orientation criteria (orientation.py:9 CRITERIA) */
#define KC_CRIT_DEGREE 0
#define KC_CRIT_DEGENERACY 1 /* the reference's sequential heap order (orientation.py:81-113),
                                rank for rank: core numbers by a bulk peel, then one heap run
                                per shell-internal component, merged (kc_peel.cu) */
#define KC_CRIT_GIVEN 2 /* use a caller-provided rank permutation */
#define KC_CRIT_DEGENERACY_EXACT 3 /* alias of KC_CRIT_DEGENERACY (round-1 name) */
#define KC_CRIT_DEGENERACY_BULK 4 /* the paper's bulk-synchronous peel order, rank = (round, id):
                                     a valid degeneracy order but not the heap's */

/* algorithms / schemes (scheduler.py:27-28) */
#define KC_ALGO_ORIENT 0
#define KC_ALGO_PIVOT 1
#define KC_SCHEME_VERTEX 0
#define KC_SCHEME_EDGE 1

typedef struct kc_graph kc_graph;

/* Library / device */
int kc_abi_version(void);
const char *kc_last_error(void);
/* number of visible CUDA devices (0 when none); never fails */
int kc_device_count(void);
/* number of SMs of the device the graph lives on (load-stats width) */
int kc_num_sms(int device);

/* ---- edge-list normal form (graph.py:93-109) ------------------------ */
/* raw: int64[2*m_raw] host pairs (row-major, ids >= 0, any order, loops and
 * repeats allowed).  On the device: drop and tally self-loops (their ids,
 * unique ascending, go to loop_ids_out), orient each pair (min, max), sort
 * lexicographically, drop and tally repeats.  pairs_out: host int64[2*m_raw]
 * capacity, receives m_out rows; loop_ids_out: host int64[m_raw] capacity.
 * ms: device time (optional).  Negative ids -> KC_EINVAL. */
int kc_normalize_edges(int device, const int64_t *raw, int64_t m_raw, int64_t *pairs_out,
                       int64_t *m_out, int64_t *loop_ids_out, int64_t *n_loop_ids,
                       int64_t *n_self_loops, int64_t *n_duplicates, double *ms);

/* ---- graph construction (graph.py:162-200) ------------------------- */
/* pairs: int64[2*m] host (any order; the reference normalizes beforehand),
 * extra: int64[n_extra] host ids that only appear in dropped self-loops
 * (EdgeList.loop_ids, graph.py:178-181).  Compacts ids ascending, symmetrizes,
 * sorts (src,dst), builds row_ptr on `device`. */
int kc_graph_from_edges(int device, const int64_t *pairs, int64_t m, const int64_t *extra,
                        int64_t n_extra, kc_graph **out);
/* read_graph's device path (graph.py:203-209 minus the text parse): K0's
 * normal form of raw host pairs (see kc_normalize_edges), kept on the device
 * and fed straight into the CSR build -- one H2D of the raw pairs, no round
 * trip.  Loop-only ids become isolated vertices, as in from_edges(EdgeList).
 * n_self_loops / n_duplicates / normalize_ms are optional outputs. */
int kc_graph_from_raw_edges(int device, const int64_t *raw, int64_t m_raw, int64_t *n_self_loops,
                            int64_t *n_duplicates, double *normalize_ms, kc_graph **out);
/* upload an existing host CSR (Graph arrays); coo_src is derived */
int kc_graph_from_csr(int device, int64_t n, int64_t m, const int64_t *row_ptr,
                      const int32_t *col, const int64_t *orig_ids, kc_graph **out);
/* n, m (undirected), max undirected degree; build time in ms (device events) */
int kc_graph_info(const kc_graph *g, int64_t *n, int64_t *m, int64_t *d_max_undirected,
                  double *build_ms);
/* copy CSR back: row_ptr int64[n+1], col/coo_src int32[2m], orig_ids int64[n]
 * (any pointer may be NULL to skip it) */
int kc_graph_download(const kc_graph *g, int64_t *row_ptr, int32_t *col, int32_t *coo_src,
                      int64_t *orig_ids);
void kc_graph_free(kc_graph *g);
/* the CUDA stream (cudaStream_t) every device call on this graph is issued
 * on, so a caller can record its own events around the library's work */
int kc_graph_stream(const kc_graph *g, void **stream);

/* ---- orientation (orientation.py:116-153) ------------------------- */
typedef struct {
    int64_t m_dir;      /* oriented edges (= m) */
    int64_t d_max;      /* max out-degree */
    int64_t degeneracy; /* degeneracy criterion only, else -1 */
    int64_t rounds;     /* bulk peeling rounds (degeneracy), else 0 */
    double rank_ms;     /* device time of the ranking */
    double orient_ms;   /* device time of the DAG rebuild */
} kc_dag_info;

/* criterion KC_CRIT_DEGREE / KC_CRIT_DEGENERACY / KC_CRIT_DEGENERACY_BULK
 * computed on the device; KC_CRIT_GIVEN uploads rank_in (int32[n]
 * permutation, host). */
int kc_orient(kc_graph *g, int criterion, const int32_t *rank_in, kc_dag_info *info);
/* copy DAG back: rank int32[n], orow_ptr int64[n+1], ocol/ocoo_src int32[m_dir] */
int kc_dag_download(const kc_graph *g, int32_t *rank, int64_t *orow_ptr, int32_t *ocol,
                    int32_t *ocoo_src);

/* ---- counting (scheduler.py:141-293) ------------------------------ */
typedef struct {
    int32_t k;          /* clique size, >= 3 (k = 1, 2 are closed forms on the host) */
    int32_t algorithm;  /* KC_ALGO_* */
    int32_t scheme;     /* KC_SCHEME_* */
    int32_t all_k;      /* pivot only: histogram for every k */
    int32_t group_size; /* orient sub-warp group: 0 = auto, else 1,2,4,8,16,32 */
    int32_t block_size; /* 0 = auto */
    int64_t task_lo;    /* shard [task_lo, task_hi) of make_tasks order */
    int64_t task_hi;    /* < 0 = to the end */
} kc_count_args;

/*
 * Raw, reducible result.  Every field is a plain sum over blocks (and over
 * ranks after an element-wise u64 all-reduce), so a multi-GPU run sums these
 * buffers and then finalizes on the host:
 *   count = limbs[0] + limbs[1]*2^32 + limbs[2]*2^64 + limbs[3]*2^96
 *         + sum_{len,np} hist[len*hist_dim + np] * C(np, len - t)      (pivot)
 *   all_k: slot_t += hist[len][np] * C(np, r) at t = len - r, r = 0..np
 */
typedef struct {
    uint64_t limbs[4];      /* 32-bit limb sums of the direct (orient / t<=1) count */
    uint64_t visits;        /* tree nodes expanded (reference load.total) */
    uint64_t tasks_run;     /* tasks with enough locals */
    int64_t hist_dim;       /* L: hist is L x L u64 (pivot), 0 for orient */
    double count_ms;        /* device time of the counting kernels */
    int32_t group_size;     /* lanes per sub-warp group the orientation warp tier ran with */
    int32_t launches;       /* counting-kernel launches of this call */
    uint64_t word_ops;      /* roofline: u32 row words ANDed (+POPC) by the traversals */
    uint64_t extract_bytes; /* roofline: global bytes read by the sub-graph builder */
} kc_count_raw;

/* hist: caller buffer of hist_cap u64 (L*L, L = d_max + 2) or NULL for orient;
 * visits_per_sm: caller buffer of n_sm u64 or NULL.  Limits: the bitmap
 * engines hold at most 4096 locals per task (oriented max out-degree <= 4096,
 * else KC_EINVAL); counts are exact to 2^128 (KC_EOVERFLOW beyond). */
int kc_count(kc_graph *g, const kc_count_args *args, kc_count_raw *raw, uint64_t *hist,
             int64_t hist_cap, uint64_t *visits_per_sm, int32_t n_sm);
/* number of make_tasks entries for a scheme (scheduler.py:89-95) */
int kc_num_tasks(const kc_graph *g, int32_t scheme, int64_t *n_tasks);
/* per-task cost estimate (int64[n_tasks], make_tasks order) for shard balancing,
 * computed on the device for args' scheme / algorithm / k:
 *   edge tasks (1 + |N+(u) n N+(v)|)^2; vertex tasks of the orientation engine
 *   at t >= 4 (hub roots split into out-edge items) the sum of their items'
 *   costs; other vertex tasks d+(v)^2 */
int kc_task_costs(kc_graph *g, const kc_count_args *args, int64_t *costs, int64_t n_tasks);
/* root-range shards: cuts int64[world+1], rank r runs [cuts[r], cuts[r+1]) of
 * make_tasks order, balanced by a prefix sum of kc_task_costs on the device
 * (only the world+1 cuts cross to the host) */
int kc_shard_ranges(kc_graph *g, const kc_count_args *args, int32_t world, int64_t *cuts);

/* ---- single-task debug / engine entry points ---------------------- */
/* bitgraph.py:125-152: l2g int64[cap], words uint64[cap][wpr_cap] (LSB-first) */
int kc_extract(kc_graph *g, int32_t scheme, int64_t task, int32_t directed, int64_t *l2g,
               uint64_t *words, int64_t cap, int64_t wpr_cap, int64_t *d_out);
/* one host-provided bit matrix: rows uint64[d][wpr] (wpr = ceil(d/64)),
 * algorithm KC_ALGO_ORIENT (directed rows) or KC_ALGO_PIVOT (undirected);
 * all_t: pivot per-t table.  out4 = {count lo, count hi, visits, overflow};
 * all_t: slots_lo/hi[d+1]. */
int kc_count_bitgraph(int device, const uint64_t *rows, int64_t d, int32_t t, int32_t algorithm,
                      int32_t all_t, uint64_t *out4, uint64_t *slots_lo, uint64_t *slots_hi);
/* engine_pivot.py:82-114: argmax |cand & row(v)|, lowest id on ties */
int kc_find_pivot(int device, const uint64_t *rows, int64_t d, const uint64_t *cand,
                  int64_t *pivot, uint64_t *pruned);

/* ---- roofline probe ------------------------------ */
/* measured full-chip AND+POPC word rate with register operands (reg_wps) and
 * with one operand streamed from shared memory (smem_wps), words/s */
int kc_probe(int device, double *reg_wps, double *smem_wps, double *sm_mhz);

#ifdef __cplusplus
}
#endif

#endif /* KCLIQUE_H */
