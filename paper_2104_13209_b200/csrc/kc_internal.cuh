// kc_internal.cuh -- shared definitions of libkc (B200 / sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/kclique.h"

// ---------------------------------------------------------------------------
// error plumbing: every C-ABI entry point catches kc_error and returns its code
// ---------------------------------------------------------------------------
struct kc_error : std::runtime_error {
    int code;
    kc_error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define KC_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t _e = (call);                                                        \
        if (_e != cudaSuccess)                                                          \
            throw kc_error(KC_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e) + \
                                         " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
    } while (0)

#define KC_REQUIRE(cond, code, msg)           \
    do {                                      \
        if (!(cond)) throw kc_error(code, msg); \
    } while (0)

// ---------------------------------------------------------------------------
// device-resident graph: undirected CSR+COO (graph.py:112-131) and its DAG
// (orientation.py:20-45).  Layout in HBM: structure-of-arrays, int64 row
// pointers, int32 columns -- exactly the reference arrays.
// ---------------------------------------------------------------------------
struct kc_graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;  // second stream for concurrent count kernels
    int num_sms = 0;
    int64_t n = 0, m = 0;
    int64_t d_max_und = 0;
    double build_ms = 0.0;
    int64_t *row_ptr = nullptr;  // [n+1]
    int32_t *col = nullptr;      // [2m]
    int32_t *coo_src = nullptr;  // [2m]
    int64_t *orig_ids = nullptr; // [n]
    // DAG
    int oriented = 0;
    int criterion = -1;
    int64_t m_dir = 0, d_max = 0, degeneracy = -1;
    int32_t *rank = nullptr;     // [n]
    int64_t *orow_ptr = nullptr; // [n+1]
    int32_t *ocol = nullptr;     // [m]
    int32_t *ocoo = nullptr;     // [m]
    int32_t *esize = nullptr;    // [m] |N+(u) n N+(v)| per oriented edge (lazy, edge tasks)
    // reusable scratch
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
};

// scoped device guard
struct kc_device_guard {
    int prev = -1;
    explicit kc_device_guard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) KC_CUDA(cudaSetDevice(dev));
    }
    ~kc_device_guard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

void *kc_tmp(kc_graph *g, size_t bytes);
void kc_free_dag(kc_graph *g);

// Device memory comes from the stream-ordered pool (cudaMallocAsync on the
// graph's stream; the pool keeps freed blocks, so repeated runs do not pay
// cudaMalloc/cudaFree or their implicit device synchronisation).
template <typename T>
static inline T *kc_alloc(size_t count, cudaStream_t s) {
    T *p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&p), count * sizeof(T), s);
    if (e != cudaSuccess)
        throw kc_error(e == cudaErrorMemoryAllocation ? KC_ENOMEM : KC_ECUDA,
                       std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
    return p;
}

static inline void kc_free(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

// keep freed pool memory for reuse (called once per device)
void kc_pool_setup(int device);

static inline int kc_bits_for(int64_t x) {  // bits needed to hold 0..x
    int b = 1;
    while (b < 63 && (int64_t(1) << b) <= x) ++b;
    return b;
}

// edge-list normal form (kc_ingest.cu)
void kc_do_normalize(kc_graph *g, const int64_t *raw, int64_t m_raw, int64_t *pairs_out,
                     int64_t *m_out, int64_t *loop_ids_out, int64_t *n_loop_ids,
                     int64_t *n_self_loops, int64_t *n_duplicates, double *ms,
                     int64_t **dev_pairs = nullptr, int64_t **dev_loop_ids = nullptr);

// graph build / orientation (kc_graph.cu); pairs / extra may be host or
// device pointers (copied with cudaMemcpyDefault)
void kc_build_from_edges(kc_graph *g, const int64_t *pairs, int64_t m, const int64_t *extra,
                         int64_t n_extra);
void kc_build_from_csr(kc_graph *g, int64_t n, int64_t m, const int64_t *row_ptr,
                       const int32_t *col, const int64_t *orig_ids);
void kc_do_orient(kc_graph *g, int criterion, const int32_t *rank_in, kc_dag_info *info);
int64_t kc_task_count(const kc_graph *g, int scheme);
// exact heap order from core numbers (kc_peel.cu): rank_out int32[n] on the device
void kc_exact_order_from_cores(kc_graph *g, const int32_t *core, int64_t degeneracy,
                               int32_t *rank_out);
void kc_make_tasks(kc_graph *g, int scheme, int64_t lo, int64_t hi, int min_d, int32_t *d_tasks,
                   int64_t *n_out);

// counting (kc_count.cu)
void kc_do_count(kc_graph *g, const kc_count_args *a, kc_count_raw *raw, uint64_t *hist,
                 int64_t hist_cap, uint64_t *visits_per_sm, int32_t n_sm);
void kc_do_task_costs(kc_graph *g, const kc_count_args *a, int64_t *costs, int64_t n_tasks);
void kc_do_shard_ranges(kc_graph *g, const kc_count_args *a, int world, int64_t *cuts);
void kc_do_extract(kc_graph *g, int scheme, int64_t task, int directed, int64_t *l2g,
                   uint64_t *words, int64_t cap, int64_t wpr_cap, int64_t *d_out);
void kc_do_count_bitgraph(int device, const uint64_t *rows, int64_t d, int t, int algorithm,
                          int all_t, uint64_t *out4, uint64_t *slots_lo, uint64_t *slots_hi);
void kc_do_find_pivot(int device, const uint64_t *rows, int64_t d, const uint64_t *cand,
                      int64_t *pivot, uint64_t *pruned);

// roofline probe (kc_probe.cu)
void kc_do_probe(int device, double *reg_wps, double *smem_wps, double *sm_mhz);

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t kc_lower_bound_i64(const int64_t *__restrict__ a, int64_t n,
                                                      int64_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int64_t kc_lower_bound_i32(const int32_t *__restrict__ a, int64_t n,
                                                      int32_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ unsigned long long kc_globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned kc_smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
