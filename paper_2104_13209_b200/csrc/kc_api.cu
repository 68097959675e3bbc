// kc_api.cu -- extern "C" boundary of libkc.so (declared in include/kclique.h).
// Each entry point converts kc_error / CUDA failures into the status codes of
// SURVEY.md §8(b) and keeps the message for kc_last_error().
#include <cstring>
#include <string>
#include <vector>

#include "kc_internal.cuh"

namespace {
thread_local std::string g_last_error;

template <typename F>
int guarded(F &&f) {
    try {
        f();
        g_last_error.clear();
        return KC_OK;
    } catch (const kc_error &e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc &) {
        g_last_error = "host allocation failed";
        return KC_ENOMEM;
    } catch (const std::exception &e) {
        g_last_error = e.what();
        return KC_ECUDA;
    }
}

void require_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw kc_error(KC_ECUDA, std::string("no CUDA device available: ") +
                                     (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
    KC_REQUIRE(device >= 0 && device < n, KC_EINVAL, "device index out of range");
    cudaDeviceProp prop;
    KC_CUDA(cudaGetDeviceProperties(&prop, device));
    KC_REQUIRE(prop.major >= 10, KC_ECUDA,
               std::string("libkc is built for sm_100a; device is ") + prop.name);
}

}  // namespace

void kc_pool_setup(int device) {
    static bool done[64] = {false};
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~uint64_t(0);
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[device] = true;
}

namespace {

kc_graph *new_graph(int device) {
    require_device(device);
    kc_graph *g = new kc_graph();
    g->device = device;
    KC_CUDA(cudaSetDevice(device));
    KC_CUDA(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device));
    KC_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    kc_pool_setup(device);
    return g;
}

void destroy(kc_graph *g) {
    if (!g) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(g->device);
    kc_free_dag(g);
    kc_free(g->row_ptr, g->stream);
    kc_free(g->col, g->stream);
    kc_free(g->coo_src, g->stream);
    kc_free(g->orig_ids, g->stream);
    kc_free(g->tmp, g->stream);
    if (g->stream) {
        cudaStreamSynchronize(g->stream);
        cudaStreamDestroy(g->stream);
    }
    if (g->aux) cudaStreamDestroy(g->aux);
    if (prev >= 0) cudaSetDevice(prev);
    delete g;
}
}  // namespace

extern "C" {

int kc_abi_version(void) { return KC_ABI_VERSION; }

const char *kc_last_error(void) { return g_last_error.c_str(); }

int kc_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int kc_num_sms(int device) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return v;
}

int kc_graph_from_edges(int device, const int64_t *pairs, int64_t m, const int64_t *extra,
                        int64_t n_extra, kc_graph **out) {
    return guarded([&] {
        KC_REQUIRE(out, KC_EINVAL, "out is NULL");
        KC_REQUIRE(m == 0 || pairs, KC_EINVAL, "pairs is NULL");
        KC_REQUIRE(n_extra == 0 || extra, KC_EINVAL, "extra is NULL");
        *out = nullptr;
        kc_graph *g = new_graph(device);
        try {
            kc_device_guard guard(device);
            kc_build_from_edges(g, pairs, m, extra, n_extra);
        } catch (...) {
            destroy(g);
            throw;
        }
        *out = g;
    });
}

int kc_normalize_edges(int device, const int64_t *raw, int64_t m_raw, int64_t *pairs_out,
                       int64_t *m_out, int64_t *loop_ids_out, int64_t *n_loop_ids,
                       int64_t *n_self_loops, int64_t *n_duplicates, double *ms) {
    return guarded([&] {
        KC_REQUIRE(m_raw >= 0, KC_EINVAL, "negative size");
        KC_REQUIRE(m_raw == 0 || (raw && pairs_out && loop_ids_out), KC_EINVAL,
                   "NULL buffer");
        kc_graph *g = new_graph(device);  // stream + scratch only; no graph is built
        try {
            kc_device_guard guard(device);
            kc_do_normalize(g, raw, m_raw, pairs_out, m_out, loop_ids_out, n_loop_ids,
                            n_self_loops, n_duplicates, ms);
        } catch (...) {
            destroy(g);
            throw;
        }
        destroy(g);
    });
}

int kc_graph_from_raw_edges(int device, const int64_t *raw, int64_t m_raw, int64_t *n_self_loops,
                            int64_t *n_duplicates, double *normalize_ms, kc_graph **out) {
    return guarded([&] {
        KC_REQUIRE(out, KC_EINVAL, "out is NULL");
        KC_REQUIRE(m_raw >= 0 && (m_raw == 0 || raw), KC_EINVAL, "bad raw pairs");
        *out = nullptr;
        kc_graph *g = new_graph(device);
        int64_t *d_pairs = nullptr, *d_loops = nullptr;
        try {
            kc_device_guard guard(device);
            int64_t m = 0, n_loop = 0;
            kc_do_normalize(g, raw, m_raw, nullptr, &m, nullptr, &n_loop, n_self_loops,
                            n_duplicates, normalize_ms, &d_pairs, &d_loops);
            kc_build_from_edges(g, d_pairs, m, d_loops, n_loop);
            kc_free(d_pairs, g->stream);
            kc_free(d_loops, g->stream);
        } catch (...) {
            kc_free(d_pairs, g->stream);
            kc_free(d_loops, g->stream);
            destroy(g);
            throw;
        }
        *out = g;
    });
}

int kc_graph_from_csr(int device, int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col,
                      const int64_t *orig_ids, kc_graph **out) {
    return guarded([&] {
        KC_REQUIRE(out && row_ptr && (m == 0 || col), KC_EINVAL, "NULL argument");
        *out = nullptr;
        kc_graph *g = new_graph(device);
        try {
            kc_device_guard guard(device);
            kc_build_from_csr(g, n, m, row_ptr, col, orig_ids);
        } catch (...) {
            destroy(g);
            throw;
        }
        *out = g;
    });
}

int kc_graph_info(const kc_graph *g, int64_t *n, int64_t *m, int64_t *d_max_undirected,
                  double *build_ms) {
    return guarded([&] {
        KC_REQUIRE(g, KC_EINVAL, "graph is NULL");
        if (n) *n = g->n;
        if (m) *m = g->m;
        if (d_max_undirected) *d_max_undirected = g->d_max_und;
        if (build_ms) *build_ms = g->build_ms;
    });
}

int kc_graph_download(const kc_graph *g, int64_t *row_ptr, int32_t *col, int32_t *coo_src,
                      int64_t *orig_ids) {
    return guarded([&] {
        KC_REQUIRE(g, KC_EINVAL, "graph is NULL");
        kc_device_guard guard(g->device);
        KC_CUDA(cudaStreamSynchronize(g->stream));
        if (row_ptr)
            KC_CUDA(cudaMemcpy(row_ptr, g->row_ptr, 8 * (g->n + 1), cudaMemcpyDeviceToHost));
        if (col && g->m) KC_CUDA(cudaMemcpy(col, g->col, 8 * g->m, cudaMemcpyDeviceToHost));
        if (coo_src && g->m)
            KC_CUDA(cudaMemcpy(coo_src, g->coo_src, 8 * g->m, cudaMemcpyDeviceToHost));
        if (orig_ids && g->n)
            KC_CUDA(cudaMemcpy(orig_ids, g->orig_ids, 8 * g->n, cudaMemcpyDeviceToHost));
    });
}

void kc_graph_free(kc_graph *g) { destroy(g); }

int kc_probe(int device, double *reg_wps, double *smem_wps, double *sm_mhz) {
    return guarded([&] {
        KC_REQUIRE(reg_wps && smem_wps && sm_mhz, KC_EINVAL, "NULL output");
        require_device(device);
        kc_do_probe(device, reg_wps, smem_wps, sm_mhz);
    });
}

int kc_graph_stream(const kc_graph *g, void **stream) {
    return guarded([&] {
        KC_REQUIRE(g && stream, KC_EINVAL, "graph or stream is NULL");
        *stream = reinterpret_cast<void *>(g->stream);
    });
}

int kc_orient(kc_graph *g, int criterion, const int32_t *rank_in, kc_dag_info *info) {
    return guarded([&] {
        KC_REQUIRE(g, KC_EINVAL, "graph is NULL");
        kc_device_guard guard(g->device);
        kc_do_orient(g, criterion, rank_in, info);
    });
}

int kc_dag_download(const kc_graph *g, int32_t *rank, int64_t *orow_ptr, int32_t *ocol,
                    int32_t *ocoo_src) {
    return guarded([&] {
        KC_REQUIRE(g && g->oriented, KC_EINVAL, "graph is not oriented");
        kc_device_guard guard(g->device);
        KC_CUDA(cudaStreamSynchronize(g->stream));
        if (rank && g->n) KC_CUDA(cudaMemcpy(rank, g->rank, 4 * g->n, cudaMemcpyDeviceToHost));
        if (orow_ptr)
            KC_CUDA(cudaMemcpy(orow_ptr, g->orow_ptr, 8 * (g->n + 1), cudaMemcpyDeviceToHost));
        if (ocol && g->m_dir)
            KC_CUDA(cudaMemcpy(ocol, g->ocol, 4 * g->m_dir, cudaMemcpyDeviceToHost));
        if (ocoo_src && g->m_dir)
            KC_CUDA(cudaMemcpy(ocoo_src, g->ocoo, 4 * g->m_dir, cudaMemcpyDeviceToHost));
    });
}

int kc_count(kc_graph *g, const kc_count_args *args, kc_count_raw *raw, uint64_t *hist,
             int64_t hist_cap, uint64_t *visits_per_sm, int32_t n_sm) {
    return guarded([&] {
        KC_REQUIRE(g && args && raw, KC_EINVAL, "NULL argument");
        kc_device_guard guard(g->device);
        kc_do_count(g, args, raw, hist, hist_cap, visits_per_sm, n_sm);
    });
}

int kc_num_tasks(const kc_graph *g, int32_t scheme, int64_t *n_tasks) {
    return guarded([&] {
        KC_REQUIRE(g && g->oriented && n_tasks, KC_EINVAL, "graph is not oriented");
        KC_REQUIRE(scheme == KC_SCHEME_VERTEX || scheme == KC_SCHEME_EDGE, KC_EINVAL,
                   "unknown scheme");
        kc_device_guard guard(g->device);
        *n_tasks = kc_task_count(g, scheme);
    });
}

int kc_task_costs(kc_graph *g, const kc_count_args *args, int64_t *costs, int64_t n_tasks) {
    return guarded([&] {
        KC_REQUIRE(g && g->oriented && args && (costs || n_tasks == 0), KC_EINVAL,
                   "graph is not oriented");
        KC_REQUIRE(args->scheme == KC_SCHEME_VERTEX || args->scheme == KC_SCHEME_EDGE, KC_EINVAL,
                   "unknown scheme");
        kc_do_task_costs(g, args, costs, n_tasks);
    });
}

int kc_shard_ranges(kc_graph *g, const kc_count_args *args, int32_t world, int64_t *cuts) {
    return guarded([&] {
        KC_REQUIRE(g && g->oriented && args && cuts, KC_EINVAL, "graph is not oriented");
        KC_REQUIRE(args->scheme == KC_SCHEME_VERTEX || args->scheme == KC_SCHEME_EDGE, KC_EINVAL,
                   "unknown scheme");
        kc_do_shard_ranges(g, args, world, cuts);
    });
}

int kc_extract(kc_graph *g, int32_t scheme, int64_t task, int32_t directed, int64_t *l2g,
               uint64_t *words, int64_t cap, int64_t wpr_cap, int64_t *d_out) {
    return guarded([&] {
        KC_REQUIRE(g && l2g && words && d_out, KC_EINVAL, "NULL argument");
        KC_REQUIRE(scheme == KC_SCHEME_VERTEX || scheme == KC_SCHEME_EDGE, KC_EINVAL,
                   "unknown scheme");
        kc_device_guard guard(g->device);
        kc_do_extract(g, scheme, task, directed, l2g, words, cap, wpr_cap, d_out);
    });
}

int kc_count_bitgraph(int device, const uint64_t *rows, int64_t d, int32_t t, int32_t algorithm,
                      int32_t all_t, uint64_t *out4, uint64_t *slots_lo, uint64_t *slots_hi) {
    return guarded([&] {
        KC_REQUIRE(out4 && (d == 0 || rows), KC_EINVAL, "NULL argument");
        KC_REQUIRE(!all_t || (slots_lo && slots_hi), KC_EINVAL, "slots required for all_t");
        KC_REQUIRE(algorithm == KC_ALGO_ORIENT || algorithm == KC_ALGO_PIVOT, KC_EINVAL,
                   "unknown algorithm");
        require_device(device);
        kc_do_count_bitgraph(device, rows, d, t, algorithm, all_t, out4, slots_lo, slots_hi);
        if (out4[3]) throw kc_error(KC_EOVERFLOW, "clique count exceeded the 128-bit accumulator");
    });
}

int kc_find_pivot(int device, const uint64_t *rows, int64_t d, const uint64_t *cand,
                  int64_t *pivot, uint64_t *pruned) {
    return guarded([&] {
        KC_REQUIRE(rows && cand && pivot && pruned, KC_EINVAL, "NULL argument");
        require_device(device);
        kc_do_find_pivot(device, rows, d, cand, pivot, pruned);
    });
}

}  // extern "C"
