// kc_ingest.cu -- K0 edge_normalize: the reference's edge-list normal form on
// the device.
//
// Restates graph.py:93-109 (load_edge_list after parsing): self-loops are
// dropped and tallied (their ids kept, unique and ascending, as loop_ids),
// every other pair is oriented (min, max), the pairs are sorted
// lexicographically and repeated pairs are dropped and tallied.
//
// Layout: raw pairs int64[2*m_raw] (row-major, as np.loadtxt returns them).
// When every id fits in 31 bits (any graph the counter can hold, n < 2^31) a
// pair packs into one u64 key (lo << bits | hi) and the sort is a single
// (2*bits)-bit radix sort; larger ids sort as a 128-bit (lo, hi) key through
// a cub decomposer.  Self-loops are written as an all-ones sentinel key that
// sorts last and is removed after the unique pass.  HBM-bound: one read of
// the raw pairs, radix-sort passes over 8 B (or 16 B) keys, one write.
#include <cub/cub.cuh>
#include <cuda/std/tuple>

#include "kc_internal.cuh"

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n, int sms) {
    int64_t b = (n + kThreads - 1) / kThreads;
    int64_t cap = int64_t(sms) * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return int(b);
}

struct pair_key {
    int64_t lo, hi;
    __host__ __device__ bool operator==(const pair_key &o) const {
        return lo == o.lo && hi == o.hi;
    }
};

struct pair_decomposer {
    __host__ __device__ cuda::std::tuple<int64_t &, int64_t &> operator()(pair_key &k) const {
        return {k.lo, k.hi};
    }
};

// warp-aggregated append of the loop ids (loops are rare: no per-row stream)
__device__ __forceinline__ void append_loop(bool loop, int64_t u, int64_t *__restrict__ loop_out,
                                            unsigned long long *__restrict__ loop_cnt) {
    const unsigned act = __activemask();
    const unsigned bal = __ballot_sync(act, loop);
    if (!bal) return;
    const int lane = threadIdx.x & 31, leader = __ffs(bal) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(loop_cnt, (unsigned long long)__popc(bal));
    base = __shfl_sync(act, base, leader);
    if (loop) loop_out[base + __popc(bal & ((1u << lane) - 1))] = u;
}

// per raw row: the oriented key (sentinel for loops); loop ids appended
__global__ void k_orient_pack(const int64_t *__restrict__ raw, int64_t m, int bits,
                              uint64_t *__restrict__ keys, int64_t *__restrict__ loop_out,
                              unsigned long long *__restrict__ loop_cnt) {
    const uint64_t sentinel = (bits >= 32) ? ~uint64_t(0) : ((uint64_t(1) << (2 * bits)) - 1);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t u = raw[2 * i], v = raw[2 * i + 1];
        const bool loop = u == v;
        const uint64_t lo = uint64_t(u < v ? u : v), hi = uint64_t(u < v ? v : u);
        keys[i] = loop ? sentinel : ((lo << bits) | hi);
        append_loop(loop, u, loop_out, loop_cnt);
    }
}

__global__ void k_orient_wide(const int64_t *__restrict__ raw, int64_t m,
                              pair_key *__restrict__ keys, int64_t *__restrict__ loop_out,
                              unsigned long long *__restrict__ loop_cnt) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t u = raw[2 * i], v = raw[2 * i + 1];
        const bool loop = u == v;
        pair_key k;
        k.lo = loop ? INT64_MAX : (u < v ? u : v);
        k.hi = loop ? INT64_MAX : (u < v ? v : u);
        keys[i] = k;
        append_loop(loop, u, loop_out, loop_cnt);
    }
}

__global__ void k_unpack_pairs(const uint64_t *__restrict__ keys, int64_t cnt, int bits,
                               int64_t *__restrict__ out) {
    const uint64_t mask = (uint64_t(1) << bits) - 1;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < cnt;
         i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t k = keys[i];
        out[2 * i] = int64_t(k >> bits);
        out[2 * i + 1] = int64_t(k & mask);
    }
}

__global__ void k_max_i64(const int64_t *__restrict__ a, int64_t cnt,
                          unsigned long long *__restrict__ out) {
    // out[0] = max id, out[1] = 1 if any id is negative
    int64_t best = 0;
    unsigned neg = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < cnt;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t x = a[i];
        best = x > best ? x : best;
        neg |= x < 0;
    }
    for (int o = 16; o; o >>= 1) {
        int64_t x = __shfl_xor_sync(0xffffffffu, best, o);
        best = x > best ? x : best;
    }
    neg = __any_sync(0xffffffffu, neg);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out, (unsigned long long)best);
        if (neg) atomicMax(out + 1, 1ull);
    }
}

template <typename T>
int64_t read_count(const T *d, cudaStream_t s) {
    T h = 0;
    KC_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
    KC_CUDA(cudaStreamSynchronize(s));
    return int64_t(h);
}

}  // namespace

void kc_do_normalize(kc_graph *g, const int64_t *raw, int64_t m_raw, int64_t *pairs_out,
                     int64_t *m_out, int64_t *loop_ids_out, int64_t *n_loop_ids,
                     int64_t *n_self_loops, int64_t *n_duplicates, double *ms,
                     int64_t **dev_pairs, int64_t **dev_loop_ids) {
    // dev_pairs / dev_loop_ids (optional): keep the results on the device and
    // hand the buffers to the caller (stream-ordered on g->stream; the caller
    // frees them) instead of copying them to pairs_out / loop_ids_out
    if (dev_pairs) *dev_pairs = nullptr;
    if (dev_loop_ids) *dev_loop_ids = nullptr;
    KC_REQUIRE(m_raw >= 0, KC_EINVAL, "negative size");
    KC_REQUIRE(m_raw < (int64_t(1) << 31), KC_EINVAL, "edge list too large");
    cudaStream_t s = g->stream;
    cudaEvent_t e0, e1;
    KC_CUDA(cudaEventCreate(&e0));
    KC_CUDA(cudaEventCreate(&e1));
    KC_CUDA(cudaEventRecord(e0, s));
    int64_t n_loops = 0, n_loop_u = 0, n_keep = 0;
    if (m_raw > 0) {
        int64_t *d_raw = kc_alloc<int64_t>(2 * m_raw, s);
        KC_CUDA(cudaMemcpyAsync(d_raw, raw, 16 * m_raw, cudaMemcpyHostToDevice, s));
        // ids must be non-negative, as the parser enforces (graph.py:61-62)
        unsigned long long *d_max = kc_alloc<unsigned long long>(2, s);
        int32_t *d_cnt = kc_alloc<int32_t>(2, s);
        KC_CUDA(cudaMemsetAsync(d_max, 0, 16, s));
        k_max_i64<<<grid_for(2 * m_raw, g->num_sms), kThreads, 0, s>>>(d_raw, 2 * m_raw, d_max);
        KC_CUDA(cudaGetLastError());
        const int64_t max_id = read_count(d_max, s);
        if (read_count(d_max + 1, s)) {
            kc_free(d_raw, s);
            kc_free(d_max, s);
            kc_free(d_cnt, s);
            throw kc_error(KC_EINVAL, "vertex ids must be non-negative");
        }
        int64_t *loop_val = kc_alloc<int64_t>(m_raw, s);
        int64_t *loop_sel = kc_alloc<int64_t>(m_raw, s);
        unsigned long long *loop_cnt = kc_alloc<unsigned long long>(1, s);
        KC_CUDA(cudaMemsetAsync(loop_cnt, 0, 8, s));
        int64_t *d_pairs = kc_alloc<int64_t>(2 * m_raw, s);
        size_t bytes = 0;
        // max_id + 1 must stay unused so the all-ones key is a free sentinel
        const int bits = kc_bits_for(max_id + 1);
        if (bits <= 31) {
            uint64_t *keys = kc_alloc<uint64_t>(m_raw, s);
            uint64_t *keys2 = kc_alloc<uint64_t>(m_raw, s);
            k_orient_pack<<<grid_for(m_raw, g->num_sms), kThreads, 0, s>>>(d_raw, m_raw, bits,
                                                                            keys, loop_val,
                                                                            loop_cnt);
            KC_CUDA(cudaGetLastError());
            // lexsort((hi, lo))                          graph.py:101-102
            KC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys, keys2, int(m_raw), 0,
                                                   2 * bits, s));
            void *tmp = kc_tmp(g, bytes);
            KC_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, keys, keys2, int(m_raw), 0,
                                                   2 * bits, s));
            // keep first of each run                     graph.py:103-105
            bytes = 0;
            KC_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, keys2, keys, d_cnt, int(m_raw), s));
            tmp = kc_tmp(g, bytes);
            KC_CUDA(cub::DeviceSelect::Unique(tmp, bytes, keys2, keys, d_cnt, int(m_raw), s));
            int64_t n_uniq = read_count(d_cnt, s);
            const uint64_t sentinel = (uint64_t(1) << (2 * bits)) - 1;
            uint64_t last = 0;
            KC_CUDA(cudaMemcpyAsync(&last, keys + n_uniq - 1, 8, cudaMemcpyDeviceToHost, s));
            KC_CUDA(cudaStreamSynchronize(s));
            n_keep = n_uniq - (last == sentinel ? 1 : 0);
            if (n_keep)
                k_unpack_pairs<<<grid_for(n_keep, g->num_sms), kThreads, 0, s>>>(keys, n_keep,
                                                                                  bits, d_pairs);
            KC_CUDA(cudaGetLastError());
            kc_free(keys, s);
            kc_free(keys2, s);
        } else {
            pair_key *keys = kc_alloc<pair_key>(m_raw, s);
            pair_key *keys2 = kc_alloc<pair_key>(m_raw, s);
            k_orient_wide<<<grid_for(m_raw, g->num_sms), kThreads, 0, s>>>(d_raw, m_raw, keys,
                                                                            loop_val, loop_cnt);
            KC_CUDA(cudaGetLastError());
            KC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys, keys2, int(m_raw),
                                                   pair_decomposer{}, s));
            void *tmp = kc_tmp(g, bytes);
            KC_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, keys, keys2, int(m_raw),
                                                   pair_decomposer{}, s));
            bytes = 0;
            KC_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, keys2, keys, d_cnt, int(m_raw), s));
            tmp = kc_tmp(g, bytes);
            KC_CUDA(cub::DeviceSelect::Unique(tmp, bytes, keys2, keys, d_cnt, int(m_raw), s));
            int64_t n_uniq = read_count(d_cnt, s);
            pair_key last{};
            KC_CUDA(cudaMemcpyAsync(&last, keys + n_uniq - 1, sizeof(pair_key),
                                    cudaMemcpyDeviceToHost, s));
            KC_CUDA(cudaStreamSynchronize(s));
            n_keep = n_uniq - (last.lo == INT64_MAX && last.hi == INT64_MAX ? 1 : 0);
            // pair_key is two int64 in (lo, hi) order: already the output layout
            if (n_keep)
                KC_CUDA(cudaMemcpyAsync(d_pairs, keys, 16 * n_keep, cudaMemcpyDeviceToDevice, s));
            kc_free(keys, s);
            kc_free(keys2, s);
        }
        // self-loop ids (appended by the pack kernel): sort, unique   graph.py:97-98
        n_loops = read_count(loop_cnt, s);
        void *tmp = nullptr;
        if (n_loops) {
            bytes = 0;
            KC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, loop_val, loop_sel,
                                                   int(n_loops), 0, 64, s));
            tmp = kc_tmp(g, bytes);
            KC_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, loop_val, loop_sel, int(n_loops),
                                                   0, 64, s));
            bytes = 0;
            KC_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, loop_sel, loop_val, d_cnt + 1,
                                              int(n_loops), s));
            tmp = kc_tmp(g, bytes);
            KC_CUDA(cub::DeviceSelect::Unique(tmp, bytes, loop_sel, loop_val, d_cnt + 1,
                                              int(n_loops), s));
            n_loop_u = read_count(d_cnt + 1, s);
        }
        if (pairs_out && n_keep && !dev_pairs)
            KC_CUDA(cudaMemcpyAsync(pairs_out, d_pairs, 16 * n_keep, cudaMemcpyDeviceToHost, s));
        if (loop_ids_out && n_loop_u && !dev_loop_ids)
            KC_CUDA(cudaMemcpyAsync(loop_ids_out, loop_val, 8 * n_loop_u, cudaMemcpyDeviceToHost,
                                    s));
        kc_free(d_raw, s);
        kc_free(d_max, s);
        kc_free(d_cnt, s);
        kc_free(loop_sel, s);
        kc_free(loop_cnt, s);
        if (dev_loop_ids) *dev_loop_ids = loop_val;
        else kc_free(loop_val, s);
        if (dev_pairs) *dev_pairs = d_pairs;
        else kc_free(d_pairs, s);
    }
    KC_CUDA(cudaEventRecord(e1, s));
    KC_CUDA(cudaEventSynchronize(e1));
    float t = 0;
    KC_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (m_out) *m_out = n_keep;
    if (n_loop_ids) *n_loop_ids = n_loop_u;
    if (n_self_loops) *n_self_loops = n_loops;
    if (n_duplicates) *n_duplicates = (m_raw - n_loops) - n_keep;
    if (ms) *ms = t;
}
