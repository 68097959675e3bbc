// kc_probe.cu -- in-repo measurement of the integer roofline of the
// traversal ("confirm for cc 10.0 with an in-repo
// microbenchmark").  The traversal's unit of work is one u32 word of a bitmap
// row ANDed with the candidate set and POPC'd (last level) or stored (inner
// levels).  Two ceilings are measured on the live device, full chip:
//   * reg:  AND + POPC + accumulate on register operands (ALU/XU issue bound)
//   * smem: the same with one operand streamed from shared memory by 128-bit
//           loads (LDS bandwidth bound) -- the access pattern of the kernel,
//           whose bitmap rows live in shared memory.
// The roofline peak is min(reg, smem) word-ops/s.
#include "kc_internal.cuh"

namespace {

constexpr int kProbeThreads = 512;

__global__ void __launch_bounds__(kProbeThreads) k_probe_reg(uint32_t seed, int iters,
                                                             unsigned long long *sink) {
    uint32_t a[8], b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        a[j] = seed * (threadIdx.x + 1) + 0x9e3779b9u * j;
        b[j] = (seed ^ (blockIdx.x + j)) * 0x85ebca6bu;
    }
    uint32_t acc0 = 0, acc1 = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
            acc0 += __popc((a[j] ^ uint32_t(i)) & b[j]);
            acc1 += __popc((a[j + 1] ^ uint32_t(i)) & b[j + 1]);
        }
    }
    if (acc0 + acc1 == 0x12345678u) atomicAdd(sink, 1ull);
}

__global__ void __launch_bounds__(kProbeThreads) k_probe_smem(uint32_t seed, int iters,
                                                              unsigned long long *sink) {
    constexpr int kWords = 8192;  // 32 KB
    __shared__ __align__(16) uint32_t buf[kWords];
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) buf[i] = seed * (i + 7) ^ (i << 13);
    __syncthreads();
    const uint4 *v = reinterpret_cast<const uint4 *>(buf);
    const uint32_t c = seed * (threadIdx.x + 3);
    uint32_t acc0 = 0, acc1 = 0;
    int idx = threadIdx.x & (kWords / 4 - 1);
    for (int i = 0; i < iters; ++i) {
        uint4 x = v[idx];
        uint4 y = v[(idx + 32) & (kWords / 4 - 1)];
        acc0 += __popc(x.x & c) + __popc(x.y & c);
        acc1 += __popc(x.z & c) + __popc(x.w & c);
        acc0 += __popc(y.x & c) + __popc(y.y & c);
        acc1 += __popc(y.z & c) + __popc(y.w & c);
        idx = (idx + 64) & (kWords / 4 - 1);
    }
    if (acc0 + acc1 == 0x12345678u) atomicAdd(sink, 1ull);
}

}  // namespace

void kc_do_probe(int device, double *reg_wps, double *smem_wps, double *sm_mhz) {
    kc_device_guard guard(device);
    int sms = 0, clk_khz = 0;
    KC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    KC_CUDA(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, device));
    unsigned long long *sink = nullptr;
    KC_CUDA(cudaMalloc(&sink, sizeof(unsigned long long)));
    cudaEvent_t e0, e1;
    KC_CUDA(cudaEventCreate(&e0));
    KC_CUDA(cudaEventCreate(&e1));
    auto timed = [&](auto kern, int iters, double words_per_iter_thread) {
        int per_sm = 0;
        KC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kProbeThreads, 0));
        const int grid = sms * (per_sm > 0 ? per_sm : 1);
        kern<<<grid, kProbeThreads>>>(12345u, iters / 8, sink);  // warm-up
        KC_CUDA(cudaGetLastError());
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            KC_CUDA(cudaEventRecord(e0));
            kern<<<grid, kProbeThreads>>>(777u + rep, iters, sink);
            KC_CUDA(cudaEventRecord(e1));
            KC_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            KC_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        return double(grid) * kProbeThreads * iters * words_per_iter_thread / (best * 1e-3);
    };
    *reg_wps = timed(k_probe_reg, 1 << 15, 8.0);
    *smem_wps = timed(k_probe_smem, 1 << 15, 8.0);
    *sm_mhz = clk_khz / 1000.0;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
}
