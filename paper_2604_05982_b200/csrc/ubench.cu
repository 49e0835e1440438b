// ubench.cu -- L2-atomic throughput probes: the denominators of the
// scheduler's roofline (no vendor figure exists for B200 L2
// atomic throughput, so it is measured). Each thread issues `ops` independent
// atomics; distinct-word kinds give every thread its own 32-B sector per
// iteration (the join-decrement pattern: one RMW per finished task on its
// parent's record).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "gtap.h"
#include "gtap_internal.cuh"

namespace {

template <int KIND>
__global__ void __launch_bounds__(1024) ubench_kernel(uint32_t* buf, uint64_t words, uint32_t ops,
                                                      unsigned long long* sink) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (uint32_t i = 0; i < ops; ++i) {
        // one 32-B sector per (thread, iteration), wrapping over the buffer
        const uint64_t w = ((tid + (uint64_t)i * nthreads) * 8u) % words;
        uint32_t* p = buf + w;
        if constexpr (KIND == 0) {
            acc += gtap::dev::atom_add_relaxed(p, 1u);
        } else if constexpr (KIND == 1) {
            asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(1u) : "memory");
        } else if constexpr (KIND == 2) {
            acc += gtap::dev::atom_cas_relaxed(p, acc, acc + 1u);
        } else if constexpr (KIND == 3) {
            acc += (uint32_t)atomicMin(reinterpret_cast<int*>(p), (int)(i ^ (uint32_t)tid));
        } else if constexpr (KIND == 4) {
            acc += gtap::dev::atom_add_relaxed(buf, 1u);
        } else if constexpr (KIND == 5) {
            acc += (uint32_t)gtap::dev::atom_add_acq_rel(reinterpret_cast<int32_t*>(p), 1);
        } else if constexpr (KIND == 6) {
            // the fused fib join: one relaxed 64-bit atom.add with return per task
            acc += (uint32_t)gtap::dev::atom_add_relaxed_u64(p, 0x1FFFFFFFFull);
        }
    }
    if (acc == 0xFFFFFFFFu) atomicAdd(sink, 1ull);
}

}  // namespace

extern "C" gtap_status gtap_ubench_atomics(void* d_buf, uint64_t words, uint32_t kind, uint32_t grid, uint32_t block,
                                           uint32_t ops_per_thread, void* stream, float* ms) {
    if (!d_buf || words < 8 || kind > 6 || grid == 0 || block == 0 || block > 1024 || !ms) return GTAP_E_INVAL;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint32_t* buf = static_cast<uint32_t*>(d_buf);
    if (cudaMemsetAsync(buf, 0, words * 4, s) != cudaSuccess) return GTAP_E_CUDA;
    unsigned long long* sink = reinterpret_cast<unsigned long long*>(buf + words - 2);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    switch (kind) {
        case 0: ubench_kernel<0><<<grid, block, 0, s>>>(buf, words - 8, ops_per_thread, sink); break;
        case 1: ubench_kernel<1><<<grid, block, 0, s>>>(buf, words - 8, ops_per_thread, sink); break;
        case 2: ubench_kernel<2><<<grid, block, 0, s>>>(buf, words - 8, ops_per_thread, sink); break;
        case 3: ubench_kernel<3><<<grid, block, 0, s>>>(buf, words - 8, ops_per_thread, sink); break;
        case 4: ubench_kernel<4><<<grid, block, 0, s>>>(buf, words - 8, ops_per_thread, sink); break;
        case 5: ubench_kernel<5><<<grid, block, 0, s>>>(buf, words - 8, ops_per_thread, sink); break;
        case 6: ubench_kernel<6><<<grid, block, 0, s>>>(buf, words - 8, ops_per_thread, sink); break;
    }
    cudaEventRecord(e1, s);
    const cudaError_t err = cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return err == cudaSuccess ? GTAP_OK : GTAP_E_CUDA;
}

// ---------------------------------------------------------------------------
// SM -> L2-die map (SURVEY.md §8(d) probe (vi)). B200 is two dies; each address is homed in one die's L2
// (2 KB granules) and an SM reaches its own die's L2 faster than the other one. One 32-thread block per SM
// (a large dynamic shared-memory request keeps a second block off every SM), taking turns by ticket so that
// no two SMs probe at once: lane 0 times `reps` dependent strong (L2) loads to each of n probe addresses.
namespace gtap {
namespace {
__global__ void __launch_bounds__(32) die_probe_kernel(const char* base, uint64_t stride, uint32_t n, uint32_t reps,
                                                      uint32_t zero, float* lat, uint32_t* ticket, uint32_t* smids) {
    extern __shared__ unsigned char die_probe_pad[];
    if (threadIdx.x != 0) return;
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    while (dev::ld_acquire(ticket) != blockIdx.x) dev::nanosleep(200);
    die_probe_pad[0] = 0;
    for (uint32_t k = 0; k < n; ++k) {
        const char* a = base + (uint64_t)k * stride;
        uint32_t x = dev::ld_relaxed(reinterpret_cast<const uint32_t*>(a));   // warm the TLB
        const long long t0 = clock64();
        for (uint32_t r = 0; r < reps; ++r)   // each address depends on the previous load's value
            x = dev::ld_relaxed(reinterpret_cast<const uint32_t*>(a + (x & zero)));
        const long long t1 = clock64();
        lat[(uint64_t)blockIdx.x * n + k] = (float)(t1 - t0) / (float)reps + (float)(x & zero);
    }
    smids[blockIdx.x] = smid;
    dev::st_release(ticket, blockIdx.x + 1u);
}
}  // namespace

// probe `n` addresses base + k * stride from every SM; die labels: 0 = SM 0's die. Returns 0 on success.
// sm_die[smid] (cap entries), addr_near[k] = die whose SMs reach address k faster, out3 = {near cycles,
// far cycles, consistency (mean fraction of addresses on which an SM agrees with its die's majority)}.
int die_probe(const void* base, uint64_t stride, uint32_t n, uint8_t* sm_die, uint32_t cap, uint8_t* addr_near,
              float* out3, cudaStream_t s) {
    int dev = 0, nsm = 0, smem = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (nsm <= 0 || n == 0 || (uint32_t)nsm > cap) return -1;
    float* d_lat = nullptr;
    uint32_t* d_aux = nullptr;
    if (cudaMalloc(&d_lat, sizeof(float) * nsm * n) != cudaSuccess) return -1;
    if (cudaMalloc(&d_aux, sizeof(uint32_t) * (nsm + 1)) != cudaSuccess) { cudaFree(d_lat); return -1; }
    cudaMemsetAsync(d_aux, 0, sizeof(uint32_t) * (nsm + 1), s);
    const int pad = smem > 120 * 1024 ? smem : 120 * 1024;   // > half an SM's shared memory: one block per SM
    cudaFuncSetAttribute(die_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pad);
    die_probe_kernel<<<nsm, 32, pad, s>>>(static_cast<const char*>(base), stride, n, 16u, 0u, d_lat, d_aux + nsm,
                                          d_aux);
    std::vector<float> lat((size_t)nsm * n);
    std::vector<uint32_t> smids(nsm);
    int rc = 0;
    if (cudaStreamSynchronize(s) != cudaSuccess ||
        cudaMemcpy(lat.data(), d_lat, sizeof(float) * lat.size(), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(smids.data(), d_aux, sizeof(uint32_t) * nsm, cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = -1;
    cudaFree(d_lat);
    cudaFree(d_aux);
    if (rc) return rc;
    // per address: an SM is "near" when its latency is in the lower half of the address's range; an SM's die = whether it
    // agrees with block 0's near/far pattern on most addresses
    std::vector<uint8_t> nearbit((size_t)nsm * n);
    for (uint32_t k = 0; k < n; ++k) {
        std::vector<float> col(nsm);
        for (int b = 0; b < nsm; ++b) col[b] = lat[(size_t)b * n + k];
        // bimodal (near ~ L2 hit, far ~ L2 hit + die crossing): split at the middle of the range
        const float lo = *std::min_element(col.begin(), col.end()), hi = *std::max_element(col.begin(), col.end());
        const float mid = 0.5f * (lo + hi);
        for (int b = 0; b < nsm; ++b) nearbit[(size_t)b * n + k] = col[b] < mid ? 1 : 0;
    }
    std::vector<uint8_t> die(nsm);
    double agree_sum = 0;
    for (int b = 0; b < nsm; ++b) {
        uint32_t same = 0;
        for (uint32_t k = 0; k < n; ++k) same += nearbit[(size_t)b * n + k] == nearbit[k];
        die[b] = same * 2 >= n ? 0 : 1;
        agree_sum += (double)std::max(same, n - same) / n;
    }
    double nsum = 0, fsum = 0;
    size_t nn = 0, nf = 0;
    for (uint32_t k = 0; k < n; ++k) {
        // the address is near the die whose SMs see the lower mean latency
        double m[2] = {0, 0};
        int c[2] = {0, 0};
        for (int b = 0; b < nsm; ++b) { m[die[b]] += lat[(size_t)b * n + k]; ++c[die[b]]; }
        for (int d = 0; d < 2; ++d) m[d] = c[d] ? m[d] / c[d] : 1e30;
        const int nd = m[1] < m[0] ? 1 : 0;
        if (addr_near) addr_near[k] = (uint8_t)nd;
        for (int b = 0; b < nsm; ++b) {
            if (die[b] == nd) { nsum += lat[(size_t)b * n + k]; ++nn; } else { fsum += lat[(size_t)b * n + k]; ++nf; }
        }
    }
    for (uint32_t i = 0; i < cap; ++i) sm_die[i] = 0;
    for (int b = 0; b < nsm; ++b) sm_die[smids[b] < cap ? smids[b] : 0] = die[b];
    if (out3) {
        out3[0] = nn ? (float)(nsum / nn) : 0.f;
        out3[1] = nf ? (float)(fsum / nf) : 0.f;
        out3[2] = (float)(agree_sum / nsm);
    }
    return 0;
}
}  // namespace gtap

extern "C" gtap_status gtap_ubench_die_probe(const void* d_buf, uint64_t bytes, uint32_t n_addr, uint8_t* h_sm_die,
                                             uint32_t sm_cap, uint8_t* h_addr_near, float* h_out3, void* stream) {
    if (!d_buf || n_addr == 0 || !h_sm_die || bytes / n_addr < 4) return GTAP_E_INVAL;
    return gtap::die_probe(d_buf, bytes / n_addr / 4 * 4, n_addr, h_sm_die, sm_cap, h_addr_near, h_out3,
                           static_cast<cudaStream_t>(stream)) == 0 ? GTAP_OK : GTAP_E_CUDA;
}
