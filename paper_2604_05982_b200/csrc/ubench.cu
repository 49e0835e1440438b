// ubench.cu -- L2-atomic throughput probes: the denominators of the
// scheduler's roofline (no vendor figure exists for B200 L2
// atomic throughput, so it is measured). Each thread issues `ops` independent
// atomics; distinct-word kinds give every thread its own 32-B sector per
// iteration (the join-decrement pattern: one RMW per finished task on its
// parent's record).
#include <cuda_runtime.h>

#include <cstdint>

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
