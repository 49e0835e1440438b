// merge_micro2.cu -- time the product merges (ms_merge, ms_merge_tma) in isolation, one thread.
#ifndef LB_THREADS
#define LB_THREADS 1024
#define LB_MIN 1
#endif
#include "../paper_2604_05982_b200/csrc/table_mergesort.cu"
// the table's board reset calls the runtime's fill helper (runtime.cu, not linked here)
namespace gtap {
cudaError_t zero_async(void* p, size_t bytes, cudaStream_t s) { return cudaMemsetAsync(p, 0, bytes, s); }
}  // namespace gtap
#include <cstdio>
#include <vector>
#include <algorithm>

__global__ void __launch_bounds__(LB_THREADS, LB_MIN) k_tma(const int* s, int* d, int n, int nt) {
    extern __shared__ __align__(128) unsigned char sm[];
    gtap::MergeSlotHolder* S = reinterpret_cast<gtap::MergeSlotHolder*>(sm);
    if (threadIdx.x == 0) gtap::MergesortTable<0u>::block_init(S);
    __syncthreads();
    if (threadIdx.x == 0) gtap::ms_merge_tma(s, d, 0, n / 2, n, nt, S);
}
__device__ volatile int g_done;
template <int MODE>
__global__ void __launch_bounds__(128, 4) k_env(const int* s, int* d, int n, int nt) {
    extern __shared__ __align__(128) unsigned char sm[];
    gtap::MergeSlotHolder* S = reinterpret_cast<gtap::MergeSlotHolder*>(sm);
    if (threadIdx.x == 0) { gtap::MergesortTable<0u>::block_init(S); g_done = 0; }
    __syncthreads();
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) { gtap::ms_merge_tma(s, d, 0, n / 2, n, nt, S); g_done = 1; }
        __syncwarp();
    } else if (MODE == 2) {
        while (!g_done) __nanosleep(8192);
    }
}
__global__ void k_win(const int* s, int* d, int n) {
    if (threadIdx.x == 0) gtap::ms_merge(s, d, 0, n / 2, n);
}
int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : (1 << 22);
    std::vector<int> h(n);
    uint64_t x = 88172645463325252ull;
    for (int i = 0; i < n; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (int)(x >> 33); }
    std::sort(h.begin(), h.begin() + n / 2);
    std::sort(h.begin() + n / 2, h.end());
    std::vector<int> ref(n);
    std::merge(h.begin(), h.begin() + n / 2, h.begin() + n / 2, h.end(), ref.begin());
    int *s, *d, *fl;
    cudaMalloc(&s, n * 4); cudaMalloc(&d, n * 4); cudaMalloc(&fl, 256 << 20);
    cudaMemcpy(s, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(gtap::MergeSlotHolder));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaFuncSetAttribute(k_env<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(gtap::MergeSlotHolder));
    cudaFuncSetAttribute(k_env<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(gtap::MergeSlotHolder));
    for (int mode = 1; mode <= 2; ++mode) {
        cudaEventRecord(e0);
        if (mode == 1) k_env<1><<<1, 128, sizeof(gtap::MergeSlotHolder)>>>(s, d, n, n);
        else k_env<2><<<1, 128, sizeof(gtap::MergeSlotHolder)>>>(s, d, n, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("env mode=%d ms=%8.2f ns/elem=%6.2f %s\n", mode, ms, ms * 1e6 / n, cudaGetErrorString(cudaGetLastError()));
    }
    for (int variant = 0; variant < 2; ++variant)
        for (int flush = 0; flush < 2; ++flush) {
            if (flush) cudaMemset(fl, 1, 256 << 20);
            cudaMemset(d, 0, n * 4);
            cudaEventRecord(e0);
            if (variant == 0) k_tma<<<1, 32, sizeof(gtap::MergeSlotHolder)>>>(s, d, n, n);
            else k_win<<<1, 32>>>(s, d, n);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            std::vector<int> o(n);
            cudaMemcpy(o.data(), d, n * 4, cudaMemcpyDeviceToHost);
#ifdef GTAP_MS_PROBE_STATS
            if (variant == 0) { long long pr[8]; cudaMemcpyFromSymbol(pr, gtap::gtap_ms_probe, sizeof(pr));
              printf("  cycles total=%lld hot=%lld stretches=%lld fast_steps=%lld checked=%lld\n", pr[0], pr[1], pr[2], pr[3], pr[4]); }
#endif
            printf("%s flush=%d n=%d ms=%8.2f ns/elem=%6.2f ok=%d %s\n", variant ? "window" : "tma   ", flush, n, ms,
                   ms * 1e6 / n, (int)(o == ref), cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
