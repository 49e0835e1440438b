// warp_merge_micro.cu -- time the warp-assist merge (warp_merge) in isolation: one warp (or W
// warps on W separate problems), two sorted runs of n/2 keys; checks the output.
#include "../paper_2604_05982_b200/csrc/table_mergesort.cu"
// the table's board reset calls the runtime's fill helper (runtime.cu, not linked here)
namespace gtap {
cudaError_t zero_async(void* p, size_t bytes, cudaStream_t s) { return cudaMemsetAsync(p, 0, bytes, s); }
}  // namespace gtap
#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void __launch_bounds__(128, 1) k_wm(const int* s, int* d, int n, int nprob) {
    extern __shared__ __align__(128) unsigned char sm[];
    gtap::WarpAssistHolder* H = reinterpret_cast<gtap::WarpAssistHolder*>(sm);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t prob = blockIdx.x * (blockDim.x >> 5) + warp;
    if (prob >= (uint32_t)nprob) return;
    const uint32_t off = prob * (uint32_t)n;
    gtap::warp_merge(s, d, off, off + n / 2, off + n / 2, off + n, off, lane, H->tiles(warp));
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : (1 << 24);
    const int nprob = argc > 2 ? atoi(argv[2]) : 1;
    const int wpb = argc > 3 ? atoi(argv[3]) : 1;   // warps per block
    std::vector<int> h((size_t)n * nprob);
    uint64_t x = 88172645463325252ull;
    for (auto& v : h) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = (int)(x >> 33); }
    for (int p = 0; p < nprob; ++p) {
        std::sort(h.begin() + (size_t)p * n, h.begin() + (size_t)p * n + n / 2);
        std::sort(h.begin() + (size_t)p * n + n / 2, h.begin() + (size_t)(p + 1) * n);
    }
    int *s, *d;
    cudaMalloc(&s, h.size() * 4); cudaMalloc(&d, h.size() * 4);
    cudaMemcpy(s, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    const int smem = (int)sizeof(gtap::WarpAssistHolder);
    cudaFuncSetAttribute(k_wm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = (nprob + wpb - 1) / wpb;
    for (int it = 0; it < 3; ++it) {
        cudaEventRecord(e0);
        k_wm<<<blocks, 32 * wpb, smem>>>(s, d, n, nprob);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("n=%d nprob=%d wpb=%d  %.3f ms  %.3f ns/key/warp  %.1f Mkeys/s/warp  %s\n", n, nprob, wpb, ms,
               ms * 1e6 / n, n / ms / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    std::vector<int> o(h.size());
    cudaMemcpy(o.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    bool ok = true;
    for (int p = 0; p < nprob && ok; ++p) {
        std::vector<int> ref((size_t)n);
        std::merge(h.begin() + (size_t)p * n, h.begin() + (size_t)p * n + n / 2, h.begin() + (size_t)p * n + n / 2,
                   h.begin() + (size_t)(p + 1) * n, ref.begin());
        ok = std::equal(ref.begin(), ref.end(), o.begin() + (size_t)p * n);
    }
    printf("ok=%d\n", ok);
}
