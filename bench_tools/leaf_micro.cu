// leaf_micro.cu -- the mergesort leaf body in isolation: W warps, each sorting L consecutive 128-key leaves
// (warp_leaf_sort_k<4>, k-major bitonic network) from keys into out; cold (L2 flushed) or warm input,
// and with 1 / 2 leaves in flight per warp (two independent networks interleaved). Checks sortedness.
#include "../paper_2604_05982_b200/csrc/warp_sort.cuh"
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

template <int G>
__global__ void __launch_bounds__(128, 4) k_leaf(const int* src, int* dst, int leaves_per_warp) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t base = w * leaves_per_warp * 128u;
    for (int i = 0; i < leaves_per_warp; i += G) {
        int32_t x[G][4];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int k = 0; k < 4; ++k) x[g][k] = src[base + (i + g) * 128u + k * 32u + lane];
#pragma unroll
        for (int g = 0; g < G; ++g) gtap::warp_bitonic<4>(x[g], lane);
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[base + (i + g) * 128u + k * 32u + lane] = x[g][k];
    }
}

__global__ void k_flush(int* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = (int)i;
}

int main() {
    const int W = 2368, L = 56;
    const size_t n = (size_t)W * L * 128;
    std::vector<int> h(n);
    uint64_t x = 88172645463325252ull;
    for (auto& v : h) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = (int)(x >> 33); }
    int *s, *d, *f;
    cudaMalloc(&s, n * 4); cudaMalloc(&d, n * 4); cudaMalloc(&f, (256u << 20));
    cudaMemcpy(s, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int g = 1; g <= 2; g *= 2) {
        for (int cold = 1; cold >= 0; --cold) {
            float best = 1e30f;
            for (int it = 0; it < 5; ++it) {
                if (cold) k_flush<<<1184, 256>>>(f, (256u << 20) / 4);
                cudaEventRecord(e0);
                if (g == 1) k_leaf<1><<<W / 4, 128>>>(s, d, L); else k_leaf<2><<<W / 4, 128>>>(s, d, L);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                best = std::min(best, ms);
            }
            std::vector<int> o(n);
            cudaMemcpy(o.data(), d, n * 4, cudaMemcpyDeviceToHost);
            bool ok = true;
            for (size_t b = 0; b < n && ok; b += 128) ok = std::is_sorted(o.begin() + b, o.begin() + b + 128);
            printf("G=%d %s: %.4f ms  %.3f us per leaf per warp  %.1f ns/key/warp  ok=%d %s\n", g, cold ? "cold" : "warm",
                   best, best * 1e3 / L, best * 1e6 / (L * 128.0), ok, cudaGetErrorString(cudaGetLastError()));
        }
    }
}
