// gather_micro.cu -- the floor for SpMV on the bench matrix: stream col/val once and gather x
// (sum val[i] * x[col[i]] into per-thread accumulators; no rows, no scheduler). Matrix shape as
// synth.powerlaw_csr(2^22): nnz ~ 1.32e8 uniform random columns over 2^22 (x = 16 MB, L2-resident).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>

__global__ void k_gather(const int* __restrict__ col, const float* __restrict__ val, const float* __restrict__ x,
                         long long nnz, float* out) {
    float acc = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < nnz; i += 4 * stride) {
        int c0 = __ldcs(col + i), c1 = __ldcs(col + i + stride), c2 = __ldcs(col + i + 2 * stride), c3 = __ldcs(col + i + 3 * stride);
        float v0 = __ldcs(val + i), v1 = __ldcs(val + i + stride), v2 = __ldcs(val + i + 2 * stride), v3 = __ldcs(val + i + 3 * stride);
        acc += v0 * __ldg(x + c0) + v1 * __ldg(x + c1) + v2 * __ldg(x + c2) + v3 * __ldg(x + c3);
    }
    for (; i < nnz; i += stride) acc += __ldcs(val + i) * __ldg(x + __ldcs(col + i));
    if (acc == 12345.f) out[0] = acc;
}
__global__ void k_stream(const int* __restrict__ col, const float* __restrict__ val, long long nnz, float* out) {
    float acc = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride)
        acc += __ldcs(val + i) + (float)__ldcs(col + i);
    if (acc == 12345.f) out[0] = acc;
}
int main() {
    const long long nnz = 132124528, n = 1 << 22;
    std::vector<int> hc(nnz);
    std::mt19937 rng(1);
    for (auto& c : hc) c = rng() & (n - 1);
    int* col; float *val, *x, *out;
    cudaMalloc(&col, nnz * 4); cudaMalloc(&val, nnz * 4); cudaMalloc(&x, n * 4); cudaMalloc(&out, 4);
    cudaMemcpy(col, hc.data(), nnz * 4, cudaMemcpyHostToDevice);
    cudaMemset(val, 0, nnz * 4); cudaMemset(x, 0, n * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int blocks : {148 * 8, 148 * 16, 148 * 32}) {
        for (int it = 0; it < 3; ++it) {
            cudaEventRecord(a); k_gather<<<blocks, 256>>>(col, val, x, nnz, out); cudaEventRecord(b);
            cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
            if (it == 2) printf("gather blocks=%d: %.3f ms  algorithmic %.0f GB/s (8 B/nnz + x)\n", blocks, ms,
                                (8.0 * nnz + 12.0 * n) / ms / 1e6);
            cudaEventRecord(a); k_stream<<<blocks, 256>>>(col, val, nnz, out); cudaEventRecord(b);
            cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
            if (it == 2) printf("stream blocks=%d: %.3f ms  %.0f GB/s\n", blocks, ms, 8.0 * nnz / ms / 1e6);
        }
    }
}
