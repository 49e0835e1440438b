// calib.cu -- single-thread issue / latency calibration on B200
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void alu(int* out, int iters) {
    if (threadIdx.x) return;
    int a = out[0], b = out[1], c = out[2], d = out[3];
    for (int i = 0; i < iters; ++i) { a = a * 3 + b; b = b ^ (c + i); c = c + (d >> 1); d = d + a; }
    out[4] = a + b + c + d;
}
__global__ void chase(const int* __restrict__ p, int* out, int iters) {  // dependent global loads
    if (threadIdx.x) return;
    int j = 0;
    for (int i = 0; i < iters; ++i) j = p[j];
    out[0] = j;
}
__global__ void chase_smem(const int* __restrict__ p, int* out, int iters) {
    __shared__ int s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = p[i] & 4095;
    __syncthreads();
    if (threadIdx.x) return;
    int j = 0;
    for (int i = 0; i < iters; ++i) j = s[j];
    out[0] = j;
}
__global__ void stream_st(int* d, int n) {  // single thread sequential stores
    if (threadIdx.x) return;
    for (int i = 0; i < n; ++i) d[i] = i;
}
__global__ void stream_ld(const int* __restrict__ s, int* out, int n) {  // single thread sequential loads (independent)
    if (threadIdx.x) return;
    int acc = 0;
    for (int i = 0; i < n; ++i) acc += s[i];
    out[0] = acc;
}
int main() {
    int *p, *o, *big;
    const int N = 1 << 24;
    cudaMalloc(&p, N * 4); cudaMalloc(&o, 64); cudaMalloc(&big, N * 4);
    int* h = new int[N];
    uint32_t x = 12345;
    for (int i = 0; i < N; ++i) { x = x * 1664525u + 1013904223u; h[i] = (x >> 8) % (1 << 20); }  // 4 MiB working set
    cudaMemcpy(p, h, N * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
#define T(label, launch, cnt) cudaEventRecord(e0); launch; cudaEventRecord(e1); cudaEventSynchronize(e1); \
    cudaEventElapsedTime(&ms, e0, e1); printf("%-28s %8.3f ms  %7.2f ns/op  %s\n", label, ms, ms * 1e6 / (cnt), cudaGetErrorString(cudaGetLastError()));
    T("alu warmup", (alu<<<1, 32>>>(o, 1000000)), 4e6);
    T("alu 4 ops/iter", (alu<<<1, 32>>>(o, 10000000)), 4e7);
    T("chase global (4MiB, L2)", (chase<<<1, 32>>>(p, o, 1000000)), 1e6);
    T("chase smem", (chase_smem<<<1, 128>>>(p, o, 1000000)), 1e6);
    T("stream_st 16M", (stream_st<<<1, 32>>>(big, N)), N);
    T("stream_ld 16M", (stream_ld<<<1, 32>>>(big, o, N)), N);
    T("stream_ld 16M again(L2)", (stream_ld<<<1, 32>>>(big, o, N)), N);
    return 0;
}
