// warp_sort.cuh -- warp-cooperative sort / merge building blocks for warp-assisted task bodies
// (R28): a lane-major register bitonic sort of <= 256 keys (leaf sorts) and a bitonic merge network
// for two sorted runs of <= 1024 keys in total. All 32 lanes call them; keys are int32 and the
// padding is INT32_MAX (equal keys are indistinguishable, so the output equals a stable sort/merge).
#pragma once
#include <climits>
#include <cstdint>

namespace gtap {

// all 32 lanes: sort the x[k] (element lane * K + k: lane-major) ascending by a bitonic network. Partners at
// strides < K are in the same lane (register compare-exchange: log2(K) of every log2(32K) stages of a merge
// step), larger strides are lane ^ (stride / K) (one shuffle + one predicated min/max per key)
template <int K>
__device__ __forceinline__ void warp_bitonic_lm(int32_t (&x)[K], uint32_t lane) {
    constexpr int N = 32 * K;
#pragma unroll
    for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride < K) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int kk = k ^ stride;
                    if (kk > k) {
                        const bool up = ((lane * (uint32_t)K + (uint32_t)k) & (uint32_t)size) == 0u;
                        const int32_t a = x[k], b = x[kk];
                        const int32_t lo = min(a, b), hi = max(a, b);
                        x[k] = up ? lo : hi;
                        x[kk] = up ? hi : lo;
                    }
                }
            } else {
                const uint32_t ls = (uint32_t)(stride / K);
                // size > stride >= K: the direction bit is a lane bit
                const bool keep_min = ((lane & ls) == 0u) == ((lane & (uint32_t)(size / K)) == 0u);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int32_t p = __shfl_xor_sync(0xffffffffu, x[k], ls);
                    x[k] = keep_min ? min(x[k], p) : max(x[k], p);
                }
            }
        }
    }
}

// all 32 lanes: src[l, r) sorted into dst[l, r) (r - l <= 32 K), padded with INT32_MAX; lane i holds keys
// [i K, i K + K) (16-B vector loads / stores when the range is whole and 16-B aligned)
template <int K>
__device__ __noinline__ void warp_leaf_sort_k(const int32_t* __restrict__ src, int32_t* __restrict__ dst, uint32_t l,
                                              uint32_t r, uint32_t lane) {
    static_assert(K % 4 == 0, "lane-major leaves load 4-key vectors");
    const uint32_t n = r - l;
    int32_t x[K];
    const bool vec = n == 32u * K && (((uintptr_t)(src + l) | (uintptr_t)(dst + l)) & 15u) == 0u;
    if (vec) {
#pragma unroll
        for (int k = 0; k < K; k += 4) {
            const int4 v = *reinterpret_cast<const int4*>(src + l + lane * K + k);
            x[k] = v.x; x[k + 1] = v.y; x[k + 2] = v.z; x[k + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t i = lane * (uint32_t)K + (uint32_t)k;
            x[k] = i < n ? src[l + i] : INT_MAX;
        }
    }
    warp_bitonic_lm<K>(x, lane);
    if (vec) {
#pragma unroll
        for (int k = 0; k < K; k += 4)
            *reinterpret_cast<int4*>(dst + l + lane * K + k) = make_int4(x[k], x[k + 1], x[k + 2], x[k + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t i = lane * (uint32_t)K + (uint32_t)k;
            if (i < n) dst[l + i] = x[k];
        }
    }
}

// all 32 lanes: merge of A[0, na) and B[0, nb) (na + nb <= 32 K) by one bitonic merge network:
// A ascending, INT32_MAX padding, B reversed is a bitonic sequence of 32 K keys; log2(32 K) half-cleaner
// stages sort it ascending and the first r - l keys are the merge (integer keys: equal keys are
// indistinguishable, so the result is the stable merge's)
template <int K>
__device__ __noinline__ void warp_merge_bitonic_k(const int32_t* __restrict__ A, uint32_t na,
                                                  const int32_t* __restrict__ B, uint32_t nb,
                                                  int32_t* __restrict__ out, uint32_t lane) {
    constexpr uint32_t N = 32u * K;
    int32_t x[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t i = (uint32_t)k * 32u + lane;
        x[k] = i < na ? A[i] : (i >= N - nb ? B[N - 1u - i] : INT_MAX);
    }
#pragma unroll
    for (uint32_t stride = N >> 1; stride > 0; stride >>= 1) {
        if (stride >= 32u) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int kk = k ^ (int)(stride >> 5);
                if (kk > k) {
                    const int32_t a = x[k], b = x[kk];
                    x[k] = min(a, b);
                    x[kk] = max(a, b);
                }
            }
        } else {
            const bool lower = (lane & stride) == 0u;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int32_t p = __shfl_xor_sync(0xffffffffu, x[k], stride);
                x[k] = lower ? min(x[k], p) : max(x[k], p);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t i = (uint32_t)k * 32u + lane;
        if (i < na + nb) out[i] = x[k];
    }
}

constexpr uint32_t kBitonicMax = 1024;  // merges up to this many keys: one bitonic network

// all 32 lanes: A[0, na) and B[0, nb) (sorted, na + nb <= kBitonicMax) merged into out[0, na + nb)
__device__ __forceinline__ void warp_merge_small(const int32_t* A, uint32_t na, const int32_t* B, uint32_t nb,
                                                 int32_t* out, uint32_t lane) {
    const uint32_t n = na + nb;
    if (n <= 32u) warp_merge_bitonic_k<1>(A, na, B, nb, out, lane);
    else if (n <= 64u) warp_merge_bitonic_k<2>(A, na, B, nb, out, lane);
    else if (n <= 128u) warp_merge_bitonic_k<4>(A, na, B, nb, out, lane);
    else if (n <= 256u) warp_merge_bitonic_k<8>(A, na, B, nb, out, lane);
    else if (n <= 512u) warp_merge_bitonic_k<16>(A, na, B, nb, out, lane);
    else warp_merge_bitonic_k<32>(A, na, B, nb, out, lane);
}

// all 32 lanes: sequential_sort of a leaf, src[l, r) -> dst[l, r), by a register bitonic sort
__device__ __forceinline__ void warp_leaf_sort(const int32_t* src, int32_t* dst, uint32_t l, uint32_t r,
                                               uint32_t lane) {
    const uint32_t n = r - l;
    if (n <= 128u) warp_leaf_sort_k<4>(src, dst, l, r, lane);
    else warp_leaf_sort_k<8>(src, dst, l, r, lane);
}

}  // namespace gtap
