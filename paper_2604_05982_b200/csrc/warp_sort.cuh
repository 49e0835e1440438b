// warp_sort.cuh -- warp-cooperative sort / merge building blocks for warp-assisted task bodies
// (R28): a register bitonic sort of <= 256 keys (leaf sorts) and a bitonic merge network
// for two sorted runs of <= 1024 keys in total. All 32 lanes call them; keys are int32 and the
// padding is INT32_MAX (equal keys are indistinguishable, so the output equals a stable sort/merge).
#pragma once
#include <climits>
#include <cstdint>

namespace gtap {

// all 32 lanes: sort the x[k] (element k * 32 + lane) ascending by a bitonic network (shuffles
// for partners in other lanes, register compare-exchange for partners in the same lane)
template <int K>
__device__ __forceinline__ void warp_bitonic(int32_t (&x)[K], uint32_t lane) {
    constexpr int N = 32 * K;
#pragma unroll
    for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int kk = k ^ (stride >> 5);
                    if (kk > k) {
                        const bool up = (((uint32_t)k * 32u + lane) & (uint32_t)size) == 0u;
                        const int32_t a = x[k], b = x[kk];
                        const bool sw = up ? (a > b) : (a < b);
                        x[k] = sw ? b : a;
                        x[kk] = sw ? a : b;
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int32_t p = __shfl_xor_sync(0xffffffffu, x[k], stride);
                    const bool up = (((uint32_t)k * 32u + lane) & (uint32_t)size) == 0u;
                    const bool lower = (lane & (uint32_t)stride) == 0u;
                    x[k] = (lower == up) ? min(x[k], p) : max(x[k], p);
                }
            }
        }
    }
}

// all 32 lanes: src[l, r) sorted into dst[l, r) (r - l <= 32 K), padded with INT32_MAX
template <int K>
__device__ __noinline__ void warp_leaf_sort_k(const int32_t* __restrict__ src, int32_t* __restrict__ dst, uint32_t l,
                                              uint32_t r, uint32_t lane) {
    const uint32_t n = r - l;
    int32_t x[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t i = (uint32_t)k * 32u + lane;
        x[k] = i < n ? src[l + i] : INT_MAX;
    }
    warp_bitonic<K>(x, lane);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint32_t i = (uint32_t)k * 32u + lane;
        if (i < n) dst[l + i] = x[k];
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

// G independent problems interleaved stage by stage (batched warp assists): the G networks'
// shuffles and compare-exchanges of one stage are independent, so a warp keeps G problems' loads
// and shuffle latencies in flight instead of one. x[g][k] is element k * 32 + lane of problem g.
template <int K, int G>
__device__ __forceinline__ void warp_bitonic_sort_multi(int32_t (&x)[G][K], uint32_t lane) {
    constexpr int N = 32 * K;
#pragma unroll
    for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride >= 32) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int kk = k ^ (stride >> 5);
                    if (kk > k) {
                        const bool up = (((uint32_t)k * 32u + lane) & (uint32_t)size) == 0u;
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            const int32_t a = x[g][k], b = x[g][kk];
                            const bool sw = up ? (a > b) : (a < b);
                            x[g][k] = sw ? b : a;
                            x[g][kk] = sw ? a : b;
                        }
                    }
                }
            } else {
                const bool lower = (lane & (uint32_t)stride) == 0u;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const bool up = (((uint32_t)k * 32u + lane) & (uint32_t)size) == 0u;
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const int32_t p = __shfl_xor_sync(0xffffffffu, x[g][k], stride);
                        x[g][k] = (lower == up) ? min(x[g][k], p) : max(x[g][k], p);
                    }
                }
            }
        }
    }
}

// the merge stages of warp_merge_bitonic_k on G problems (x[g] = A ascending, padding, B reversed)
template <int K, int G>
__device__ __forceinline__ void warp_bitonic_merge_multi(int32_t (&x)[G][K], uint32_t lane) {
    constexpr uint32_t N = 32u * K;
#pragma unroll
    for (uint32_t stride = N >> 1; stride > 0; stride >>= 1) {
        if (stride >= 32u) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int kk = k ^ (int)(stride >> 5);
                if (kk > k) {
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const int32_t a = x[g][k], b = x[g][kk];
                        x[g][k] = min(a, b);
                        x[g][kk] = max(a, b);
                    }
                }
            }
        } else {
            const bool lower = (lane & stride) == 0u;
#pragma unroll
            for (int k = 0; k < K; ++k) {
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const int32_t p = __shfl_xor_sync(0xffffffffu, x[g][k], stride);
                    x[g][k] = lower ? min(x[g][k], p) : max(x[g][k], p);
                }
            }
        }
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

// all 32 lanes: src[l, r) sorted into dst[l, r) (r - l <= 32 K) by a bitonic sort in the LANE-MAJOR
// layout (element lane * K + k in x[k]): compare-exchanges at strides < K stay in registers, so a
// 128-key sort needs 15 shuffle stages instead of 25 (shuffles are the SM-shared resource here), and
// each lane loads / stores K consecutive keys (16-B accesses when aligned)
template <int K>
__device__ __noinline__ void warp_leaf_sort_lm(const int32_t* __restrict__ src, int32_t* __restrict__ dst, uint32_t l,
                                               uint32_t r, uint32_t lane) {
    static_assert(K == 4 || K == 8, "lane-major leaf sort: 4 or 8 keys per lane");
    constexpr uint32_t N = 32u * K;
    const uint32_t n = r - l, e0 = lane * (uint32_t)K;
    int32_t x[K];
    const bool vec = n == N && ((reinterpret_cast<uintptr_t>(src + l) | reinterpret_cast<uintptr_t>(dst + l)) & 15u) == 0u;
    if (vec) {
#pragma unroll
        for (int k = 0; k < K; k += 4) {
            const int4 v = *reinterpret_cast<const int4*>(src + l + e0 + k);
            x[k] = v.x; x[k + 1] = v.y; x[k + 2] = v.z; x[k + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = e0 + k < n ? src[l + e0 + k] : INT_MAX;
    }
#pragma unroll
    for (uint32_t size = 2; size <= N; size <<= 1) {
#pragma unroll
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride < (uint32_t)K) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int kk = k ^ (int)stride;
                    if (kk > k) {
                        const bool up = ((e0 + (uint32_t)k) & size) == 0u;
                        const int32_t a = x[k], b = x[kk];
                        const bool sw = up ? (a > b) : (a < b);
                        x[k] = sw ? b : a;
                        x[kk] = sw ? a : b;
                    }
                }
            } else {
                const uint32_t ls = stride / (uint32_t)K;
                const bool lower = (lane & ls) == 0u;
                const bool up = (e0 & size) == 0u;   // same for every k of the lane (size > K)
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int32_t p = __shfl_xor_sync(0xffffffffu, x[k], ls);
                    x[k] = (lower == up) ? min(x[k], p) : max(x[k], p);
                }
            }
        }
    }
    if (vec) {
#pragma unroll
        for (int k = 0; k < K; k += 4)
            *reinterpret_cast<int4*>(dst + l + e0 + k) = make_int4(x[k], x[k + 1], x[k + 2], x[k + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (e0 + k < n) dst[l + e0 + k] = x[k];
    }
}

#ifndef GTAP_LEAF_LANE_MAJOR
#define GTAP_LEAF_LANE_MAJOR 0   // 1: lane-major bitonic leaf sort (fewer shuffles; measured slower: 1.72 vs 1.65 ms at 2^24)
#endif
__device__ __forceinline__ void warp_leaf_sort(const int32_t* src, int32_t* dst, uint32_t l, uint32_t r,
                                               uint32_t lane) {
    const uint32_t n = r - l;
    if (n <= 32u) warp_leaf_sort_k<1>(src, dst, l, r, lane);
    else if (n <= 64u) warp_leaf_sort_k<2>(src, dst, l, r, lane);
    else if (n <= 128u) { if (GTAP_LEAF_LANE_MAJOR) warp_leaf_sort_lm<4>(src, dst, l, r, lane); else warp_leaf_sort_k<4>(src, dst, l, r, lane); }
    else { if (GTAP_LEAF_LANE_MAJOR) warp_leaf_sort_lm<8>(src, dst, l, r, lane); else warp_leaf_sort_k<8>(src, dst, l, r, lane); }
}

}  // namespace gtap
