// table_cilksort.cu -- Cilksort task table (thread-level): mergesort whose
// merge is itself fork-join.
//
// fn 0 sort(l, r, depth):  case 0: r - l <= CUTOFF_SORT -> insertion sort into
//                                  buf(depth); else fork sort halves; join(1)
//                          case 1: fork merge([l, m), [m, r)) from buf(depth+1)
//                                  into buf(depth); join(2)
//                          case 2: finish            (two taskwaits)
// fn 1 merge(A = [a0, a1) of the left run, B = [b0, b1) of the right run, m):
//                          writes dst[a0 + b0 - m, ...); <= CUTOFF_MERGE keys ->
//                          two-pointer merge; else split the longer run at its
//                          middle, binary-search the other run, fork both halves,
//                          join(1), finish.
// Split rule, cutoffs (64 / 256) and ping-pong by depth as in the
// oracle (reading R26). The merge payload packs a0, a1, b0, b1, m (25 bits
// each) and the destination parity into the 16-B record payload: n < 2^25.
#include "table_common.cuh"
#include "warp_sort.cuh"

namespace gtap {

constexpr uint32_t kCsMaxSortCut = 256;

struct MergeDesc {
    uint32_t a0, a1, b0, b1, m, p;
};
__device__ __forceinline__ void pack_merge(const MergeDesc& x, uint32_t (&d)[kDataWords]) {
    const unsigned long long lo = (unsigned long long)x.a0 | ((unsigned long long)x.a1 << 25) |
                                  ((unsigned long long)(x.b0 & 0x3FFFu) << 50);
    const unsigned long long hi = (unsigned long long)(x.b0 >> 14) | ((unsigned long long)x.b1 << 11) |
                                  ((unsigned long long)x.m << 36) | ((unsigned long long)x.p << 61);
    d[0] = (uint32_t)lo; d[1] = (uint32_t)(lo >> 32); d[2] = (uint32_t)hi; d[3] = (uint32_t)(hi >> 32);
}
__device__ __forceinline__ MergeDesc unpack_merge(const uint32_t (&d)[kDataWords]) {
    const unsigned long long lo = (unsigned long long)d[0] | ((unsigned long long)d[1] << 32);
    const unsigned long long hi = (unsigned long long)d[2] | ((unsigned long long)d[3] << 32);
    const uint32_t M25 = (1u << 25) - 1u;
    MergeDesc x;
    x.a0 = (uint32_t)lo & M25;
    x.a1 = (uint32_t)(lo >> 25) & M25;
    x.b0 = (uint32_t)(lo >> 50) | (((uint32_t)hi & 0x7FFu) << 14);
    x.b1 = (uint32_t)(hi >> 11) & M25;
    x.m = (uint32_t)(hi >> 36) & M25;
    x.p = (uint32_t)(hi >> 61) & 1u;
    return x;
}

__device__ __noinline__ void cs_leaf_sort(const int32_t* __restrict__ src, int32_t* __restrict__ dst, uint32_t l,
                                          uint32_t r) {
    int32_t t[kCsMaxSortCut];
    const uint32_t n = r - l;
    for (uint32_t i = 0; i < n; ++i) {
        const int32_t v = src[l + i];
        int32_t j = (int32_t)i - 1;
        while (j >= 0 && t[j] > v) { t[j + 1] = t[j]; --j; }
        t[j + 1] = v;
    }
    for (uint32_t i = 0; i < n; ++i) dst[l + i] = t[i];
}

__device__ __noinline__ void cs_seq_merge(const int32_t* __restrict__ a, uint32_t na, const int32_t* __restrict__ b,
                                          uint32_t nb, int32_t* __restrict__ out) {
    uint32_t i = 0, j = 0, k = 0;
    while (i < na && j < nb) out[k++] = (b[j] < a[i]) ? b[j++] : a[i++];
    while (i < na) out[k++] = a[i++];
    while (j < nb) out[k++] = b[j++];
}

// lower bound in src[lo, hi) of the first key that is not (< v) (LE = false) / not (<= v) (LE = true),
// by one lane with 15 independent probes per round (a 16-ary search): ~log16(n) + 1 dependent round
// trips instead of log2(n) for the plain binary search -- the split is on Cilksort's critical path
// once per merge level of every sort level. Same result as the binary search (the predicate is
// monotone over a sorted run).
#ifndef GTAP_CS_KARY
#define GTAP_CS_KARY 1
#endif
template <bool LE>
__device__ __forceinline__ uint32_t cs_search(const int32_t* __restrict__ src, uint32_t lo, uint32_t hi, int32_t v) {
    auto pred = [&](int32_t x) { return LE ? (x <= v) : (x < v); };
    if (GTAP_CS_KARY) {
        while (hi - lo > 16u) {
            const uint32_t w = hi - lo;
            int32_t pv[15];
#pragma unroll
            for (int k = 1; k <= 15; ++k) pv[k - 1] = src[lo + (uint32_t)(((unsigned long long)k * w) >> 4)];
            uint32_t cnt = 0;
#pragma unroll
            for (int k = 0; k < 15; ++k) cnt += pred(pv[k]) ? 1u : 0u;
            const uint32_t nlo = cnt == 0u ? lo : lo + (uint32_t)(((unsigned long long)cnt * w) >> 4) + 1u;
            const uint32_t nhi = cnt == 15u ? hi : lo + (uint32_t)(((unsigned long long)(cnt + 1u) * w) >> 4);
            lo = nlo;
            hi = nhi;
        }
        int32_t pv[16];
        const uint32_t w = hi - lo;
#pragma unroll
        for (int k = 0; k < 16; ++k) pv[k] = (uint32_t)k < w ? src[lo + k] : 0;
        uint32_t cnt = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) cnt += ((uint32_t)k < w && pred(pv[k])) ? 1u : 0u;
        return lo + cnt;
    }
    while (lo < hi) { const uint32_t mid = lo + (hi - lo) / 2u; if (pred(src[mid])) lo = mid + 1u; else hi = mid; }
    return lo;
}

struct CsArgs {
    int32_t* keys;
    int32_t* scratch;
    uint32_t cut_sort, cut_merge;
    uint32_t mode;
    uint32_t n;         // array length (roots are validated against it)
};

// MODE: GTAP_MERGE_THREAD (0: leaf sorts and sequential merges on the task's lane) or
// GTAP_MERGE_WARP (1: those bodies run by the task's warp, R28; same task graph)
template <uint32_t MODE>
struct CilksortTable {
    static constexpr uint32_t kKind = GTAP_WORKER_THREAD;
    static constexpr bool kAssist = MODE == 1u;
#ifndef GTAP_CS_STATS_SMEM
#define GTAP_CS_STATS_SMEM 0
#endif
    static constexpr bool kStatsSmem = GTAP_CS_STATS_SMEM && MODE == 1u;  // 1: no spills at 128 registers, but measured 2 % slower
    static constexpr int kFreeStack = 0;   // own free stack measured slower here (2^24: 5.47 -> 5.24 ms without)
    static constexpr uint32_t kMergeBit = 0x80000000u;  // ap[3] bit 31 (free in the packed descriptor)
    static constexpr int kMaxChildren = 2;
    static constexpr bool kTaskwait = true;
    static constexpr bool kHasHeavy = false;
    static constexpr uint32_t kNumFn = 2;
    static constexpr bool kJoinReduceAdd = false;
    static constexpr int kMaxThreads = 256, kMinBlocks = 2;  // __launch_bounds__
    using Args = CsArgs;
    struct BlockExtra {
        uint32_t unused;
    };
    __device__ __forceinline__ static void block_init(BlockExtra*) {}
    __device__ __forceinline__ static int32_t* buf(const Args& a, uint32_t parity) {
        return parity ? a.scratch : a.keys;
    }

    // warp assist (all 32 lanes): ap = {l, r, parity, 0} for a leaf sort, the packed merge
    // descriptor with kMergeBit for a sequential merge
    __device__ __forceinline__ static bool assist(const Args& a, const uint32_t (&ap)[kDataWords], uint32_t lane,
                                                  BlockExtra*) {
        if (ap[3] & kMergeBit) {
            const uint32_t md[kDataWords] = {ap[0], ap[1], ap[2], ap[3] & ~kMergeBit};
            const MergeDesc x = unpack_merge(md);
            const int32_t* src = buf(a, x.p ^ 1u);
            int32_t* out = buf(a, x.p) + (x.a0 + x.b0 - x.m);
            const uint32_t na = x.a1 - x.a0, nb = x.b1 - x.b0;
            if (na + nb <= kBitonicMax) warp_merge_small(src + x.a0, na, src + x.b0, nb, out, lane);
            else if (lane == 0) cs_seq_merge(src + x.a0, na, src + x.b0, nb, out);
            return true;
        }
        warp_leaf_sort(a.keys, buf(a, ap[2]), ap[0], ap[1], lane);
        return true;
    }
    // no shared assist boards: the scheduler's help hooks are no-ops
    __device__ __forceinline__ static void help(const Args&, uint32_t, BlockExtra*) {}
    __device__ __forceinline__ static bool help_idle(const Args&, uint32_t, BlockExtra*) { return false; }

    __device__ __forceinline__ static void exec(const Args& a, uint32_t fn, uint32_t state,
                                                const uint32_t (&d)[kDataWords], TOut<kMaxChildren>& o,
                                                BlockExtra*) {
        if (fn == 0u) {  // sort
            const uint32_t l = d[0], r = d[1], depth = d[2];
            const uint32_t m = l + (r - l) / 2u;
            switch (state) {
                case 0:
                    if (r - l <= a.cut_sort) {
                        if constexpr (MODE == 1u) o.request_assist(l, r, depth & 1u, 0u);
                        else cs_leaf_sort(a.keys, buf(a, depth & 1u), l, r);
                        o.finish_void();
                    } else {
                        o.spawn(0, 0u, l, m, depth + 1u);
                        o.spawn(1, 0u, m, r, depth + 1u);
                        o.suspend(1);
                    }
                    return;
                case 1: {  // both halves sorted in buf(depth + 1): one parallel merge into buf(depth)
                    uint32_t md[kDataWords];
                    pack_merge(MergeDesc{l, m, m, r, m, depth & 1u}, md);
                    o.spawn(0, 1u, md[0], md[1], md[2], md[3]);
                    o.suspend(2);
                    return;
                }
                case 2:
                    o.finish_void();
                    return;
                default:
                    o.bad_state();
                    return;
            }
        }
        if (fn == 1u) {  // merge
            if (state == 1u) { o.finish_void(); return; }
            if (state != 0u) { o.bad_state(); return; }
            const MergeDesc x = unpack_merge(d);
            const int32_t* src = buf(a, x.p ^ 1u);
            int32_t* dst = buf(a, x.p);
            const uint32_t na = x.a1 - x.a0, nb = x.b1 - x.b0;
            if (na + nb <= a.cut_merge) {
                if constexpr (MODE == 1u) o.request_assist(d[0], d[1], d[2], d[3] | kMergeBit);
                else cs_seq_merge(src + x.a0, na, src + x.b0, nb, dst + (x.a0 + x.b0 - x.m));
                o.finish_void();
                return;
            }
            uint32_t sa, sb;
            if (na >= nb) {  // split the left run at its middle; B keys < A[sa] go left
                sa = x.a0 + na / 2u;
                sb = cs_search<false>(src, x.b0, x.b1, src[sa]);
            } else {         // split the right run at its middle; A keys <= B[sb] go left
                sb = x.b0 + nb / 2u;
                sa = cs_search<true>(src, x.a0, x.a1, src[sb]);
            }
            uint32_t c0[kDataWords], c1[kDataWords];
            pack_merge(MergeDesc{x.a0, sa, x.b0, sb, x.m, x.p}, c0);
            pack_merge(MergeDesc{sa, x.a1, sb, x.b1, x.m, x.p}, c1);
            o.spawn(0, 1u, c0[0], c0[1], c0[2], c0[3]);
            o.spawn(1, 1u, c1[0], c1[1], c1[2], c1[3]);
            o.suspend(1);
            return;
        }
        o.bad_state();
    }
};

// a root {l, r} must lie inside keys[0, n) (n < 2^25: the packed merge descriptor's index width)
static int validate_cs(const gtap_task_table* t, uint32_t fn, const uint32_t* d) {
    CsArgs a;
    std::memcpy(&a, t->args, sizeof(a));
    return (fn == 0u && d[0] <= d[1] && d[1] <= a.n && d[2] == 0u) ? 0 : -1;
}

}  // namespace gtap

// Cilksort: keys/scratch int32[n] device buffers, n < 2^25; cut_sort in [1, 256],
// cut_merge >= 2 (paper: 64 / 256). fn 0 = sort, root args {uint32 l, uint32 r} (normally {0, n}).
extern "C" const gtap_task_table* gtap_table_cilksort_ex(int32_t* keys, int32_t* scratch, uint64_t n,
                                                         int32_t cut_sort, int32_t cut_merge, uint32_t merge_mode) {
    if (((!keys || !scratch) && n > 0) || n >= (1ull << 25) || cut_sort < 1 ||
        cut_sort > (int32_t)gtap::kCsMaxSortCut || cut_merge < 2 || merge_mode > 1u)
        return nullptr;
    gtap::CsArgs a{keys, scratch, (uint32_t)cut_sort, (uint32_t)cut_merge, merge_mode, (uint32_t)n};
    return merge_mode == 1u ? gtap::make_table<gtap::CilksortTable<1u>>("cilksort_warp", a, &gtap::validate_cs)
                            : gtap::make_table<gtap::CilksortTable<0u>>("cilksort", a, &gtap::validate_cs);
}

extern "C" const gtap_task_table* gtap_table_cilksort(int32_t* keys, int32_t* scratch, uint64_t n, int32_t cut_sort,
                                                      int32_t cut_merge) {
    return gtap_table_cilksort_ex(keys, scratch, n, cut_sort, cut_merge, 1u);
}
