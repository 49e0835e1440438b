// table_mergesort.cu -- cutoff mergesort task table (thread-level).
//
// PAPER.md P:153-165 (Prog. cutoff mergesort) with the state machine of
// P:59-74:  case 0: if (right - left <= CUTOFF) { sequential_sort; return; }
//                   mid = (left + right) / 2; fork [left, mid), [mid, right);
//                   store_state(1); return;
//           case 1: merge(data, left, mid, right); return;
// Readings: half-open ranges, mid = l + (r - l) / 2 (R14);
// sequential_sort = insertion sort, merge = two-pointer stable merge (R15).
//
// B200 layout choice (not in the paper): ping-pong buffers by depth. A task
// at depth e leaves its sorted range in buf(e) = (e even ? keys : scratch):
// a leaf sorts keys[l, r) into buf(e); an internal task merges its two
// children's ranges from buf(e + 1) into buf(e). Every key is read and
// written exactly once per tree level (8 B/key/level, no copy-back), and the
// root (depth 0) ends in `keys`. The output is the unique sorted permutation
// either way. Payload: d[0] = l, d[1] = r, d[2] = depth.
#include "table_common.cuh"

namespace gtap {

constexpr int kMsMaxCutoff = 256;

struct MergesortTable {
    static constexpr uint32_t kKind = GTAP_WORKER_THREAD;
    static constexpr int kMaxChildren = 2;
    static constexpr bool kTaskwait = true;
    static constexpr uint32_t kNumFn = 1;
    struct Args {
        int32_t* keys;
        int32_t* scratch;
        uint32_t cutoff;
        uint32_t pad;
    };

    __device__ __forceinline__ static int32_t* buf(const Args& a, uint32_t depth) {
        return (depth & 1u) ? a.scratch : a.keys;
    }

    // sequential_sort: insertion sort of src[l, r) into dst[l, r).
    __device__ __noinline__ static void leaf_sort(const int32_t* __restrict__ src, int32_t* __restrict__ dst,
                                                  uint32_t l, uint32_t r) {
        int32_t t[kMsMaxCutoff];
        const uint32_t n = r - l;
        for (uint32_t i = 0; i < n; ++i) {
            const int32_t v = src[l + i];
            int32_t j = (int32_t)i - 1;
            while (j >= 0 && t[j] > v) {
                t[j + 1] = t[j];
                --j;
            }
            t[j + 1] = v;
        }
        for (uint32_t i = 0; i < n; ++i) dst[l + i] = t[i];
    }

    // merge: stable merge of src[l, m) and src[m, r) into dst[l, r).
    // One thread, two independent chains: the front chain emits the
    // ceil(n/2) smallest keys (ties -> left run first), the back chain the
    // floor(n/2) largest (ties -> right run first), so the result equals the
    // plain two-pointer merge. Each run is read through a 4-key register
    // window refilled one key ahead, with L1 prefetches 128 B further out,
    // so the dependent chain is compare + select rather than load latency.
    __device__ __noinline__ static void merge(const int32_t* __restrict__ src, int32_t* __restrict__ dst, uint32_t l,
                                              uint32_t m, uint32_t r) {
        const long long PINF = 0x7fffffffffffffffll, NINF = (long long)0x8000000000000000ull;
        const uint32_t n = r - l;
        const uint32_t nf = (n + 1u) >> 1, nb = n - nf;
        // front chain state: A = [l, m), B = [m, r), windows a0..a3 / b0..b3
        uint32_t ia = l, ib = m;
        auto ldA = [&](uint32_t i) -> long long { return i < m ? (long long)src[i] : PINF; };
        auto ldB = [&](uint32_t i) -> long long { return i < r ? (long long)src[i] : PINF; };
        long long a0 = ldA(ia), a1 = ldA(ia + 1), a2 = ldA(ia + 2), a3 = ldA(ia + 3);
        long long b0 = ldB(ib), b1 = ldB(ib + 1), b2 = ldB(ib + 2), b3 = ldB(ib + 3);
        // back chain state: A' = A from the top, B' = B from the top
        int32_t ja = (int32_t)m - 1, jb = (int32_t)r - 1;
        auto ldA2 = [&](int32_t i) -> long long { return i >= (int32_t)l ? (long long)src[i] : NINF; };
        auto ldB2 = [&](int32_t i) -> long long { return i >= (int32_t)m ? (long long)src[i] : NINF; };
        long long c0 = ldA2(ja), c1 = ldA2(ja - 1), c2 = ldA2(ja - 2), c3 = ldA2(ja - 3);
        long long e0 = ldB2(jb), e1 = ldB2(jb - 1), e2 = ldB2(jb - 2), e3 = ldB2(jb - 3);
        uint32_t kf = l;
        uint32_t kb = r - 1u;
        for (uint32_t s = 0; s < nb; ++s) {
            // front: take B only if strictly smaller (stable: left first on ties)
            if (b0 < a0) {
                dst[kf] = (int32_t)b0;
                b0 = b1; b1 = b2; b2 = b3;
                ++ib;
                b3 = ldB(ib + 3);
                if (((ib + 3) & 31u) == 0u && ib + 35 < r) asm volatile("prefetch.global.L1 [%0];" ::"l"(src + ib + 35));
            } else {
                dst[kf] = (int32_t)a0;
                a0 = a1; a1 = a2; a2 = a3;
                ++ia;
                a3 = ldA(ia + 3);
                if (((ia + 3) & 31u) == 0u && ia + 35 < m) asm volatile("prefetch.global.L1 [%0];" ::"l"(src + ia + 35));
            }
            ++kf;
            // back: take A only if strictly larger (stable: right last on ties)
            if (c0 > e0) {
                dst[kb] = (int32_t)c0;
                c0 = c1; c1 = c2; c2 = c3;
                --ja;
                c3 = ldA2(ja - 3);
                if (((uint32_t)(ja - 3) & 31u) == 31u && ja - 35 >= (int32_t)l) asm volatile("prefetch.global.L1 [%0];" ::"l"(src + ja - 35));
            } else {
                dst[kb] = (int32_t)e0;
                e0 = e1; e1 = e2; e2 = e3;
                --jb;
                e3 = ldB2(jb - 3);
                if (((uint32_t)(jb - 3) & 31u) == 31u && jb - 35 >= (int32_t)m) asm volatile("prefetch.global.L1 [%0];" ::"l"(src + jb - 35));
            }
            --kb;
        }
        if (nf > nb) dst[kf] = (int32_t)(b0 < a0 ? b0 : a0);
    }

    __device__ __forceinline__ static void exec(const Args& a, uint32_t fn, uint32_t state,
                                                const uint32_t (&d)[kDataWords], TOut<kMaxChildren>& o) {
        if (fn != 0u) { o.bad_state(); return; }
        const uint32_t l = d[0], r = d[1], depth = d[2];
        switch (state) {
            case 0:
                if (r - l <= a.cutoff) {
                    leaf_sort(a.keys, buf(a, depth), l, r);
                    o.finish_void();
                    return;
                } else {
                    const uint32_t m = l + (r - l) / 2u;
                    o.spawn(0, 0u, l, m, depth + 1u);         // fork [l, m)
                    o.spawn(1, 0u, m, r, depth + 1u);         // fork [m, r)
                    o.suspend(1);                             // join
                    return;
                }
            case 1: {
                const uint32_t m = l + (r - l) / 2u;
                merge(buf(a, depth + 1u), buf(a, depth), l, m, r);
                o.finish_void();
                return;
            }
            default:
                o.bad_state();
        }
    }
};

static int validate_ms(const gtap_task_table* t, uint32_t fn, const uint32_t* d) {
    (void)t;
    return (fn == 0u && d[0] <= d[1] && d[2] == 0u) ? 0 : -1;
}

}  // namespace gtap

extern "C" const gtap_task_table* gtap_table_mergesort(int32_t* keys, int32_t* scratch, uint64_t n, int32_t cutoff) {
    if (((!keys || !scratch) && n > 0) || cutoff < 1 || cutoff > gtap::kMsMaxCutoff || n >= (1ull << 31)) return nullptr;
    gtap::MergesortTable::Args a{keys, scratch, (uint32_t)cutoff, 0u};
    return gtap::make_table<gtap::MergesortTable>("mergesort", a, &gtap::validate_ms);
}
