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


// One thread merges src[l, m) and src[m, r) into dst[l, r) (thread-executed
// task; the paper's merge is "largely sequential and executed by a
// single thread-level worker"). Two independent dependency chains run
// interleaved: the front chain emits the ceil(n/2) smallest keys (ties: left
// run first), the back chain the floor(n/2) largest (ties: right run last), so
// the output equals the plain two-pointer stable merge. In long stretches
// where no run can end, each chain reads its runs through 4-key register
// windows refilled 4 keys ahead (no bounds checks, no sentinels) with L1
// prefetches 512 B further out; near the run ends a checked scalar step is used.
__device__ __noinline__ void ms_merge(const int32_t* __restrict__ src, int32_t* __restrict__ dst, uint32_t l,
                                      uint32_t m, uint32_t r) {
    const uint32_t n = r - l;
    const uint32_t nf = (n + 1u) >> 1, nb = n - nf;
    uint32_t ia = l, ib = m, kf = l;          // front chain
    int32_t ja = (int32_t)m - 1, jb = (int32_t)r - 1;  // back chain (inclusive tails)
    uint32_t kb = r - 1u;
    uint32_t done = 0;                         // paired steps done (front and back each)
    while (done < nb) {
        // unchecked steps available: every window refill index stays inside its run
        int64_t S = (int64_t)min(min(m - ia, r - ib), min((uint32_t)(ja - (int32_t)l + 1), (uint32_t)(jb - (int32_t)m + 1))) - 5;
        S = min(S, (int64_t)(nb - done));
        if (S >= 16) {
            int32_t a0 = src[ia], a1 = src[ia + 1], a2 = src[ia + 2], a3 = src[ia + 3];
            int32_t b0 = src[ib], b1 = src[ib + 1], b2 = src[ib + 2], b3 = src[ib + 3];
            int32_t c0 = src[ja], c1 = src[ja - 1], c2 = src[ja - 2], c3 = src[ja - 3];
            int32_t e0 = src[jb], e1 = src[jb - 1], e2 = src[jb - 2], e3 = src[jb - 3];
            const uint32_t steps = (uint32_t)S;
            for (uint32_t t = 0; t < steps; ++t) {
                if ((t & 7u) == 0u) {
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(src + min(ia + 128u, m - 1u)));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(src + min(ib + 128u, r - 1u)));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(src + max(ja - 128, (int32_t)l)));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(src + max(jb - 128, (int32_t)m)));
                }
                if (b0 < a0) {  // front: right run only if strictly smaller
                    dst[kf] = b0; b0 = b1; b1 = b2; b2 = b3; b3 = src[ib + 4]; ++ib;
                } else {
                    dst[kf] = a0; a0 = a1; a1 = a2; a2 = a3; a3 = src[ia + 4]; ++ia;
                }
                ++kf;
                if (c0 > e0) {  // back: left run only if strictly larger
                    dst[kb] = c0; c0 = c1; c1 = c2; c2 = c3; c3 = src[ja - 4]; --ja;
                } else {
                    dst[kb] = e0; e0 = e1; e1 = e2; e2 = e3; e3 = src[jb - 4]; --jb;
                }
                --kb;
            }
            done += steps;
        } else {
            // checked scalar step for each chain
            const bool takeB = ib < r && (ia >= m || src[ib] < src[ia]);
            dst[kf++] = takeB ? src[ib++] : src[ia++];
            const bool takeA = ja >= (int32_t)l && (jb < (int32_t)m || src[ja] > src[jb]);
            dst[kb--] = takeA ? src[ja--] : src[jb--];
            ++done;
        }
    }
    if (nf > nb) {
        const bool takeB = ib < r && (ia >= m || src[ib] < src[ia]);
        dst[kf] = takeB ? src[ib] : src[ia];
    }
}

struct MergesortTable {
    static constexpr uint32_t kKind = GTAP_WORKER_THREAD;
    static constexpr int kMaxChildren = 2;
    static constexpr bool kTaskwait = true;
    static constexpr uint32_t kNumFn = 1;
    static constexpr int kMaxThreads = 128, kMinBlocks = 4;  // __launch_bounds__: 128 regs, no spills
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
    __device__ __forceinline__ static void merge(const int32_t* src, int32_t* dst, uint32_t l, uint32_t m,
                                                 uint32_t r) {
        ms_merge(src, dst, l, m, r);
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
