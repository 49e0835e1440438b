// table_nqueens.cu -- N-Queens task table (thread-level, no taskwait).
//
// PAPER.md P:465 ("count solutions via bitmask-based backtracking with a fixed
// cutoff depth (7)"), P:476 (-DGTAP_ASSUME_NO_TASKWAIT), P:484 (grid 2000 x 32):
//   nq(row, cols, d1, d2): if row == n or row >= cutoff: count serially;
//                          else spawn nq on every free column of `row`.
// No taskwait: tasks carry no join metadata and the counts are
// summed into one 64-bit device counter (red.add). Children are described by a
// generator (the parent's masks + the free-column mask): the scheduler writes
// child c from the c-th set bit, so n children cost no per-child registers.
// Diagonal masks are left unmasked (bits beyond the board fall off the
// `avail` mask). Payload: d[0] = row, d[1] = cols, d[2] = d1, d[3] = d2.
#include "table_common.cuh"

namespace gtap {

constexpr int kNqMax = 20;

__device__ __noinline__ unsigned long long nq_serial(uint32_t full, uint32_t rows_left, uint32_t cols, uint32_t d1,
                                                     uint32_t d2) {
    if (rows_left == 0) return 1ull;
    uint32_t avail = ~(cols | d1 | d2) & full;
    unsigned long long c = 0;
    while (avail) {
        const uint32_t bit = avail & (0u - avail);
        avail ^= bit;
        c += nq_serial(full, rows_left - 1u, cols | bit, (d1 | bit) << 1, (d2 | bit) >> 1);
    }
    return c;
}

// Iterative count (one lane): the same search as nq_serial as a flat loop over an explicit stack,
// so lanes at different depths still run the same instructions (recursion diverges at every call).
// The last row is counted with one popcount.
__device__ __forceinline__ unsigned long long nq_iter(uint32_t full, uint32_t rows, uint32_t c0, uint32_t e0,
                                                      uint32_t f0) {
    if (rows == 0u) return 1ull;
    uint32_t sc[kNqMax], se[kNqMax], sf[kNqMax], sa[kNqMax];
    int sp = 0;
    sc[0] = c0; se[0] = e0; sf[0] = f0; sa[0] = ~(c0 | e0 | f0) & full;
    unsigned long long cnt = 0;
    while (sp >= 0) {
        const uint32_t av = sa[sp];
        if ((uint32_t)sp + 1u == rows) { cnt += (uint32_t)__popc(av); --sp; continue; }
        if (av == 0u) { --sp; continue; }
        const uint32_t bit = av & (0u - av);
        sa[sp] = av ^ bit;
        const uint32_t c = sc[sp] | bit, e = (se[sp] | bit) << 1, f = (sf[sp] | bit) >> 1;
        ++sp;
        sc[sp] = c; se[sp] = e; sf[sp] = f; sa[sp] = ~(c | e | f) & full;
    }
    return cnt;
}

struct NqArgs {
    unsigned long long* count;
    uint32_t n;
    uint32_t cutoff;
    uint32_t mode;      // 0: serial leaf on the task's lane; 1: the warp counts the leaf (warp assist)
    uint32_t pad;
};

// all 32 lanes: count the completions of the leaf (row, cols, d1, d2). The warp expands two rows
// (lane i takes the i-th free column of the first, a warp scan numbers the pairs), then lanes
// take the pairs round robin and count each with nq_iter; one warp reduction, one red.add.
__device__ __noinline__ void nq_warp_leaf(const NqArgs& a, uint32_t row, uint32_t cols, uint32_t d1, uint32_t d2,
                                          uint32_t lane) {
    const uint32_t full = (a.n >= 32u) ? 0xFFFFFFFFu : ((1u << a.n) - 1u);
    const uint32_t rows = a.n - row;
    unsigned long long cnt = 0;
    if (rows <= 2u) {
        if (lane == 0) cnt = nq_iter(full, rows, cols, d1, d2);
    } else {
        const uint32_t av0 = ~(cols | d1 | d2) & full;
        const uint32_t p1 = __fns(av0, 0u, (int)lane + 1);
        uint32_t c1 = 0, e1 = 0, f1 = 0, av1 = 0, k = 0;
        if (p1 != 0xFFFFFFFFu) {
            const uint32_t b = 1u << p1;
            c1 = cols | b; e1 = (d1 | b) << 1; f1 = (d2 | b) >> 1;
            av1 = ~(c1 | e1 | f1) & full;
            k = (uint32_t)__popc(av1);
        }
        uint32_t incl = k;
#pragma unroll
        for (uint32_t o = 1; o < 32u; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - k;
        for (uint32_t base = 0; base < total; base += 32u) {   // uniform trip count
            const uint32_t q = base + lane;
            uint32_t j = 0;                                     // owner: the last lane with excl <= q
#pragma unroll
            for (uint32_t st = 16; st >= 1u; st >>= 1) {
                const uint32_t ex = __shfl_sync(0xffffffffu, excl, j + st);
                if (ex <= q) j += st;
            }
            const uint32_t oc = __shfl_sync(0xffffffffu, c1, j), oe = __shfl_sync(0xffffffffu, e1, j);
            const uint32_t of = __shfl_sync(0xffffffffu, f1, j), oa = __shfl_sync(0xffffffffu, av1, j);
            const uint32_t ox = __shfl_sync(0xffffffffu, excl, j);
            if (q < total) {
                const uint32_t b2 = 1u << __fns(oa, 0u, (int)(q - ox) + 1);
                cnt += nq_iter(full, rows - 2u, oc | b2, (oe | b2) << 1, (of | b2) >> 1);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0 && cnt) dev::red_add_relaxed(a.count, cnt);
}

// MODE 0: the paper's serial leaf on the task's lane; MODE 1: the warp counts each leaf
template <uint32_t MODE>
struct NQueensTable {
    static constexpr uint32_t kKind = GTAP_WORKER_THREAD;
    static constexpr bool kAssist = MODE == 1u;
    static constexpr int kMaxChildren = kNqMax;
    static constexpr bool kTaskwait = false;
    static constexpr bool kHasHeavy = false;
    static constexpr bool kGenChildren = true;
    static constexpr uint32_t kNumFn = 1;
    static constexpr bool kJoinReduceAdd = false;
    static constexpr int kMaxThreads = 256, kMinBlocks = 2;  // __launch_bounds__
    using Args = NqArgs;
    struct BlockExtra {
        uint32_t unused;
    };
    __device__ __forceinline__ static void block_init(BlockExtra*) {}

    // child c: place a queen on the c-th free column of the parent's row
    __device__ __forceinline__ static void gen_child(const uint32_t (&g)[kDataWords], uint32_t gmask, uint32_t c,
                                                     uint32_t& fn, uint32_t& q, uint32_t (&d)[kDataWords]) {
        uint32_t m = gmask;
        for (uint32_t i = 0; i < c; ++i) m &= m - 1u;  // drop the c lowest set bits
        const uint32_t bit = m & (0u - m);
        fn = 0u;
        q = 0u;
        d[0] = g[0] + 1u;
        d[1] = g[1] | bit;
        d[2] = (g[2] | bit) << 1;
        d[3] = (g[3] | bit) >> 1;
    }

    __device__ __forceinline__ static bool assist(const Args& a, const uint32_t (&ap)[kDataWords], uint32_t lane,
                                                  BlockExtra*) {
        nq_warp_leaf(a, ap[0], ap[1], ap[2], ap[3], lane);
        return true;
    }
    __device__ __forceinline__ static void help(const Args&, uint32_t, BlockExtra*) {}
    __device__ __forceinline__ static bool help_idle(const Args&, uint32_t, BlockExtra*) { return false; }

    __device__ __forceinline__ static void exec(const Args& a, uint32_t fn, uint32_t state,
                                                const uint32_t (&d)[kDataWords], TOut<1>& o, BlockExtra*) {
        if (fn != 0u || state != 0u) { o.bad_state(); return; }
        const uint32_t row = d[0];
        const uint32_t full = (a.n >= 32u) ? 0xFFFFFFFFu : ((1u << a.n) - 1u);
        if (row >= a.n || row >= a.cutoff) {               // cutoff: serial backtracking
            if constexpr (MODE == 1u) {
                o.request_assist(d[0], d[1], d[2], d[3]);
            } else {
                const unsigned long long c = nq_serial(full, a.n - row, d[1], d[2], d[3]);
                if (c) dev::red_add_relaxed(a.count, c);
            }
            o.finish_void();
            return;
        }
        const uint32_t avail = ~(d[1] | d[2] | d[3]) & full;
        o.gen[0] = d[0]; o.gen[1] = d[1]; o.gen[2] = d[2]; o.gen[3] = d[3];
        o.gmask = avail;
        o.nchild = (uint32_t)__popc(avail);                 // one task per free column
        o.finish_void();                                    // no taskwait
    }
};

static int validate_nq(const gtap_task_table*, uint32_t fn, const uint32_t* d) {
    return (fn == 0u && d[0] == 0u && d[1] == 0u && d[2] == 0u && d[3] == 0u) ? 0 : -1;
}

}  // namespace gtap

// N-Queens: board n (1..20), cutoff depth (rows placed as tasks), d_count: caller-owned
// unsigned long long on the device, incremented by the run (zero it before). fn 0, root args {}.
extern "C" const gtap_task_table* gtap_table_nqueens_ex(int32_t n, int32_t cutoff, unsigned long long* d_count,
                                                       uint32_t leaf_mode) {
    if (n < 1 || n > gtap::kNqMax || cutoff < 0 || !d_count || leaf_mode > 1u) return nullptr;
    gtap::NqArgs a{d_count, (uint32_t)n, (uint32_t)cutoff, leaf_mode, 0u};
    return leaf_mode == 1u ? gtap::make_table<gtap::NQueensTable<1u>>("nqueens_warp", a, &gtap::validate_nq)
                           : gtap::make_table<gtap::NQueensTable<0u>>("nqueens", a, &gtap::validate_nq);
}

extern "C" const gtap_task_table* gtap_table_nqueens(int32_t n, int32_t cutoff, unsigned long long* d_count) {
    return gtap_table_nqueens_ex(n, cutoff, d_count, 1u);
}
