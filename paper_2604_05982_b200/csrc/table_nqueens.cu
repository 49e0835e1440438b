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

struct NQueensTable {
    static constexpr uint32_t kKind = GTAP_WORKER_THREAD;
    static constexpr int kMaxChildren = kNqMax;
    static constexpr bool kTaskwait = false;
    static constexpr bool kHasHeavy = false;
    static constexpr bool kGenChildren = true;
    static constexpr uint32_t kNumFn = 1;
    static constexpr bool kJoinReduceAdd = false;
    static constexpr int kMaxThreads = 256, kMinBlocks = 2;  // __launch_bounds__
    struct Args {
        unsigned long long* count;
        uint32_t n;
        uint32_t cutoff;
    };
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

    __device__ __forceinline__ static void exec(const Args& a, uint32_t fn, uint32_t state,
                                                const uint32_t (&d)[kDataWords], TOut<1>& o, BlockExtra*) {
        if (fn != 0u || state != 0u) { o.bad_state(); return; }
        const uint32_t row = d[0];
        const uint32_t full = (a.n >= 32u) ? 0xFFFFFFFFu : ((1u << a.n) - 1u);
        if (row >= a.n || row >= a.cutoff) {               // cutoff: serial backtracking
            const unsigned long long c = nq_serial(full, a.n - row, d[1], d[2], d[3]);
            if (c) dev::red_add_relaxed(a.count, c);
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
extern "C" const gtap_task_table* gtap_table_nqueens(int32_t n, int32_t cutoff, unsigned long long* d_count) {
    if (n < 1 || n > gtap::kNqMax || cutoff < 0 || !d_count) return nullptr;
    gtap::NQueensTable::Args a{d_count, (uint32_t)n, (uint32_t)cutoff};
    return gtap::make_table<gtap::NQueensTable>("nqueens", a, &gtap::validate_nq);
}
