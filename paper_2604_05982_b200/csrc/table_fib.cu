// table_fib.cu -- Fibonacci task table (thread-level, no cutoff).
//
// PAPER.md P:1023-1033 (Prog. fib) as transformed by the compiler, P:1160-1190:
//   struct fib_task_data { __cap_n; __cap_a; __cap_b; __cap_result; }
//   case 0: if (n < 2) { result = n; finish; }  spawn fib(n-1), fib(n-2);
//           __gtap_prepare_for_join(1); return;
//   case 1: a = load_result(0); b = load_result(1); result = a + b; finish;
// Record payload: d[0] = n; d[2], d[3] = the children's results (written by
// the children at finish, copy-at-finish reading R8) = __cap_a / __cap_b.
#include "table_common.cuh"

namespace gtap {

struct FibTable {
    static constexpr uint32_t kKind = GTAP_WORKER_THREAD;
    static constexpr int kMaxChildren = 2;
    static constexpr bool kTaskwait = true;
    static constexpr bool kHasHeavy = false;
    static constexpr uint32_t kNumFn = 1;
    static constexpr bool kJoinReduceAdd = true;  // see TaskRec
#ifndef GTAP_FIB_FSTACK
#define GTAP_FIB_FSTACK 1024  // own free-stack depth (fib(40): 64 -> 13.1 ms, 256 -> 12.66, 1024 -> 12.45)
#endif
    static constexpr int kFreeStack = GTAP_FIB_FSTACK;
#ifndef GTAP_FIB_MINB
#define GTAP_FIB_MINB 3  // 72 regs, no spills (4: 64 regs + spills, 2% slower)
#endif
    static constexpr int kMaxThreads = 256, kMinBlocks = GTAP_FIB_MINB;  // __launch_bounds__
    struct Args {
        uint32_t unused;
    };
    struct BlockExtra {
        uint32_t unused;
    };
    __device__ __forceinline__ static void block_init(BlockExtra*) {}
    __device__ __forceinline__ static void exec(const Args&, uint32_t fn, uint32_t state,
                                                const uint32_t (&d)[kDataWords], TOut<kMaxChildren>& o,
                                                BlockExtra*) {
        if (fn != 0u) { o.bad_state(); return; }
        switch (state) {
            case 0: {
                const int32_t n = (int32_t)d[0];
                if (n < 2) { o.finish(n); return; }
                o.spawn(0, 0u, (uint32_t)(n - 1));           // a = fib(n-1)
                o.spawn(1, 0u, (uint32_t)(n - 2));           // b = fib(n-2)
                o.suspend(1);                                 // __gtap_prepare_for_join(1)
                return;
            }
            case 1:
                o.finish((int32_t)d[2] + (int32_t)d[3]);
                return;
            default:
                o.bad_state();                                // P:1188 default: __trap()
        }
    }
};

// fib with a cutoff (the EPAQ experiment): n < cutoff runs the serial
// recursion inside the task ("tasks that reach the cutoff execute additional serial work");
// otherwise spawn fib(n-1), fib(n-2) and join. With NQ = 3 the paper's queue classifier
// (P:1027-1031): non-cutoff children -> queue 0, cutoff children -> queue 1, the
// post-taskwait continuation -> queue 2. NQ = 1 is the same program without EPAQ.
__device__ __noinline__ int32_t fib_serial(int32_t n) {
    if (n < 2) return n;
    return fib_serial(n - 1) + fib_serial(n - 2);
}

template <int NQ>
struct FibCutoffTable {
    static constexpr uint32_t kKind = GTAP_WORKER_THREAD;
    static constexpr int kMaxChildren = 2;
    static constexpr bool kTaskwait = true;
    static constexpr bool kHasHeavy = false;
    static constexpr uint32_t kNumFn = 1;
    static constexpr bool kJoinReduceAdd = true;
    static constexpr int kNumQueues = NQ;
    static constexpr int kFreeStack = 0;   // own free stack measured slower here (fib(40) cutoff 10: 4.27 / 3.72 -> 4.08 / 3.58 ms without)
    static constexpr int kMaxThreads = 256, kMinBlocks = 4;  // __launch_bounds__
    struct Args {
        uint32_t cutoff;
    };
    struct BlockExtra {
        uint32_t unused;
    };
    __device__ __forceinline__ static void block_init(BlockExtra*) {}
    __device__ __forceinline__ static uint32_t qof(int32_t m, uint32_t cutoff) {
        return NQ > 1 ? (((uint32_t)m < cutoff || m < 2) ? 1u : 0u) : 0u;
    }
    __device__ __forceinline__ static void exec(const Args& a, uint32_t fn, uint32_t state,
                                                const uint32_t (&d)[kDataWords], TOut<kMaxChildren>& o,
                                                BlockExtra*) {
        if (fn != 0u) { o.bad_state(); return; }
        switch (state) {
            case 0: {
                const int32_t n = (int32_t)d[0];
                if ((uint32_t)n < a.cutoff || n < 2) { o.finish(fib_serial(n)); return; }
                o.spawn_q(0, qof(n - 1, a.cutoff), 0u, (uint32_t)(n - 1));   // queue((n-1) < cutoff ? 1 : 0)
                o.spawn_q(1, qof(n - 2, a.cutoff), 0u, (uint32_t)(n - 2));   // queue((n-2) < cutoff ? 1 : 0)
                o.suspend(1, NQ > 1 ? 2u : 0u);                               // taskwait queue(2)
                return;
            }
            case 1:
                o.finish((int32_t)d[2] + (int32_t)d[3]);
                return;
            default:
                o.bad_state();
        }
    }
};

static int validate_fib(const gtap_task_table*, uint32_t fn, const uint32_t* d) {
    const int32_t n = (int32_t)d[0];
    return (fn == 0u && n >= 0 && n <= 46) ? 0 : -1;  // fib(47) overflows int32 (reading R17)
}

}  // namespace gtap

extern "C" const gtap_task_table* gtap_table_fib(void) {
    gtap::FibTable::Args a{0};
    return gtap::make_table<gtap::FibTable>("fib", a, &gtap::validate_fib);
}

extern "C" const gtap_task_table* gtap_table_fib_cutoff(int32_t cutoff, uint32_t num_queues) {
    if (cutoff < 0 || (num_queues != 1 && num_queues != 3)) return nullptr;
    if (num_queues == 3) {
        gtap::FibCutoffTable<3>::Args a{(uint32_t)cutoff};
        return gtap::make_table<gtap::FibCutoffTable<3>>("fib_cutoff_epaq3", a, &gtap::validate_fib);
    }
    gtap::FibCutoffTable<1>::Args a{(uint32_t)cutoff};
    return gtap::make_table<gtap::FibCutoffTable<1>>("fib_cutoff", a, &gtap::validate_fib);
}

#ifdef GTAP_CYC_HIST
extern "C" int gtap_cyc_hist_read(unsigned long long* h) {   // diagnostic build only (sched_thread.cuh)
    cudaMemcpyFromSymbol(h, gtap::gtap_cyc_hist, sizeof(unsigned long long) * 40);
    unsigned long long z[40] = {};
    cudaMemcpyToSymbol(gtap::gtap_cyc_hist, z, sizeof(z));
    return 0;
}
#endif
