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
    static constexpr int kMaxThreads = 256, kMinBlocks = 4;  // __launch_bounds__
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

static int validate_fib(const gtap_task_table*, uint32_t fn, const uint32_t* d) {
    const int32_t n = (int32_t)d[0];
    return (fn == 0u && n >= 0 && n <= 46) ? 0 : -1;  // fib(47) overflows int32 (reading R17)
}

}  // namespace gtap

extern "C" const gtap_task_table* gtap_table_fib(void) {
    gtap::FibTable::Args a{0};
    return gtap::make_table<gtap::FibTable>("fib", a, &gtap::validate_fib);
}
