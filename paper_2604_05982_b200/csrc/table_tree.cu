// table_tree.cu -- synthetic tree task tables (§6.3), one
// per worker granularity: thread-level (one task per lane) and block-level
// (one task per block, the body data-parallel over the block's threads).
//
//   node(id, depth): spawn the node's children (if any), taskwait, then
//                    do_memory_and_compute(id)
//   full binary tree: every node above depth D has children 2id, 2id+1;
//   pruned B-ary tree: child k of node id at depth d is B*id + 1 + k and
//   exists iff mix(seed ^ child) >> 11 < floor((D - d) * 2^53 / D), i.e. with
//   probability p(d) = 1 - d/D from a counter-based draw (reading R27).
//   do_memory_and_compute(id) = sum of mem_ops 64-bit words buf[mix(id*G + i) & (len-1)]
//     + bits of the final values of min(64, compute_iters) independent FMA chains
//     (chain c: compute_iters/64 + (c < compute_iters%64) FMAs), mod 2^64.
// Each task adds its value into one of 32 device counters (spread to avoid a
// single hot L2 address); the run's value is their sum mod 2^64.
// Payload: d[0] = id low word, d[1] = id high word, d[2] = depth.
#include "table_common.cuh"

namespace gtap {

constexpr uint32_t kTreeMaxB = 8;

struct TreeArgs {
    const unsigned long long* buf;
    unsigned long long* total;     // 32 counters
    unsigned long long lmask;      // len - 1 (len a power of two)
    unsigned long long seed;
    uint32_t mem_ops, compute_iters;
    uint32_t D, B;                 // B = 0: full binary tree
};

__device__ __forceinline__ unsigned long long tree_mix(unsigned long long z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27; z *= 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// bit k set: child k of node (id, depth) exists
__device__ __forceinline__ uint32_t tree_children(const TreeArgs& a, unsigned long long id, uint32_t depth) {
    if (depth >= a.D) return 0u;
    if (a.B == 0u) return 3u;
    const unsigned long long thr =
        (unsigned long long)(((unsigned __int128)(a.D - depth) << 53) / a.D);
    uint32_t gm = 0;
    for (uint32_t k = 0; k < a.B; ++k) {
        const unsigned long long c = (unsigned long long)a.B * id + 1ull + k;
        if ((tree_mix(a.seed ^ c) >> 11) < thr) gm |= 1u << k;
    }
    return gm;
}

__device__ __forceinline__ double chain_init(unsigned long long id, uint32_t c) {
    return 1.0 + (double)(uint32_t)((id + c) & 1023ull) * (1.0 / 1024.0);
}

__device__ __forceinline__ void tree_add(const TreeArgs& a, uint32_t slot, unsigned long long s) {
    if (s) dev::red_add_relaxed(&a.total[slot & 31u], s);
}

struct TreeThreadTable {
    static constexpr uint32_t kKind = GTAP_WORKER_THREAD;
    static constexpr int kMaxChildren = kTreeMaxB;
    static constexpr bool kTaskwait = true;
    static constexpr bool kHasHeavy = false;
    static constexpr bool kGenChildren = true;
    static constexpr uint32_t kNumFn = 1;
    static constexpr bool kJoinReduceAdd = false;
    static constexpr int kMaxThreads = 256, kMinBlocks = 2;
    using Args = TreeArgs;
    struct BlockExtra {
        uint32_t unused;
    };
    __device__ __forceinline__ static void block_init(BlockExtra*) {}

    // child c = the c-th existing child; g = {id lo, id hi, depth, B (0: binary)}
    __device__ __forceinline__ static void gen_child(const uint32_t (&g)[kDataWords], uint32_t gmask, uint32_t c,
                                                     uint32_t& fn, uint32_t& q, uint32_t (&d)[kDataWords]) {
        uint32_t m = gmask;
        for (uint32_t i = 0; i < c; ++i) m &= m - 1u;
        const uint32_t k = (uint32_t)__ffs(m) - 1u;
        const unsigned long long id = ((unsigned long long)g[1] << 32) | g[0];
        const unsigned long long ch = g[3] ? (unsigned long long)g[3] * id + 1ull + k : 2ull * id + k;
        fn = 0u;
        q = 0u;
        d[0] = (uint32_t)ch;
        d[1] = (uint32_t)(ch >> 32);
        d[2] = g[2] + 1u;
        d[3] = 0u;
    }

    // one lane runs the whole node: independent loads (unrolled), FMA chains four at a time
    __device__ __forceinline__ static unsigned long long work(const Args& a, unsigned long long id) {
        unsigned long long s = 0;
        const unsigned long long base = id * 0x9E3779B97F4A7C15ull;
        uint32_t i = 0;
        for (; i + 8u <= a.mem_ops; i += 8u) {  // 8 independent loads in flight per lane
            unsigned long long v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(&a.buf[tree_mix(base + i + u) & a.lmask]);
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        for (; i < a.mem_ops; ++i) s += __ldg(&a.buf[tree_mix(base + i) & a.lmask]);
        const uint32_t ci = a.compute_iters, nch = min(64u, ci), per = ci / 64u, rem = ci % 64u;
        for (uint32_t c = 0; c < nch; c += 4) {
            double f0 = chain_init(id, c), f1 = chain_init(id, c + 1), f2 = chain_init(id, c + 2),
                   f3 = chain_init(id, c + 3);
            for (uint32_t j = 0; j < per; ++j) {  // per > 0 only when all 64 chains run
                f0 = __fma_rn(f0, 0.999999, 1e-7); f1 = __fma_rn(f1, 0.999999, 1e-7);
                f2 = __fma_rn(f2, 0.999999, 1e-7); f3 = __fma_rn(f3, 0.999999, 1e-7);
            }
            if (c < rem) f0 = __fma_rn(f0, 0.999999, 1e-7);
            if (c + 1 < rem) f1 = __fma_rn(f1, 0.999999, 1e-7);
            if (c + 2 < rem) f2 = __fma_rn(f2, 0.999999, 1e-7);
            if (c + 3 < rem) f3 = __fma_rn(f3, 0.999999, 1e-7);
            s += (unsigned long long)__double_as_longlong(f0);
            if (c + 1 < nch) s += (unsigned long long)__double_as_longlong(f1);
            if (c + 2 < nch) s += (unsigned long long)__double_as_longlong(f2);
            if (c + 3 < nch) s += (unsigned long long)__double_as_longlong(f3);
        }
        return s;
    }

    __device__ __forceinline__ static void exec(const Args& a, uint32_t fn, uint32_t state,
                                                const uint32_t (&d)[kDataWords], TOut<1>& o, BlockExtra*) {
        if (fn != 0u || state > 1u) { o.bad_state(); return; }
        const unsigned long long id = ((unsigned long long)d[1] << 32) | d[0];
        if (state == 0u) {
            const uint32_t gm = tree_children(a, id, d[2]);
            if (gm) {                                   // spawn the children, taskwait
                o.gen[0] = d[0]; o.gen[1] = d[1]; o.gen[2] = d[2]; o.gen[3] = a.B;
                o.gmask = gm;
                o.nchild = (uint32_t)__popc(gm);
                o.suspend(1u);
                return;
            }
        }
        tree_add(a, threadIdx.x, work(a, id));          // after the join: do_memory_and_compute
        o.finish_void();
    }
};

struct TreeBlockTable {
    static constexpr uint32_t kKind = GTAP_WORKER_BLOCK;
    static constexpr int kMaxChildren = kTreeMaxB;
    static constexpr bool kTaskwait = true;
    static constexpr uint32_t kNumFn = 1;
    static constexpr bool kJoinReduceAdd = false;
    static constexpr int kMaxThreads = 1024, kMinBlocks = 1;
    static constexpr int kSpawnCap = kTreeMaxB;
    struct Scratch {
        uint32_t unused;
    };
    using Args = TreeArgs;

    template <class Ctx>
    __device__ __forceinline__ static void exec_block(const Args& a, Ctx& ctx, uint32_t fn, uint32_t state,
                                                      const uint32_t (&d)[kDataWords]) {
        const uint32_t tid = threadIdx.x, bd = blockDim.x;
        if (fn != 0u || state > 1u) {
            if (tid == 0) ctx.bad_state();
            return;
        }
        const unsigned long long id = ((unsigned long long)d[1] << 32) | d[0];
        if (state == 0u) {
            const uint32_t gm = tree_children(a, id, d[2]);   // uniform over the block
            if (gm) {
                if (tid < 32u && ((gm >> tid) & 1u)) {         // thread k spawns child k
                    const unsigned long long ch = a.B ? (unsigned long long)a.B * id + 1ull + tid : 2ull * id + tid;
                    ctx.spawn(0u, (uint32_t)ch, (uint32_t)(ch >> 32), d[2] + 1u);
                }
                if (tid == 0) ctx.suspend(1u);
                return;
            }
        }
        // do_memory_and_compute, data-parallel: loads strided over the block, one FMA chain per thread
        unsigned long long s = 0;
        const unsigned long long base = id * 0x9E3779B97F4A7C15ull;
        uint32_t i = tid;
        for (; i + 7u * bd < a.mem_ops; i += 8u * bd) {  // 8 independent loads in flight per thread
            unsigned long long v[8];
#pragma unroll
            for (uint32_t u = 0; u < 8u; ++u) v[u] = __ldg(&a.buf[tree_mix(base + i + u * bd) & a.lmask]);
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        for (; i < a.mem_ops; i += bd) s += __ldg(&a.buf[tree_mix(base + i) & a.lmask]);
        const uint32_t ci = a.compute_iters, nch = min(64u, ci), per = ci / 64u, rem = ci % 64u;
        for (uint32_t c = tid; c < nch; c += bd) {
            double f = chain_init(id, c);
            const uint32_t it = per + (c < rem ? 1u : 0u);
            for (uint32_t j = 0; j < it; ++j) f = __fma_rn(f, 0.999999, 1e-7);
            s += (unsigned long long)__double_as_longlong(f);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((tid & 31u) == 0) tree_add(a, blockIdx.x * (bd >> 5) + (tid >> 5), s);
        if (tid == 0) ctx.finish_void();
    }
};

static int validate_tree(const gtap_task_table* t, uint32_t fn, const uint32_t* d) {
    TreeArgs a;
    std::memcpy(&a, t->args, sizeof(a));
    const unsigned long long root = a.B ? 0ull : 1ull;
    return (fn == 0u && d[0] == (uint32_t)root && d[1] == 0u && d[2] == 0u && d[3] == 0u) ? 0 : -1;
}

}  // namespace gtap

// Synthetic tree: see include/gtap.h.
extern "C" const gtap_task_table* gtap_table_tree(int32_t worker_kind, int32_t D, int32_t B, uint64_t seed,
                                                  const unsigned long long* buf, uint64_t len, uint32_t mem_ops,
                                                  uint32_t compute_iters, unsigned long long* d_total) {
    if (!buf || !d_total || len == 0 || (len & (len - 1)) != 0 || D < 0 || D > 40) return nullptr;
    if (B != 0 && (B < 1 || B > (int32_t)gtap::kTreeMaxB || D < 1)) return nullptr;
    gtap::TreeArgs a{buf, d_total, len - 1, seed, mem_ops, compute_iters, (uint32_t)D, (uint32_t)B};
    if (worker_kind == GTAP_WORKER_THREAD)
        return gtap::make_table<gtap::TreeThreadTable>("tree_thread", a, &gtap::validate_tree);
    if (worker_kind == GTAP_WORKER_BLOCK)
        return gtap::make_table<gtap::TreeBlockTable>("tree_block", a, &gtap::validate_tree);
    return nullptr;
}
