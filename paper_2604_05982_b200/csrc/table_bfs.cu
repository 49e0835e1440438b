// table_bfs.cu -- BFS frontier-expansion task table (block-level, no taskwait).
//
// PAPER.md P:1053-1068 (Prog. parallel graph traversal):
//   bfs(v): dv = g_depth[v];
//           for (e = row_start + threadIdx.x; e < row_end; e += blockDim.x) {
//             u = g_col_indices[e]; old = atomicMin(&g_depth[u], dv + 1);
//             if (old > dv + 1) spawn bfs(u);
//           }
// dv is read with an L1-bypassing load (depth is shared mutable
// state written by other SMs). The edge loop runs in chunks of blockDim with
// a uniform flush point every kChunk chunks, so a hub vertex cannot overflow
// the shared-memory spawn staging (kSpawnCap). Payload: d[0] = v.
#include "table_common.cuh"

namespace gtap {

// ORDER 0: the paper's owner order (LIFO pops of the own deque; the block keeps its newest child);
// ORDER 1: oldest-first batch pops and every child pushed (the deques behave FIFO, closer to level order:
// RMAT-22 x 16 sources 9.4 -> 8.4 ms, expansions per reached vertex 2.0 -> 1.7), at the price of deques that
// hold a frontier (size max_tasks_per_worker / queue_capacity for it)
struct BfsArgs {
    const int32_t* row_ptr;
    const int32_t* col;
    int32_t* depth;
    uint32_t nv;
    uint32_t split;   // bfs(v) with more than `split` edges spawns bfs_edges pieces of `split` edges (0: never)
};
// CAP: shared-memory spawn staging (ChildSpecs) and free-stack depth. Blocks of <= 64 threads run the
// CAP = 128 instantiation (3.3 KB of shared memory: 32 one-warp blocks fit on an SM), larger blocks CAP = 512
// (a step stages up to 2 x blockDim spawns); gtap_run picks the kernel by block size (launch_bfs below)
template <uint32_t ORDER, int CAP, int MT = 1>
struct BfsTable {
    static constexpr uint32_t kKind = GTAP_WORKER_BLOCK;
    static constexpr int kMaxChildren = 0;  // dynamic (no taskwait: no join metadata)
    static constexpr bool kTaskwait = false;
    static constexpr uint32_t kNumFn = 2;
    static constexpr bool kJoinReduceAdd = false;  // see TaskRec
    static constexpr int kMaxThreads = 1024, kMinBlocks = 1;  // __launch_bounds__
    static constexpr int kSpawnCap = CAP;
    static constexpr uint32_t kBlockFreeStack = CAP < 256 ? (uint32_t)CAP : 256u;
#ifndef GTAP_BFS_U
#define GTAP_BFS_U 4
#endif
    static constexpr uint32_t kU = GTAP_BFS_U;       // edges per thread per step
#ifndef GTAP_BFS_MT_EDGES
#define GTAP_BFS_MT_EDGES 64
#endif
    static constexpr uint32_t kMtEdges = GTAP_BFS_MT_EDGES;   // edges per task scanned by its lane group
#ifdef GTAP_BFS_POP_BATCH
    static constexpr int kPopBatch = GTAP_BFS_POP_BATCH;  // sched_block.cuh batch pop
#else
    // one-warp blocks: 8 (RMAT-22 x 16 sources 4.66 -> 4.46 ms; 6: 4.52); 64-thread blocks: 4 (9.0 ms, 8: 10.8)
    static constexpr int kPopBatch = CAP < 256 ? 8 : 4;
#endif
    // MT > 1 (one-warp blocks): a cycle expands up to MT tasks of a popped batch side by side, 32 / MT lanes each
    static constexpr int kMultiTask = kPopBatch >= MT ? MT : 1;   // the batch supplies the extra tasks
    static constexpr bool kPopOldest = ORDER == 1u;
    static constexpr bool kKeepChild = ORDER == 0u;
#ifndef GTAP_BFS_TTAS
#define GTAP_BFS_TTAS 1   // read depth[u] before the atomicMin, skip it when no improvement is possible (8.4 -> 7.8 ms; 0: always the atomic)
#endif
#ifndef GTAP_BFS_SKIP_STALE
#define GTAP_BFS_SKIP_STALE 0   // 1: a task whose vertex improved since its spawn returns at once (measured slower)
#endif
    struct Scratch {
        uint32_t unused;
    };
    using Args = BfsArgs;
    // expand edges [s, e) of a vertex whose depth is dv; uniform over the block
    template <class Ctx>
    __device__ __forceinline__ static void expand(const Args& a, Ctx& ctx, int32_t s, int32_t e, int32_t dv) {
        const int32_t nd = dv + 1;
        const uint32_t bd = blockDim.x;
        // kU edges per thread per step: the kU col loads and then the kU atomicMin are independent,
        // so a hub's expansion keeps kU round trips in flight per thread (data-parallel body)
        // ue <= kU edges per thread per step, so that one step stages at most half the spawn buffer
        const uint32_t ue = max(1u, min(kU, (uint32_t)kSpawnCap / (2u * bd)));
        const uint32_t step = ue * bd;
        const uint32_t chunk_every = max(1u, (uint32_t)kSpawnCap / (2u * step));  // spawns between checks
        uint32_t k = 0;
        for (int32_t base = s; base < e; base += (int32_t)step) {
            int32_t u[kU];
#pragma unroll
            for (int j = 0; j < kU; ++j) {
                const int32_t i = base + (int32_t)(threadIdx.x + j * bd);
                u[j] = ((uint32_t)j < ue && i < e) ? __ldg(&a.col[i]) : -1;
            }
            int32_t old[kU];
#if GTAP_BFS_TTAS
            // test before the atomic: a neighbour already at depth <= nd cannot improve (depth only decreases)
            int32_t cur[kU];
#pragma unroll
            for (int j = 0; j < kU; ++j) cur[j] = u[j] >= 0 ? dev::ld_relaxed(&a.depth[u[j]]) : nd;
#pragma unroll
            for (int j = 0; j < kU; ++j) old[j] = cur[j] > nd ? atomicMin(&a.depth[u[j]], nd) : nd;
#else
#pragma unroll
            for (int j = 0; j < kU; ++j) old[j] = u[j] >= 0 ? atomicMin(&a.depth[u[j]], nd) : nd;
#endif
#pragma unroll
            for (int j = 0; j < kU; ++j)
                if (old[j] > nd) ctx.spawn(0u, (uint32_t)u[j], (uint32_t)nd);   // P:1063-1065 (d[1]: spawn depth)
            if (++k == chunk_every) {                               // uniform
                k = 0;
                if (base + (int32_t)step < e) ctx.flush(chunk_every * step);
            }
        }
    }
    // fn 0 = bfs(v). fn 1 = bfs_edges(v, lo, hi): edges [lo, hi) of v, spawned by bfs(v) when v
    // has more than a.split edges (B200 choice, R29: a hub's expansion is cut into pieces other
    // blocks steal, instead of one block scanning ~1e5 edges on the critical path; same depth writes)
    template <class Ctx>
    __device__ __forceinline__ static void exec_block(const Args& a, Ctx& ctx, uint32_t fn, uint32_t state,
                                                      const uint32_t (&d)[kDataWords]) {
        if (fn > 1u || state != 0u) {
            if (threadIdx.x == 0) ctx.bad_state();
            return;
        }
        const uint32_t v = d[0];
        const int32_t dv = dev::ld_relaxed(&a.depth[v]);
        if (fn == 1u) {   // a piece of a hub's edge list; dv re-read: it can only have improved since the split
            expand(a, ctx, (int32_t)d[1], (int32_t)d[2], dv);
            if (threadIdx.x == 0) ctx.finish_void();
            return;
        }
#if GTAP_BFS_SKIP_STALE
        // d[1] = the depth v had when this task was spawned; a smaller depth now means a later improvement
        // spawned a newer task for v, which will expand it with that depth: this one has nothing to add
        if (dv < (int32_t)d[1]) {
            if (threadIdx.x == 0) ctx.finish_void();
            return;
        }
#endif
        const int32_t s = __ldg(&a.row_ptr[v]), e = __ldg(&a.row_ptr[v + 1]);
        int32_t e0 = e;
        if (a.split != 0u && (uint32_t)(e - s) > a.split) {
            // pieces 1.. of [s, e) become bfs_edges tasks; this task scans piece 0
            const uint32_t sp = a.split;
            const uint32_t np = (uint32_t)(e - s + (int32_t)sp - 1) / sp;
            const uint32_t bd = blockDim.x;
            const uint32_t per = min(bd, (uint32_t)kSpawnCap / 2u);
            for (uint32_t b = 1; b < np; b += per) {                // uniform
                const uint32_t i = b + threadIdx.x;
                if (threadIdx.x < per && i < np) {
                    const int32_t lo = s + (int32_t)(i * sp);
                    ctx.spawn(1u, v, (uint32_t)lo, (uint32_t)min(e, lo + (int32_t)sp));
                }
                ctx.flush(per);
            }
            ctx.flush((uint32_t)kSpawnCap / 2u);   // the edge loop below stages up to half the buffer before its first check
            e0 = s + (int32_t)sp;
        }
        expand(a, ctx, s, e0, dv);
        if (threadIdx.x == 0) ctx.finish_void();
    }
    // MT tasks of a popped batch in one cycle of a one-warp block (B200 choice, DESIGN.md §5 "Multi-task cycles"):
    // group g = lanes [g G, g G + G), G = 32 / MT, expands task g's first kMtEdges edges (its hub pieces spawned
    // first); what is left of larger tasks is then expanded by the whole warp, task by task. Same depth writes as
    // MT single-task cycles, with one dependent chain of round trips for all of them.
    template <class Ctx>
    __device__ __forceinline__ static void exec_multi(const Args& a, Ctx& ctx, uint32_t cnt, const uint32_t (&fs)[MT],
                                                      const uint32_t (&dd)[MT][kDataWords]) {
        static_assert(MT > 1 && 32 % MT == 0, "lane groups of one warp");
        constexpr uint32_t G = 32u / (uint32_t)MT;
        constexpr uint32_t kUa = 2;                         // edges per lane per group step
        static_assert(32u * kUa <= (uint32_t)CAP / 2u, "a group step stages at most half the buffer");
        const uint32_t lane = threadIdx.x & 31u;
        bool bad = false;
#pragma unroll
        for (int k = 0; k < MT; ++k)
            if ((uint32_t)k < cnt && ((fs[k] & 0xFFu) > 1u || (fs[k] >> 8) != 0u)) bad = true;
        if (bad) {
            if (lane == 0) ctx.bad_state();
            return;
        }
        const uint32_t g = lane / G, gl = lane % G;
        const bool act = g < cnt;
        const uint32_t fn = act ? (fs[g] & 0xFFu) : 0u;
        const uint32_t v = act ? dd[g][0] : 0u;
        int32_t dv = 0, s = 0, e = 0;
        if (act) {
            dv = dev::ld_relaxed(&a.depth[v]);
            if (fn == 1u) { s = (int32_t)dd[g][1]; e = (int32_t)dd[g][2]; }
            else { s = __ldg(&a.row_ptr[v]); e = __ldg(&a.row_ptr[v + 1]); }
        }
        // hub pieces (R29), G per group per round
        if (a.split != 0u) {
            const uint32_t sp = a.split;
            const uint32_t np = (act && fn == 0u && (uint32_t)(e - s) > sp) ? (uint32_t)(e - s + (int32_t)sp - 1) / sp : 1u;
            const uint32_t mx = __reduce_max_sync(0xffffffffu, np);
            if (mx > 1u) {
                for (uint32_t b = 1; b < mx; b += G) {
                    const uint32_t i = b + gl;
                    if (i < np) {
                        const int32_t lo = s + (int32_t)(i * sp);
                        ctx.spawn(1u, v, (uint32_t)lo, (uint32_t)min(e, lo + (int32_t)sp));
                    }
                    ctx.flush(32u);
                }
                ctx.flush((uint32_t)CAP / 2u);
                if (np > 1u) e = s + (int32_t)sp;
            }
        }
        const int32_t nd = dv + 1;
        // phase A: every group its task's first kMtEdges edges
        const int32_t ea = min(e, s + (int32_t)kMtEdges);
        const uint32_t steps = (uint32_t)__reduce_max_sync(0xffffffffu, (uint32_t)max(0, ea - s)) ;
        for (uint32_t base = 0; base < steps; base += G * kUa) {
            int32_t u[kUa];
#pragma unroll
            for (uint32_t j = 0; j < kUa; ++j) {
                const int32_t i = s + (int32_t)(base + gl + j * G);
                u[j] = (act && i < ea) ? __ldg(&a.col[i]) : -1;
            }
            int32_t cur[kUa];
#pragma unroll
            for (uint32_t j = 0; j < kUa; ++j) cur[j] = u[j] >= 0 ? dev::ld_relaxed(&a.depth[u[j]]) : nd;
#pragma unroll
            for (uint32_t j = 0; j < kUa; ++j) {
                const int32_t old = cur[j] > nd ? atomicMin(&a.depth[u[j]], nd) : nd;
                if (old > nd) ctx.spawn(0u, (uint32_t)u[j], (uint32_t)nd);
            }
            ctx.flush(32u * kUa);
        }
        // phase B: the rest of larger tasks, whole warp, one task at a time
        const uint32_t rest = __ballot_sync(0xffffffffu, act && gl == 0u && ea < e);
        for (uint32_t k = 0; k < (uint32_t)MT; ++k) {
            if (!((rest >> (k * G)) & 1u)) continue;            // uniform
            const int32_t sk = __shfl_sync(0xffffffffu, ea, k * G), ek = __shfl_sync(0xffffffffu, e, k * G);
            const int32_t dk = __shfl_sync(0xffffffffu, dv, k * G);
            expand(a, ctx, sk, ek, dk);
            ctx.flush((uint32_t)CAP / 2u);
        }
        if (lane == 0) ctx.finish_void();
    }
};

static int validate_bfs(const gtap_task_table* t, uint32_t fn, const uint32_t* d) {
    BfsArgs a;
    std::memcpy(&a, t->args, sizeof(a));
    return (fn == 0u && d[0] < a.nv) ? 0 : -1;
}

static constexpr uint32_t kBfsSmallBlock = 64;   // blocks up to this size run the small-staging kernel

#ifndef GTAP_BFS_MT
#define GTAP_BFS_MT 4   // tasks per cycle of a one-warp block (1: one task per cycle)
#endif
template <uint32_t ORDER>
cudaError_t launch_bfs(const gtap_task_table* t, const KParams& p, uint32_t grid, uint32_t block, cudaStream_t s) {
    if (block == 32u) return launch_block<BfsTable<ORDER, 128, GTAP_BFS_MT>>(t, p, grid, block, s);
    return block <= kBfsSmallBlock ? launch_block<BfsTable<ORDER, 128>>(t, p, grid, block, s)
                                   : launch_block<BfsTable<ORDER, 512>>(t, p, grid, block, s);
}
template <uint32_t ORDER>
cudaError_t occupancy_bfs(const gtap_task_table* t, uint32_t block, int* bps, size_t* smem) {
    if (block == 32u) return occupancy_block<BfsTable<ORDER, 128, GTAP_BFS_MT>>(t, block, bps, smem);
    return block <= kBfsSmallBlock ? occupancy_block<BfsTable<ORDER, 128>>(t, block, bps, smem)
                                   : occupancy_block<BfsTable<ORDER, 512>>(t, block, bps, smem);
}
template <uint32_t ORDER>
gtap_task_table* make_bfs(const char* name, const BfsArgs& a) {
    gtap_task_table* t = make_table<BfsTable<ORDER, 512>>(name, a, &validate_bfs);
    if (t) { t->launch = &launch_bfs<ORDER>; t->occupancy = &occupancy_bfs<ORDER>; }
    return t;
}

}  // namespace gtap

extern "C" const gtap_task_table* gtap_table_bfs_split(const int32_t* row_ptr, const int32_t* col, int32_t* depth,
                                                       uint32_t nv, uint32_t order, uint32_t edge_split) {
    if (!row_ptr || !col || !depth || nv == 0 || order > 1u) return nullptr;
    gtap::BfsArgs a{row_ptr, col, depth, nv, edge_split};
    return order == 0u ? gtap::make_bfs<0>("bfs", a) : gtap::make_bfs<1>("bfs_fifo", a);
}

extern "C" const gtap_task_table* gtap_table_bfs_ex(const int32_t* row_ptr, const int32_t* col, int32_t* depth,
                                                    uint32_t nv, uint32_t order) {
    return gtap_table_bfs_split(row_ptr, col, depth, nv, order, 0u);
}

extern "C" const gtap_task_table* gtap_table_bfs(const int32_t* row_ptr, const int32_t* col, int32_t* depth,
                                                 uint32_t nv) {
    return gtap_table_bfs_ex(row_ptr, col, depth, nv, 0u);
}

namespace {
__global__ void bfs_init_depth_kernel(int32_t* __restrict__ depth, uint32_t nv, int32_t src) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = i; v < nv; v += stride) depth[v] = (v == (uint32_t)src) ? 0 : 0x7fffffff;
}
}  // namespace

// depth[v] = INT32_MAX for v != src, depth[src] = 0 (reading R18), on `stream`.
extern "C" gtap_status gtap_bfs_init_depth(int32_t* depth, uint32_t nv, int32_t src, void* stream) {
    if (!depth || nv == 0 || src < 0 || (uint32_t)src >= nv) return GTAP_E_INVAL;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t blocks = min((nv + 255u) / 256u, (uint32_t)sms * 8u);
    bfs_init_depth_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(depth, nv, src);
    return cudaGetLastError() == cudaSuccess ? GTAP_OK : GTAP_E_CUDA;
}

#ifdef GTAP_TRACE
GTAP_TRACE_READER(bfs)
#endif
