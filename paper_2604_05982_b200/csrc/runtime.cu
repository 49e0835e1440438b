// runtime.cu -- host side of the C ABI (include/gtap.h).
//
// gtap_init bulk-allocates every task-management region on the host before any
// spawn; gtap_run launches ONE persistent kernel
// per run with the staged roots; gtap_sync waits, reads the
// sticky device error word and the device-side counters. Nothing here touches
// task data: every step of the hot path runs in the kernels of sched_*.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "gtap.h"
#include "table_common.cuh"

using gtap::Ctl;
using gtap::KParams;
using gtap::Layout;
using gtap::RootSpec;

struct gtap_runtime {
    gtap_config cfg;
    int device;
    int sm_count;
    uint32_t wpb;          // workers per block (thread-level: warps per block; block-level: 1)
    uint32_t W_alloc;      // workers the workspace is sized for
    uint32_t M, Q, max_roots;
    Layout L;
    char* ws;
    bool owns_ws;
    std::vector<RootSpec> roots;
    const gtap_task_table* table;
    RootSpec* h_roots;     // pinned, mapped: root staging (max_roots)
    Ctl* h_ctl;            // pinned, mapped: control block staging / readback
    RootSpec* dh_roots;    // device aliases of the two mapped buffers
    Ctl* dh_ctl;
    cudaEvent_t ev0, ev1, ev2;   // kernel start / end, control-block readback done
    cudaEvent_t ev_reset;        // recorded after gtap_reset's fill kernels: gtap_run's stream waits on it
    bool reset_pending;          // ev_reset recorded and not yet waited for by a run
    bool in_flight;
    bool dirty;            // workspace used since the last reset
    uint32_t run_grid, run_block, run_W;
    uint32_t run_nroots;
    gtap_status last_launch;
    gtap::CheckBuf* chk;   // GTAP_CHECK builds: device check buffer (header + 3 token arrays)
    // victim_policy 1: device copy of {sm_die[256] | vlist[W_alloc]} and the host lists (ascending worker ids)
    unsigned char* vbuf;
    std::vector<uint32_t> vl[2];
};

namespace {

bool is_pow2(uint32_t x) { return x && !(x & (x - 1)); }
uint32_t log2u(uint32_t x) { uint32_t l = 0; while ((1u << l) < x) ++l; return l; }

gtap_status cuda_status(cudaError_t e) { return e == cudaSuccess ? GTAP_OK : GTAP_E_CUDA; }

// resolve defaults; returns GTAP_E_INVAL for bad fields
gtap_status resolve(const gtap_config* in, gtap_config* c, int sm_count) {
    if (!in || in->struct_size != sizeof(gtap_config)) return GTAP_E_INVAL;
    *c = *in;
    if (c->worker_kind > GTAP_WORKER_BLOCK) return GTAP_E_INVAL;
    if (c->block_size == 0) c->block_size = 128;
    if (c->block_size % 32 || c->block_size < 32 || c->block_size > 1024) return GTAP_E_INVAL;
    if (c->max_tasks_per_worker == 0) c->max_tasks_per_worker = 4096;
    if (!is_pow2(c->max_tasks_per_worker) || c->max_tasks_per_worker < 64 || c->max_tasks_per_worker > (1u << 20))
        return GTAP_E_INVAL;
    if (c->queue_capacity == 0) c->queue_capacity = c->max_tasks_per_worker;
    if (!is_pow2(c->queue_capacity) || c->queue_capacity < 64 || c->queue_capacity > (1u << 24)) return GTAP_E_INVAL;
    if (c->num_queues == 0) c->num_queues = 1;
    if (c->num_queues > 8) return GTAP_E_INVAL;
    if (c->worker_kind == GTAP_WORKER_BLOCK && c->num_queues != 1) return GTAP_E_INVAL;  // EPAQ: thread-level
    if (c->max_task_data_size == 0) c->max_task_data_size = 16;
    if (c->max_task_data_size > 16) return GTAP_E_UNSUPPORTED;
    if (c->steal_attempts == 0) c->steal_attempts = 4;
    if (c->steal_max == 0) c->steal_max = (c->worker_kind == GTAP_WORKER_THREAD) ? 32 : 1;
    if (c->worker_kind == GTAP_WORKER_THREAD && c->steal_max > 32) return GTAP_E_INVAL;
    if (c->worker_kind == GTAP_WORKER_BLOCK && c->steal_max > 32) return GTAP_E_INVAL;  // default 1
    if (c->max_roots == 0) c->max_roots = 65536;
    if (c->idle_backoff_ns == 0) c->idle_backoff_ns = 8192;
    if (c->idle_backoff_ns < 32 || c->idle_backoff_ns > 1000000) return GTAP_E_INVAL;
    if (c->queue_policy > 1) return GTAP_E_INVAL;
    if (c->victim_policy > 1) return GTAP_E_INVAL;
    const uint32_t wpb = (c->worker_kind == GTAP_WORKER_THREAD) ? c->block_size / 32 : 1;
    uint64_t W;
    if (c->grid_size) W = (uint64_t)c->grid_size * wpb;
    else W = (c->worker_kind == GTAP_WORKER_THREAD) ? (uint64_t)sm_count * 64 : (uint64_t)sm_count * 32;
    if (W == 0 || W * c->max_tasks_per_worker >= (1ull << 31)) return GTAP_E_INVAL;  // ids are u32, kNone reserved
    return GTAP_OK;
}

uint32_t workers_alloc(const gtap_config& c, int sm_count) {
    const uint32_t wpb = (c.worker_kind == GTAP_WORKER_THREAD) ? c.block_size / 32 : 1;
    if (c.grid_size) return c.grid_size * wpb;
    return (c.worker_kind == GTAP_WORKER_THREAD) ? (uint32_t)sm_count * 64 : (uint32_t)sm_count * 32;
}

int device_sm_count(int dev) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return n;
}

gtap_status geometry(gtap_runtime* rt, const gtap_task_table* t, uint32_t* W, uint32_t* grid, uint32_t* block) {
    if (t->kind != rt->cfg.worker_kind) return GTAP_E_INVAL;
    const uint32_t bs = rt->cfg.block_size;
    if (bs > t->max_block) return GTAP_E_INVAL;  // beyond the table kernel's __launch_bounds__
    if (t->num_queues > rt->cfg.num_queues) return GTAP_E_INVAL;  // EPAQ table needs its queues
    int bps = 0;
    size_t smem = 0;
    if (t->occupancy(t, bs, &bps, &smem) != cudaSuccess) return GTAP_E_CUDA;
    if (bps <= 0) return GTAP_E_INVAL;
    const uint32_t max_grid = (uint32_t)bps * (uint32_t)rt->sm_count;
    uint32_t g = rt->cfg.grid_size ? rt->cfg.grid_size : std::min(max_grid, rt->W_alloc / rt->wpb);
    if (g == 0 || g > max_grid) return GTAP_E_INVAL;  // persistent grid must be co-resident
    if (g * rt->wpb > rt->W_alloc) return GTAP_E_INVAL;
    *W = g * rt->wpb;
    *grid = g;
    *block = bs;
    return GTAP_OK;
}

// Small transfers and fills by SM kernels instead of cudaMemcpyAsync / cudaMemsetAsync: a run's
// root / control-block staging and readback then never queue behind a user's bulk copy on the
// same copy engine (the bench's pipelined e2e overlaps 64 MB H2D and D2H copies with the sort; the
// 200-byte control-block readback waited ~1 ms behind them before each gtap_sync returned).
__global__ void word_copy_kernel(const uint32_t* __restrict__ s0, uint32_t* __restrict__ d0, uint32_t n0,
                                 const uint32_t* __restrict__ s1, uint32_t* __restrict__ d1, uint32_t n1) {
    for (uint32_t i = threadIdx.x; i < n0; i += blockDim.x) d0[i] = s0[i];
    for (uint32_t i = threadIdx.x; i < n1; i += blockDim.x) d1[i] = s1[i];
}
__global__ void zero_kernel(uint32_t* __restrict__ p, size_t words) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint4* p4 = reinterpret_cast<uint4*>(p);
    const size_t n4 = words / 4u;
    for (size_t k = i; k < n4; k += stride) p4[k] = make_uint4(0u, 0u, 0u, 0u);
    for (size_t k = n4 * 4u + i; k < words; k += stride) p[k] = 0u;
}

}  // namespace

namespace gtap {
cudaError_t zero_async(void* p, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return cudaSuccess;
    if ((bytes & 3u) || ((uintptr_t)p & 15u)) return cudaMemsetAsync(p, 0, bytes, s);
    const size_t words = bytes / 4u;
    const unsigned blocks = (unsigned)std::min<size_t>((words / 4u + 255u) / 256u + 1u, 148u * 8u);
    zero_kernel<<<blocks, 256, 0, s>>>(static_cast<uint32_t*>(p), words);
    return cudaGetLastError();
}
}  // namespace gtap

namespace {

#ifdef GTAP_CHECK
// header (counters + pointers, padded to 256 B) + live / runnable / kids arrays of W * M words
size_t check_words(const gtap_runtime* rt) { return (size_t)rt->L.W * rt->L.M; }
size_t check_bytes(const gtap_runtime* rt) { return 256 + 3 * 4 * check_words(rt); }
#endif

gtap_status do_reset(gtap_runtime* rt, cudaStream_t s) {
    cudaSetDevice(rt->device);
    const Layout& L = rt->L;
    // control block, deque metadata, free-ring metadata (contiguous at the front)
    if (gtap::zero_async(rt->ws + L.ctl, L.roots - L.ctl, s) != cudaSuccess) return GTAP_E_CUDA;
    // free rings: entry 0 = empty
    if (gtap::zero_async(rt->ws + L.fring, sizeof(uint32_t) * (size_t)L.W * L.M, s) != cudaSuccess)
        return GTAP_E_CUDA;
#ifdef GTAP_CHECK
    if (rt->chk && gtap::zero_async(rt->chk, check_bytes(rt), s) != cudaSuccess) return GTAP_E_CUDA;
#endif
    // a run on another stream must not start before these fills (gtap_run waits on the event)
    if (cudaEventRecord(rt->ev_reset, s) != cudaSuccess) return GTAP_E_CUDA;
    rt->reset_pending = true;
    rt->dirty = false;
    return GTAP_OK;
}

}  // namespace

extern "C" {

uint32_t gtap_abi_version(void) { return GTAP_ABI_VERSION; }

const char* gtap_status_str(gtap_status s) {
    switch (s) {
        case GTAP_OK: return "GTAP_OK";
        case GTAP_E_INVAL: return "GTAP_E_INVAL";
        case GTAP_E_CUDA: return "GTAP_E_CUDA";
        case GTAP_E_NOMEM: return "GTAP_E_NOMEM";
        case GTAP_E_BUSY: return "GTAP_E_BUSY";
        case GTAP_E_POOL_EXHAUSTED: return "GTAP_E_POOL_EXHAUSTED";
        case GTAP_E_QUEUE_OVERFLOW: return "GTAP_E_QUEUE_OVERFLOW";
        case GTAP_E_CHILD_LIMIT: return "GTAP_E_CHILD_LIMIT";
        case GTAP_E_TIMEOUT: return "GTAP_E_TIMEOUT";
        case GTAP_E_BAD_STATE: return "GTAP_E_BAD_STATE";
        case GTAP_E_NO_DEVICE: return "GTAP_E_NO_DEVICE";
        case GTAP_E_UNSUPPORTED: return "GTAP_E_UNSUPPORTED";
        case GTAP_E_INVARIANT: return "GTAP_E_INVARIANT";
    }
    return "GTAP_E_UNKNOWN";
}

gtap_status gtap_config_default(gtap_config* cfg, int32_t device, uint32_t kind) {
    if (!cfg || kind > GTAP_WORKER_BLOCK) return GTAP_E_INVAL;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->struct_size = sizeof(gtap_config);
    cfg->device = device;
    cfg->worker_kind = kind;
    cfg->block_size = (kind == GTAP_WORKER_THREAD) ? 128 : 256;
    cfg->max_tasks_per_worker = (kind == GTAP_WORKER_THREAD) ? 4096 : 4096;
    cfg->num_queues = 1;
    cfg->steal_attempts = 4;
    cfg->seed = 0x5EEDull;
    return GTAP_OK;
}

size_t gtap_workspace_bytes(const gtap_config* in) {
    gtap_config c;
    const int sm = in ? device_sm_count(in->device) : 0;
    if (resolve(in, &c, sm > 0 ? sm : 148) != GTAP_OK) return 0;
    const uint32_t W = workers_alloc(c, sm > 0 ? sm : 148);
    return gtap::make_layout(W, c.max_tasks_per_worker, c.queue_capacity, c.max_roots, c.num_queues).total;
}

gtap_status gtap_init(const gtap_config* in, void* d_workspace, size_t bytes, gtap_runtime** out) {
    if (!out) return GTAP_E_INVAL;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return GTAP_E_NO_DEVICE;
    if (!in || in->device < 0 || in->device >= ndev) return GTAP_E_INVAL;
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, in->device);
    if (major != 10) return GTAP_E_NO_DEVICE;  // built for sm_100a only
    const int sm = device_sm_count(in->device);
    gtap_config c;
    gtap_status st = resolve(in, &c, sm);
    if (st != GTAP_OK) return st;
    if (cudaSetDevice(c.device) != cudaSuccess) return GTAP_E_CUDA;

    gtap_runtime* rt = new (std::nothrow) gtap_runtime();
    if (!rt) return GTAP_E_NOMEM;
    rt->cfg = c;
    rt->device = c.device;
    rt->sm_count = sm;
    rt->wpb = (c.worker_kind == GTAP_WORKER_THREAD) ? c.block_size / 32 : 1;
    rt->W_alloc = workers_alloc(c, sm);
    rt->M = c.max_tasks_per_worker;
    rt->Q = c.queue_capacity;
    rt->max_roots = c.max_roots;
    rt->L = gtap::make_layout(rt->W_alloc, rt->M, rt->Q, rt->max_roots, c.num_queues);
    if (d_workspace) {
        if (bytes < rt->L.total || ((uintptr_t)d_workspace & 255u)) { delete rt; return GTAP_E_INVAL; }
        rt->ws = static_cast<char*>(d_workspace);
        rt->owns_ws = false;
    } else {
        if (cudaMalloc(&rt->ws, rt->L.total) != cudaSuccess) { delete rt; return GTAP_E_NOMEM; }
        rt->owns_ws = true;
    }
    if (cudaHostAlloc(&rt->h_roots, sizeof(RootSpec) * rt->max_roots, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostAlloc(&rt->h_ctl, sizeof(Ctl), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&rt->dh_roots), rt->h_roots, 0) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&rt->dh_ctl), rt->h_ctl, 0) != cudaSuccess) {
        gtap_finalize(rt);
        return GTAP_E_NOMEM;
    }
    if (cudaEventCreate(&rt->ev0) != cudaSuccess || cudaEventCreate(&rt->ev1) != cudaSuccess ||
        cudaEventCreate(&rt->ev2) != cudaSuccess ||
        cudaEventCreateWithFlags(&rt->ev_reset, cudaEventDisableTiming) != cudaSuccess) {
        gtap_finalize(rt);
        return GTAP_E_CUDA;
    }
#ifdef GTAP_CHECK
    if (cudaMalloc(&rt->chk, check_bytes(rt)) != cudaSuccess) { gtap_finalize(rt); return GTAP_E_NOMEM; }
#endif
    if (c.victim_policy == 1u) {
        // which die homes each worker's deque line (2 KB L2-home granules of the DequeMeta array), and the
        // SM -> die map: one probe address per granule
        const uintptr_t dq = (uintptr_t)(rt->ws + rt->L.dq);
        const size_t bytes = sizeof(gtap::DequeMeta) * (size_t)rt->W_alloc * c.num_queues;
        const uintptr_t g0 = dq / 2048u, g1 = (dq + bytes - 1u) / 2048u;
        const uint32_t ng = (uint32_t)(g1 - g0 + 1u);
        // one probe address per full granule (from the first 2 KB boundary inside the array); workers whose
        // line lies in the partial first granule are left out of both lists (uniform lanes still reach them)
        std::vector<uint8_t> gnear(ng, 2u), smd(256);
        const uintptr_t first_full = (dq % 2048u) ? (g0 + 1u) * 2048u : dq;
        const uint32_t nfull = first_full / 2048u <= g1 ? (uint32_t)(g1 - first_full / 2048u + 1u) : 0u;
        // (an array inside one partial granule -- a handful of workers -- leaves both lists empty: uniform victims)
        if (nfull > 0u && gtap::die_probe(reinterpret_cast<const void*>(first_full), 2048, nfull, smd.data(), 256,
                                          gnear.data() + (first_full / 2048u - g0), nullptr, 0) != 0) {
            gtap_finalize(rt);
            return GTAP_E_CUDA;
        }
        for (uint32_t w = 0; w < rt->W_alloc; ++w) {
            const uintptr_t a = dq + sizeof(gtap::DequeMeta) * (size_t)w * c.num_queues;
            const uint8_t d = gnear[a / 2048u - g0];
            if (d < 2u) rt->vl[d].push_back(w);
        }
        if (cudaMalloc(&rt->vbuf, 256 + sizeof(uint32_t) * (size_t)rt->W_alloc) != cudaSuccess) {
            gtap_finalize(rt);
            return GTAP_E_NOMEM;
        }
        std::vector<uint32_t> all(rt->vl[0]);
        all.insert(all.end(), rt->vl[1].begin(), rt->vl[1].end());
        if (cudaMemcpy(rt->vbuf, smd.data(), 256, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(rt->vbuf + 256, all.data(), sizeof(uint32_t) * all.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
            gtap_finalize(rt);
            return GTAP_E_CUDA;
        }
    }
    rt->dirty = true;
    if ((st = do_reset(rt, 0)) != GTAP_OK || cudaStreamSynchronize(0) != cudaSuccess) {
        gtap_finalize(rt);
        return st != GTAP_OK ? st : GTAP_E_CUDA;
    }
    *out = rt;
    return GTAP_OK;
}

gtap_status gtap_spawn_root(gtap_runtime* rt, const gtap_task_table* t, uint32_t fn, const void* args,
                            uint32_t nbytes, uint32_t* root_idx) {
    if (!rt || !t || nbytes > sizeof(uint32_t) * gtap::kDataWords || (nbytes && !args)) return GTAP_E_INVAL;
    if (rt->in_flight) return GTAP_E_BUSY;
    if (t->kind != rt->cfg.worker_kind) return GTAP_E_INVAL;
    if (rt->table && rt->table != t && !rt->roots.empty()) return GTAP_E_INVAL;  // one table per run
    if (rt->roots.size() >= rt->max_roots) return GTAP_E_INVAL;
    RootSpec r{};
    r.fn = fn;
    if (nbytes) std::memcpy(r.d, args, nbytes);  // firstprivate copy
    if (fn >= t->nfn || (t->validate_root && t->validate_root(t, fn, r.d) != 0)) return GTAP_E_INVAL;
    rt->table = t;
    if (root_idx) *root_idx = (uint32_t)rt->roots.size();
    rt->roots.push_back(r);
    return GTAP_OK;
}

gtap_status gtap_reset(gtap_runtime* rt, void* stream) {
    if (!rt) return GTAP_E_INVAL;
    if (rt->in_flight) return GTAP_E_BUSY;
    rt->roots.clear();
    rt->table = nullptr;
    return do_reset(rt, static_cast<cudaStream_t>(stream));
}

gtap_status gtap_geometry(gtap_runtime* rt, const gtap_task_table* t, uint32_t* workers, uint32_t* grid,
                          uint32_t* block) {
    if (!rt || !t) return GTAP_E_INVAL;
    cudaSetDevice(rt->device);
    uint32_t W = 0, g = 0, b = 0;
    gtap_status st = geometry(rt, t, &W, &g, &b);
    if (st != GTAP_OK) return st;
    if (workers) *workers = W;
    if (grid) *grid = g;
    if (block) *block = b;
    return GTAP_OK;
}

static gtap_status run_impl(gtap_runtime* rt, cudaStream_t s) {
    uint32_t W = 0, grid = 0, block = 0;
    gtap_status st = geometry(rt, rt->table, &W, &grid, &block);
    if (st != GTAP_OK) return st;
    if (rt->dirty && (st = do_reset(rt, s)) != GTAP_OK) return st;
    // gtap_reset may have been enqueued on another stream: order its fills before this run
    if (rt->reset_pending) {
        if (cudaStreamWaitEvent(s, rt->ev_reset, 0) != cudaSuccess) return GTAP_E_CUDA;
        rt->reset_pending = false;
    }
    const uint32_t nroots = (uint32_t)rt->roots.size();
    // roots + termination counters: one pinned H2D copy each
    std::memcpy(rt->h_roots, rt->roots.data(), sizeof(RootSpec) * nroots);
    std::memset(rt->h_ctl, 0, sizeof(Ctl));
    rt->h_ctl->roots_left = nroots;
    rt->h_ctl->outstanding = nroots;
    rt->h_ctl->vinfo = nullptr;
    if (rt->vbuf) {   // victim_policy 1: the lists restricted to this run's workers (ids < W, lists ascending)
        rt->h_ctl->vcnt[0] = (uint32_t)(std::lower_bound(rt->vl[0].begin(), rt->vl[0].end(), W) - rt->vl[0].begin());
        rt->h_ctl->vcnt[1] = (uint32_t)(std::lower_bound(rt->vl[1].begin(), rt->vl[1].end(), W) - rt->vl[1].begin());
        rt->h_ctl->vcnt[2] = (uint32_t)rt->vl[0].size();
        rt->h_ctl->vinfo = reinterpret_cast<const uint32_t*>(rt->vbuf);
    }
    // one SM kernel reads both from the mapped host buffers (no copy engine, see word_copy_kernel)
    static_assert(sizeof(RootSpec) % 4 == 0 && sizeof(Ctl) % 4 == 0, "word copies");
    word_copy_kernel<<<1, 256, 0, s>>>(reinterpret_cast<const uint32_t*>(rt->dh_roots),
                                       reinterpret_cast<uint32_t*>(rt->ws + rt->L.roots),
                                       (uint32_t)(sizeof(RootSpec) * nroots / 4), reinterpret_cast<const uint32_t*>(rt->dh_ctl),
                                       reinterpret_cast<uint32_t*>(rt->ws + rt->L.ctl), (uint32_t)(sizeof(Ctl) / 4));
    if (cudaGetLastError() != cudaSuccess) return GTAP_E_CUDA;

    KParams p{};
    p.W = W;
    p.logM = log2u(rt->M);
    p.qmask = rt->Q - 1u;
    p.steal_rounds = rt->cfg.steal_attempts;
    p.steal_max = rt->cfg.steal_max;
    p.nroots = nroots;
    // GTAP_MAX_CHILD_TASKS: the config's limit, never above the table's compile-time bound (0 = dynamic table:
    // only the config's limit, if any, applies)
    {
        const uint32_t tb = rt->table->max_children, cl = rt->cfg.max_child_tasks;
        p.max_child = tb == 0u ? cl : (cl ? std::min(cl, tb) : tb);
    }
    p.seed = rt->cfg.seed;
    p.watchdog_ns = rt->cfg.watchdog_ns;
    p.idle_backoff = rt->cfg.idle_backoff_ns;
    p.nq = rt->cfg.num_queues;
    p.policy = (rt->cfg.queue_policy == 1u ? gtap::kPolQueueStay : 0u) | (rt->vbuf ? gtap::kPolDieVictims : 0u);
    p.rec = reinterpret_cast<gtap::TaskRec*>(rt->ws + rt->L.rec);
    p.ring = reinterpret_cast<uint32_t*>(rt->ws + rt->L.ring);
    p.dq = reinterpret_cast<gtap::DequeMeta*>(rt->ws + rt->L.dq);
    p.fring = reinterpret_cast<uint32_t*>(rt->ws + rt->L.fring);
    p.fm = reinterpret_cast<gtap::FreeMeta*>(rt->ws + rt->L.fm);
    p.ctl = reinterpret_cast<Ctl*>(rt->ws + rt->L.ctl);
    p.roots = reinterpret_cast<const RootSpec*>(rt->ws + rt->L.roots);
    p.root_results = reinterpret_cast<long long*>(rt->ws + rt->L.results);
    p.chk = nullptr;
#ifdef GTAP_CHECK
    {   // the header's array pointers (device addresses inside the check buffer), written before the run
        gtap::CheckBuf hb{};
        char* base = reinterpret_cast<char*>(rt->chk);
        hb.live = reinterpret_cast<uint32_t*>(base + 256);
        hb.runnable = hb.live + check_words(rt);
        hb.kids = reinterpret_cast<int32_t*>(hb.runnable + check_words(rt));
        if (cudaMemcpyAsync(reinterpret_cast<char*>(rt->chk) + offsetof(gtap::CheckBuf, live), &hb.live,
                            3 * sizeof(void*), cudaMemcpyHostToDevice, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return GTAP_E_CUDA;
        p.chk = rt->chk;
    }
#endif

    if (rt->table->prepare && rt->table->prepare(rt->table, s) != cudaSuccess) return GTAP_E_CUDA;
    if (cudaEventRecord(rt->ev0, s) != cudaSuccess) return GTAP_E_CUDA;
    const cudaError_t le = rt->table->launch(rt->table, p, grid, block, s);
    if (le != cudaSuccess) return GTAP_E_CUDA;
    if (cudaEventRecord(rt->ev1, s) != cudaSuccess) return GTAP_E_CUDA;
    // the control block (error word, counters) comes back on the same stream right behind the kernel,
    // so gtap_sync waits for this run only (no legacy-stream synchronous copy)
    word_copy_kernel<<<1, 256, 0, s>>>(reinterpret_cast<const uint32_t*>(rt->ws + rt->L.ctl),
                                       reinterpret_cast<uint32_t*>(rt->dh_ctl), (uint32_t)(sizeof(Ctl) / 4), nullptr,
                                       nullptr, 0u);
    if (cudaGetLastError() != cudaSuccess || cudaEventRecord(rt->ev2, s) != cudaSuccess) return GTAP_E_CUDA;
    rt->in_flight = true;
    rt->dirty = true;
    rt->run_grid = grid;
    rt->run_block = block;
    rt->run_W = W;
    rt->run_nroots = nroots;
    rt->roots.clear();
    return GTAP_OK;
}

}  // extern "C"

namespace {
// any failure of gtap_run drops the staged roots and the table binding (the caller may destroy the
// table next; a later run must not pick up stale roots) and forces a full reset before the next run
gtap_status run_failed(gtap_runtime* rt, gtap_status st) {
    rt->roots.clear();
    rt->table = nullptr;
    rt->dirty = true;
    return st;
}
}  // namespace

extern "C" {

gtap_status gtap_run(gtap_runtime* rt, void* stream) {
    if (!rt) return GTAP_E_INVAL;
    if (rt->in_flight) return GTAP_E_BUSY;
    if (rt->roots.empty() || !rt->table) return run_failed(rt, GTAP_E_INVAL);
    cudaSetDevice(rt->device);
    const gtap_status st = run_impl(rt, static_cast<cudaStream_t>(stream));
    return st == GTAP_OK ? st : run_failed(rt, st);
}

gtap_status gtap_sync(gtap_runtime* rt, gtap_stats* out) {
    if (!rt) return GTAP_E_INVAL;
    if (!rt->in_flight) return GTAP_E_INVAL;
    cudaSetDevice(rt->device);
    rt->in_flight = false;
    if (cudaEventSynchronize(rt->ev2) != cudaSuccess) return GTAP_E_CUDA;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, rt->ev0, rt->ev1);
    const Ctl& c = *rt->h_ctl;
    if (out) {
        std::memset(out, 0, sizeof(*out));
        out->tasks = c.stats[gtap::ST_TASKS];
        out->invocations = c.stats[gtap::ST_INVOC];
        out->pops = c.stats[gtap::ST_POPS];
        out->kept = c.stats[gtap::ST_KEPT];
        out->steals_ok = c.stats[gtap::ST_STEALS_OK];
        out->steals_failed = c.stats[gtap::ST_STEALS_FAILED];
        out->stolen_tasks = c.stats[gtap::ST_STOLEN];
        out->pushes = c.stats[gtap::ST_PUSHES];
        out->cycles = c.stats[gtap::ST_CYCLES];
        out->idle_cycles = c.stats[gtap::ST_IDLE];
        out->remote_frees = c.stats[gtap::ST_REMOTE_FREES];
        out->max_pool_used = c.stats[gtap::ST_MAX_POOL];
        out->assists = (uint32_t)c.stats[gtap::ST_ASSISTS];
        out->error_word = c.error;
        out->workers = rt->run_W;
        out->device_ms = ms;
        out->grid_size = rt->run_grid;
        out->block_size = rt->run_block;
    }
    if (c.error) return static_cast<gtap_status>(c.error);
    if (!c.done) return GTAP_E_BAD_STATE;  // kernel exited without termination (should not happen)
    return GTAP_OK;
}

gtap_status gtap_root_result(gtap_runtime* rt, uint32_t root_idx, void* out, uint32_t nbytes) {
    if (!rt || !out || nbytes > 8) return GTAP_E_INVAL;
    if (rt->in_flight) return GTAP_E_BUSY;
    if (root_idx >= rt->run_nroots) return GTAP_E_INVAL;
    cudaSetDevice(rt->device);
    long long v = 0;
    if (cudaMemcpy(&v, rt->ws + rt->L.results + sizeof(long long) * root_idx, sizeof(v), cudaMemcpyDeviceToHost) !=
        cudaSuccess)
        return GTAP_E_CUDA;
    std::memcpy(out, &v, nbytes);
    return GTAP_OK;
}

gtap_status gtap_finalize(gtap_runtime* rt) {
    if (!rt) return GTAP_OK;
    cudaSetDevice(rt->device);
    if (rt->in_flight) cudaEventSynchronize(rt->ev2);
    if (rt->owns_ws && rt->ws) cudaFree(rt->ws);
    if (rt->chk) cudaFree(rt->chk);
    if (rt->vbuf) cudaFree(rt->vbuf);
    if (rt->h_roots) cudaFreeHost(rt->h_roots);
    if (rt->h_ctl) cudaFreeHost(rt->h_ctl);
    if (rt->ev0) cudaEventDestroy(rt->ev0);
    if (rt->ev1) cudaEventDestroy(rt->ev1);
    if (rt->ev2) cudaEventDestroy(rt->ev2);
    if (rt->ev_reset) cudaEventDestroy(rt->ev_reset);
    delete rt;
    return GTAP_OK;
}

gtap_status gtap_check_read(gtap_runtime* rt, uint64_t* out, uint32_t n) {
    if (!rt || !out || n < 21) return GTAP_E_INVAL;
#ifdef GTAP_CHECK
    if (rt->in_flight) return GTAP_E_BUSY;
    cudaSetDevice(rt->device);
    const size_t nw = check_words(rt);
    std::vector<uint32_t> a(3 * nw);
    unsigned long long ctr[gtap::CK_COUNT];
    if (cudaMemcpy(ctr, rt->chk, sizeof(ctr), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(a.data(), reinterpret_cast<char*>(rt->chk) + 256, 4 * a.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
        return GTAP_E_CUDA;
    for (int i = 0; i < gtap::CK_COUNT; ++i) out[i] = ctr[i];
    uint64_t live = 0, runnable = 0, kids = 0;
    for (size_t i = 0; i < nw; ++i) {
        live += a[i] != 0u;
        runnable += a[nw + i] != 0u;
        kids += a[2 * nw + i] != 0u;
    }
    out[16] = live;
    out[17] = runnable;
    out[18] = kids;
    const Ctl& c = *rt->h_ctl;
    out[19] = (uint64_t)c.outstanding;
    out[20] = c.roots_left;
    return GTAP_OK;
#else
    return GTAP_E_UNSUPPORTED;
#endif
}

void gtap_table_destroy(const gtap_task_table* t) {
    if (t && t->dev_scratch) cudaFree(t->dev_scratch);
    delete const_cast<gtap_task_table*>(t);
}


}  // extern "C"
