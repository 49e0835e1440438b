// gtap_internal.cuh -- workspace layout and sm_100a primitives shared by the
// persistent schedulers (sched_thread.cuh, sched_block.cuh) and the host
// runtime (runtime.cu). Product code: never includes anything from oracle/.
//
// Memory-consistency contract (§4.5: per-SM L1 is not
// coherent; use L1-bypassing accesses + fences for shared metadata):
//   * every read of shared mutable scheduler state (task records, deque ring
//     entries, deque metadata, free rings, control words) is a .relaxed.gpu
//     "strong" load (SASS LDG.E.STRONG.GPU: served by L2, never a stale L1
//     line) -- the sm_100a spelling of the paper's ld.global.cg;
//   * publication edges use release (MEMBAR.ALL.GPU + op): deque publication
//     (red.release on the packed head|split word) and the join decrement
//     (atom.acq_rel);
//   * every edge that hands a runnable task to another warp/SM ends in an
//     acquire on the receiving SM (steal CAS .acquire, join decrement
//     .acq_rel), which also invalidates that SM's L1 (CCTL.IVALL), so task
//     bodies may use ordinary cached loads for data their ancestors wrote.
#pragma once
#include <cstdint>

#ifndef GTAP_HOST_ONLY
#include <cuda_runtime.h>
#endif

namespace gtap {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kExit = 0xFFFFFFFEu;   // block scheduler: the cycle's task word when the block leaves
constexpr uint32_t kRootFlag = 0x80000000u;
constexpr int kDataWords = 4;  // 16-B payload per record (GTAP_MAX_TASK_DATA_SIZE default)

// Task record ("(i) a payload ... and (ii) metadata ... the task
// function, parent/child IDs, and a resumption state"). 32 B = one L2 sector;
// two 16-B vector accesses. Child results land in the parent's data[2 + ordinal]
// (copy-at-finish, R8), so a finished child's record is freed at once.
// The 8-B head {pending, acc} is one 64-bit atomic word: tables whose
// continuation only needs the SUM of the child results (fib, "a + b")
// deliver the result and the join decrement in one relaxed atom.add.u64
// (kJoinReduceAdd); other tables store into d[2 + ordinal] and decrement
// `pending` with acq_rel.
struct __align__(32) TaskRec {
    int32_t pending;   // outstanding children of the current join epoch
    uint32_t acc;      // sum of child results delivered with the decrement (kJoinReduceAdd)
    uint32_t meta;     // fn:8 | state:8 | ordinal:8 | queue:8
    uint32_t parent;   // parent record id; kRootFlag | root index for roots; kNone: no parent
    uint32_t d[kDataWords];
};
__host__ __device__ inline bool is_root_link(uint32_t parent) { return parent != 0xFFFFFFFFu && (parent & 0x80000000u); }
static_assert(sizeof(TaskRec) == 32, "record must be one 32-B sector");

__host__ __device__ inline uint32_t make_meta(uint32_t fn, uint32_t state, uint32_t ord, uint32_t q) {
    return (fn & 0xFF) | ((state & 0xFF) << 8) | ((ord & 0xFF) << 16) | ((q & 0xFF) << 24);
}
__host__ __device__ inline uint32_t meta_fn(uint32_t m) { return m & 0xFF; }
__host__ __device__ inline uint32_t meta_state(uint32_t m) { return (m >> 8) & 0xFF; }
__host__ __device__ inline uint32_t meta_ord(uint32_t m) { return (m >> 16) & 0xFF; }

// Per-deque shared metadata, one 64-B line each (no false sharing between
// victims). S packs head (steal end, low 32 bits) and split (high 32 bits):
// [head, split) is public (stealable), [split, tail) is the owner's private
// part (tail lives in the owner's registers, "tail is kept in
// shared memory because only the owner warp updates it").
struct __align__(64) DequeMeta {
    unsigned long long S;   // head | split << 32   (CAS by thieves / owner reclaim, red.add by owner publish)
    uint32_t steal_done;    // tasks whose ring slots thieves have finished reading
    uint32_t lock;          // serialises thieves of this deque
    uint32_t pad[12];
};
static_assert(sizeof(DequeMeta) == 64, "");

// Per-worker free-record ring (MPSC: any worker frees, the home worker
// allocates). Entries hold id+1 (0 = not yet written).
struct __align__(64) FreeMeta {
    uint32_t tail;          // producers atomicAdd
    uint32_t pad[15];
};

enum StatIdx : int {
    ST_TASKS = 0, ST_INVOC, ST_POPS, ST_KEPT, ST_STEALS_OK, ST_STEALS_FAILED, ST_STOLEN,
    ST_PUSHES, ST_CYCLES, ST_IDLE, ST_REMOTE_FREES, ST_MAX_POOL, ST_ASSISTS, ST_COUNT = 16
};

// Control block: each hot word on its own 128-B line.
struct __align__(128) Ctl {
    uint32_t done;            // termination flag (set once)
    uint32_t pad0[31];
    uint32_t error;           // sticky gtap_status
    uint32_t pad1[31];
    long long outstanding;    // no-taskwait termination counter (SPEC S:321 reading)
    uint32_t pad2[30];
    uint32_t roots_left;      // taskwait-closed termination: roots not yet finished
    // victim_policy 1 (die-aware stealing): vinfo = device {sm_die[256 bytes], vlist[]} -- the workers whose
    // deque line is homed in die 0's / die 1's L2 are vlist[0, vcnt[0]) / vlist[vcnt[2], vcnt[2] + vcnt[1]),
    // counts restricted to the run's workers; vinfo nullptr = uniform victims. Staged with the control block,
    // read-only during the run (kept out of KParams: a larger kernel-parameter block cost the fib kernel 13
    // registers)
    uint32_t vcnt[3];
    uint32_t pad3[25];
    const uint32_t* vinfo;
    unsigned long long stats[ST_COUNT];
    uint32_t pad4[32];
};

struct RootSpec {
    uint32_t fn;
    uint32_t d[kDataWords];
};

// GTAP_CHECK diagnostic build (§4.3.2 P:137-141 correctness sketch):
// per-record protocol tokens kept beside the workspace, checked at every scheduler event --
//   live[id]      1 while the record is allocated     (alloc / free must alternate: conservation),
//   runnable[id]  1 while the task is published and unclaimed (publish / dispatch alternate: every
//                 published (record, state) is claimed and dispatched exactly once),
//   kids[id]      children of the record's current join epoch not yet finished (a continuation may
//                 only be dispatched at 0; an independent count, not the scheduler's join word).
// Counters of events and violations live in ctr[]; a violation also raises GTAP_E_INVARIANT.
enum CheckCtr : int {
    CK_ALLOC = 0, CK_FREE, CK_PUBLISH, CK_DISPATCH, CK_SUSPEND, CK_JOIN, CK_RESUME,
    CK_V_DOUBLE_ALLOC, CK_V_DOUBLE_FREE, CK_V_DOUBLE_PUBLISH, CK_V_DISPATCH_UNPUBLISHED, CK_V_EARLY_RESUME,
    CK_V_JOIN_UNDERFLOW, CK_V_SUSPEND_DIRTY, CK_COUNT = 16
};
struct CheckBuf {
    unsigned long long ctr[CK_COUNT];
    uint32_t* live;
    uint32_t* runnable;
    int32_t* kids;
};

constexpr uint32_t kPolQueueStay = 1u, kPolDieVictims = 2u;   // KParams::policy bits

// Kernel parameters (by value): geometry + device pointers into one workspace.
struct KParams {
    uint32_t W;              // workers (warps or blocks)
    uint32_t logM;           // records per worker = 1 << logM
    uint32_t qmask;          // ring capacity - 1 (power of two)
    uint32_t steal_rounds;   // probe rounds per idle cycle
    uint32_t steal_max;      // max tasks per steal
    uint32_t nroots;
    uint32_t max_child;      // GTAP_MAX_CHILD_TASKS (runtime check)
    uint32_t idle_backoff;   // max idle nanosleep (ns)
    uint32_t nq;             // deques per worker in the workspace (GTAP_NUM_QUEUES, EPAQ)
    uint32_t policy;         // kPolQueueStay (EPAQ kept class: stay while the class has work, else rotate every
                             // cycle) | kPolDieVictims (victim_policy 1: die-aware steal victims, Ctl::vinfo)
    unsigned long long seed;
    unsigned long long watchdog_ns;
    TaskRec* rec;            // W << logM records
    uint32_t* ring;          // W * nq * (qmask+1)
    DequeMeta* dq;           // W * nq
    uint32_t* fring;         // W << logM
    FreeMeta* fm;            // W
    Ctl* ctl;
    const RootSpec* roots;   // nroots
    long long* root_results; // nroots
    CheckBuf* chk;           // GTAP_CHECK builds only (else nullptr)
    // victim_policy 1 (die-aware stealing): die of every SM, and the workers whose deque metadata line is
    // homed in die 0's / die 1's L2 (vlist[0, vcnt0) / vlist[vcnt0, vcnt0 + vcnt1)); nullptr: uniform victims
};

// die-aware victim choice: 3 of 4 probing lanes draw from the workers whose deque line is
// near the thief's die (their steal CAS and lock RMW stay in the near L2), the rest uniformly
int die_probe(const void* base, uint64_t stride, uint32_t n, uint8_t* sm_die, uint32_t cap, uint8_t* addr_near,
              float* out3, cudaStream_t s);

// Host-side layout of the workspace (offsets in bytes).
struct Layout {
    size_t rec, ring, dq, fring, fm, ctl, roots, results, total;
    uint32_t W, M, Q, max_roots, NQ;
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

inline Layout make_layout(uint32_t W, uint32_t M, uint32_t Q, uint32_t max_roots, uint32_t NQ = 1) {
    Layout L{};
    L.W = W; L.M = M; L.Q = Q; L.max_roots = max_roots; L.NQ = NQ;
    size_t o = 0;
    L.ctl = o;     o = align_up(o + sizeof(Ctl), 256);
    L.dq = o;      o = align_up(o + sizeof(DequeMeta) * (size_t)W * NQ, 256);
    L.fm = o;      o = align_up(o + sizeof(FreeMeta) * (size_t)W, 256);
    L.roots = o;   o = align_up(o + sizeof(RootSpec) * (size_t)max_roots, 256);
    L.results = o; o = align_up(o + sizeof(long long) * (size_t)max_roots, 256);
    L.fring = o;   o = align_up(o + sizeof(uint32_t) * (size_t)W * M, 256);
    L.ring = o;    o = align_up(o + sizeof(uint32_t) * (size_t)W * NQ * Q, 256);
    L.rec = o;     o = align_up(o + sizeof(TaskRec) * (size_t)W * M, 256);
    L.total = o;
    return L;
}

// Bytes that gtap_reset must zero: control block, deque metadata, free-ring
// metadata, and the free rings themselves (entries 0 = empty).
inline size_t reset_span_front(const Layout& L) { return L.roots; }

}  // namespace gtap

#ifndef GTAP_HOST_ONLY
namespace gtap {
// zero `bytes` of device memory on `s` with an SM kernel (runtime.cu; no copy engine, so it never
// queues behind a user's bulk copies); falls back to cudaMemsetAsync for unaligned ranges
cudaError_t zero_async(void* p, size_t bytes, cudaStream_t s);

namespace dev {

// ---- strong (L1-bypassing, L2-coherent) accesses ---------------------------
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int32_t ld_relaxed(const int32_t* p) {
    int32_t v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ long long ld_relaxed(const long long* p) {
    long long v;
    asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint4 ld_relaxed_v4(const void* p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
    return v;
}
// one 32-B record (one L2 sector) in a single 256-bit strong load (LDG.E.ENL2.256.STRONG.GPU on sm_100a)
__device__ __forceinline__ void ld_relaxed_v8(const void* p, uint4& lo, uint4& hi) {
    asm volatile("ld.relaxed.gpu.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(int32_t* p, int32_t v) {
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// weak vector store (published later by a release)
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
// one 32-B record in a single 256-bit store (STG.E.ENL2.256 on sm_100a)
__device__ __forceinline__ void st_v8(void* p, uint4 lo, uint4 hi) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(lo.x), "r"(lo.y), "r"(lo.z),
                 "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w)
                 : "memory");
}
__device__ __forceinline__ void st_v2(void* p, uint32_t a, uint32_t b) {
    asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}

// ---- atomics ----------------------------------------------------------------
__device__ __forceinline__ int32_t atom_add_acq_rel(int32_t* p, int32_t v) {
    int32_t o;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
    return o;
}
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
    uint32_t o;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
    return o;
}
__device__ __forceinline__ long long atom_add_acq_rel(long long* p, long long v) {
    long long o;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(v) : "memory");
    return o;
}
__device__ __forceinline__ uint32_t atom_add_acquire(uint32_t* p, uint32_t v) {
    uint32_t r;
    asm volatile("atom.acquire.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
    return r;
}
__device__ __forceinline__ uint32_t atom_add_relaxed(uint32_t* p, uint32_t v) {
    uint32_t o;
    asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
    return o;
}
__device__ __forceinline__ unsigned long long atom_add_relaxed_u64(void* p, unsigned long long v) {
    unsigned long long o;
    asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(v) : "memory");
    return o;
}
__device__ __forceinline__ void red_add_release(unsigned long long* p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_release(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_cas_acquire(unsigned long long* p, unsigned long long cmp,
                                                              unsigned long long val) {
    unsigned long long o;
    asm volatile("atom.acquire.gpu.global.cas.b64 %0, [%1], %2, %3;" : "=l"(o) : "l"(p), "l"(cmp), "l"(val)
                 : "memory");
    return o;
}
__device__ __forceinline__ unsigned long long atom_cas_relaxed(unsigned long long* p, unsigned long long cmp,
                                                              unsigned long long val) {
    unsigned long long o;
    asm volatile("atom.relaxed.gpu.global.cas.b64 %0, [%1], %2, %3;" : "=l"(o) : "l"(p), "l"(cmp), "l"(val)
                 : "memory");
    return o;
}
__device__ __forceinline__ uint32_t atom_cas_relaxed(uint32_t* p, uint32_t cmp, uint32_t val) {
    uint32_t o;
    asm volatile("atom.relaxed.gpu.global.cas.b32 %0, [%1], %2, %3;" : "=r"(o) : "l"(p), "r"(cmp), "r"(val)
                 : "memory");
    return o;
}
__device__ __forceinline__ uint32_t atom_exch_relaxed(uint32_t* p, uint32_t v) {
    uint32_t o;
    asm volatile("atom.relaxed.gpu.global.exch.b32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
    return o;
}
__device__ __forceinline__ uint32_t atom_exch_release(uint32_t* p, uint32_t v) {
    uint32_t o;
    asm volatile("atom.release.gpu.global.exch.b32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
    return o;
}
__device__ __forceinline__ void red_add_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void nanosleep(uint32_t ns) { asm volatile("nanosleep.u32 %0;" ::"r"(ns)); }

__device__ __forceinline__ uint32_t smid() {
    uint32_t s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}
__device__ __forceinline__ uint32_t xorshift32(uint32_t& s) {
    s ^= s << 13;
    s ^= s >> 17;
    s ^= s << 5;
    return s;
}

// a steal victim != w from the random draw r: with victim_policy 1 (policy & kPolDieVictims) lanes < 24 draw from
// the workers whose deque line is near the thief's die, the others uniformly. The uniform draw is a
// multiply-high range reduction of r (no integer division: idle warps probing for work share the issue slots
// of the busy warps on their SM; `r % (W - 1)` was 5 % of the mergesort kernel's instructions)
__device__ __forceinline__ uint32_t pick_victim(uint32_t W, uint32_t w, uint32_t lane, uint32_t r, const Ctl* ctl,
                                                uint32_t policy) {
    if ((policy & kPolDieVictims) && lane < 24u) {
        const uint32_t* vi = reinterpret_cast<const uint32_t*>(__ldg(reinterpret_cast<const unsigned long long*>(&ctl->vinfo)));
        if (vi != nullptr) {
            const uint32_t mydie = __ldg(reinterpret_cast<const uint8_t*>(vi) + smid());
            const uint32_t cnt = __ldg(&ctl->vcnt[mydie]);
            if (cnt > 1u) {
                const uint32_t v = __ldg(vi + 64 + (mydie ? __ldg(&ctl->vcnt[2]) : 0u) + __umulhi(r, cnt));
                return v != w ? v : (v + 1u < W ? v + 1u : 0u);
            }
        }
    }
    const uint32_t v = __umulhi(r, W - 1u);
    return v + (v >= w);
}
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}


__device__ __forceinline__ uint32_t hash32(unsigned long long x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return (uint32_t)x | 1u;
}

// Warp-wide exclusive prefix sum of v (all 32 lanes participate).
__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t lane, uint32_t& total) {
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

// Sticky device error: first writer wins; also raises the termination flag.
__device__ __forceinline__ void raise_error(Ctl* ctl, uint32_t code) {
    atom_cas_relaxed(&ctl->error, 0u, code);
    st_release(&ctl->done, 1u);
}

// ---- GTAP_CHECK hooks (compiled only into the diagnostic check build) -------
#ifdef GTAP_CHECK
#define GTAP_CK(...) do { __VA_ARGS__; } while (0)
__device__ __forceinline__ void ck_violation(const KParams& p, int k) {
    atomicAdd(&p.chk->ctr[k], 1ull);
    raise_error(p.ctl, GTAP_E_INVARIANT);
}
// a record leaves the free pool (root entry, child spawn); the fence orders the token before the
// record's later hand-over (its ring / free-ring store)
__device__ __forceinline__ void ck_alloc(const KParams& p, uint32_t id) {
    __threadfence();
    atomicAdd(&p.chk->ctr[CK_ALLOC], 1ull);
    if (atomicExch(&p.chk->live[id], 1u) != 0u) ck_violation(p, CK_V_DOUBLE_ALLOC);
}
__device__ __forceinline__ void ck_free(const KParams& p, uint32_t id) {
    atomicAdd(&p.chk->ctr[CK_FREE], 1ull);
    if (atomicExch(&p.chk->live[id], 0u) != 1u) ck_violation(p, CK_V_DOUBLE_FREE);
    __threadfence();
}
// a (record, state) becomes runnable: root entry, spawn, last-child resume, empty-join resume
__device__ __forceinline__ void ck_publish(const KParams& p, uint32_t id) {
    atomicAdd(&p.chk->ctr[CK_PUBLISH], 1ull);
    if (atomicExch(&p.chk->runnable[id], 1u) != 0u) ck_violation(p, CK_V_DOUBLE_PUBLISH);
#if defined(GTAP_CHECK_SELFTEST) && GTAP_CHECK_SELFTEST == 1
    if (id == 0u && atomicExch(&p.chk->runnable[id], 1u) != 0u) ck_violation(p, CK_V_DOUBLE_PUBLISH);  // injected
#endif
    __threadfence();
}
// a worker claimed the task and is about to run (record, state)
__device__ __forceinline__ void ck_dispatch(const KParams& p, uint32_t id, uint32_t state) {
    __threadfence();
    atomicAdd(&p.chk->ctr[CK_DISPATCH], 1ull);
    if (atomicExch(&p.chk->runnable[id], 0u) != 1u) ck_violation(p, CK_V_DISPATCH_UNPUBLISHED);
    if (state != 0u) {
        atomicAdd(&p.chk->ctr[CK_RESUME], 1ull);
        if (ld_relaxed(&p.chk->kids[id]) != 0) ck_violation(p, CK_V_EARLY_RESUME);
    }
}
__device__ __forceinline__ void ck_suspend(const KParams& p, uint32_t id, uint32_t nchildren) {
    atomicAdd(&p.chk->ctr[CK_SUSPEND], 1ull);
    if (atomicExch(reinterpret_cast<uint32_t*>(&p.chk->kids[id]), nchildren) != 0u) ck_violation(p, CK_V_SUSPEND_DIRTY);
    __threadfence();
}
// a child of `parent` finished (before the scheduler's own join RMW; the fence orders the two)
__device__ __forceinline__ void ck_join(const KParams& p, uint32_t parent) {
#if defined(GTAP_CHECK_SELFTEST) && GTAP_CHECK_SELFTEST == 2
    if (parent % 5u == 0u) return;   // injected: a lost child join, so that parent's continuation must be flagged
#endif
    atomicAdd(&p.chk->ctr[CK_JOIN], 1ull);
    if (atomicAdd(&p.chk->kids[parent], -1) < 1) ck_violation(p, CK_V_JOIN_UNDERFLOW);
    __threadfence();
}
#else
#define GTAP_CK(...) do { } while (0)
#endif

}  // namespace dev

#ifdef GTAP_TRACE
// Diagnostic task trace (diagnostic builds only, SURVEY.md §5 "tracing"): one record per task
// invocation {start ns, end ns, worker | state << 24, d0, d1}.
struct TraceRec {
    unsigned long long t0, t1;
    uint32_t who, d0, d1, pad;
};
constexpr uint32_t kTraceCap = 1u << 22;
__device__ TraceRec g_trace[kTraceCap];
__device__ uint32_t g_trace_n;
__device__ __forceinline__ void trace_rec(unsigned long long t0, uint32_t who, uint32_t d0, uint32_t d1) {
    const uint32_t i = atomicAdd(&g_trace_n, 1u);
    if (i < kTraceCap) {
        TraceRec r;
        r.t0 = t0; r.t1 = dev::globaltimer(); r.who = who; r.d0 = d0; r.d1 = d1; r.pad = 0;
        g_trace[i] = r;
    }
}
// device globals are per translation unit (no -rdc): each table file defines its own reader
#define GTAP_TRACE_READER(NAME)                                                                        \
    extern "C" int gtap_trace_read_##NAME(void* host, uint32_t cap, uint32_t* n) {                     \
        uint32_t cnt = 0;                                                                              \
        cudaMemcpyFromSymbol(&cnt, gtap::g_trace_n, 4);                                                \
        *n = cnt;                                                                                      \
        uint32_t m = cnt < cap ? cnt : cap;                                                            \
        if (m > gtap::kTraceCap) m = gtap::kTraceCap;                                                  \
        if (m) cudaMemcpyFromSymbol(host, gtap::g_trace, sizeof(gtap::TraceRec) * m);                  \
        const uint32_t z = 0;                                                                          \
        cudaMemcpyToSymbol(gtap::g_trace_n, &z, 4);                                                    \
        return 0;                                                                                      \
    }
#endif
}  // namespace gtap
#endif
