// sched_thread.cuh -- thread-level persistent scheduler ("thread-executed"
// mode, §4.1; queue design §4.3.2; EPAQ §4.4
// P:146-178).
//
// One worker = one warp. Each persistent-kernel cycle a warp
//   (1) acquires up to 32 runnable task IDs: the set kept from its previous
//       cycle, then a LIFO batch from its own deque, then (only if still
//       empty) a FIFO batch stolen from a random victim;
//   (2) executes them, one task per lane, as switch-on-state functions
//       (P:52-55): exec() returns spawn requests + finish/suspend;
//   (3) allocates child records from the warp's pool, joins (atomic pending
//       decrement, last child re-enqueues the parent), keeps up to 32
//       runnable tasks for the next cycle and pushes the rest, and
//       publishes part of its private deque when thieves have drained the
//       public part.
//
// Deque (B200 design): a power-of-two ring per warp and
// queue in HBM with a packed 64-bit word S = head | split << 32. The owner
// pushes and pops at the tail of the PRIVATE part [split, tail) with no
// atomics at all (tail and split live in registers -- only the owner moves
// them). Thieves CAS S to claim [head, head + c) of the PUBLIC part
// [head, split) under a per-victim try-lock; the owner
// publishes the oldest half of its private part with one red.release when it
// sees the public part empty, and reclaims from the public part by CAS only
// when its private part and kept set are empty. This keeps the paper's
// batched claim-by-CAS for steals but moves the owner's common-case
// pop off the shared counter whose contention the paper identifies as its
// scaling limit.
//
// EPAQ (NQ = T::kNumQueues > 1): every warp owns NQ such deques.
// A child's queue is chosen at spawn (queue(expr)) and a
// continuation's at taskwait; the suspended parent keeps that
// index in the top byte of its join word, so the last child learns it from
// the atomic's return value. Acquisition goes round-robin over the queues
// starting from the one used last, thieves probe the victims'
// queues the same way, and the kept set holds ONE queue class (the next one in
// the rotation), so a warp runs tasks of one execution path per cycle.
#pragma once
#include "gtap.h"
#include "gtap_internal.cuh"

namespace gtap {

// What one thread-level invocation produced (the runtime side of
// __gtap_prepare_for_join / __gtap_finish_task).
template <int MAXC>
struct TOut {
    uint32_t action;      // 0 = none, 1 = finish, 2 = suspend
    uint32_t nchild;
    uint32_t next_state;
    uint32_t next_queue;  // taskwait queue(expr) (EPAQ)
    uint32_t has_result;
    int32_t result;
    uint32_t err;
    uint32_t cfn[MAXC];
    uint32_t cq[MAXC];    // spawn queue(expr) (EPAQ)
    uint32_t cd[MAXC][kDataWords];
    // generated children (tables with kGenChildren): child c is T::gen_child(gen, gmask, c, ...)
    uint32_t gen[kDataWords];
    uint32_t gmask;
    // warp assist (tables with kAssist): the body's heavy leaf routine is run by the whole warp
    // after this cycle's bodies, before the task's spawns/join/finish are processed
    uint32_t assist;
    uint32_t ap[kDataWords];
    static constexpr uint32_t kFinish = 1, kSuspend = 2;
    __device__ __forceinline__ void init() {
        action = 0; nchild = 0; has_result = 0; err = 0; result = 0; next_state = 0; next_queue = 0;
        assist = 0;
    }
    __device__ __forceinline__ void request_assist(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
        assist = 1; ap[0] = a0; ap[1] = a1; ap[2] = a2; ap[3] = a3;
    }
    // spawn child #i (i is a compile-time constant after inlining) into queue q
    __device__ __forceinline__ void spawn_q(int i, uint32_t q, uint32_t fn, uint32_t d0, uint32_t d1 = 0,
                                            uint32_t d2 = 0, uint32_t d3 = 0) {
        if (i >= MAXC) { err = GTAP_E_CHILD_LIMIT; return; }
        cfn[i] = fn; cq[i] = q; cd[i][0] = d0; cd[i][1] = d1; cd[i][2] = d2; cd[i][3] = d3;
        nchild = (uint32_t)i + 1 > nchild ? (uint32_t)i + 1 : nchild;
    }
    __device__ __forceinline__ void spawn(int i, uint32_t fn, uint32_t d0, uint32_t d1 = 0, uint32_t d2 = 0,
                                          uint32_t d3 = 0) {
        spawn_q(i, 0u, fn, d0, d1, d2, d3);
    }
    __device__ __forceinline__ void suspend(uint32_t next, uint32_t q = 0) {
        action = kSuspend; next_state = next; next_queue = q;
    }
    __device__ __forceinline__ void finish(int32_t r) { action = kFinish; has_result = 1; result = r; }
    __device__ __forceinline__ void finish_void() { action = kFinish; }
    __device__ __forceinline__ void bad_state() { action = kFinish; err = GTAP_E_BAD_STATE; }
};

constexpr uint32_t kHeavyBit = 0x80000000u;  // transient flag on runnable IDs (IDs < 2^31)
constexpr uint32_t kPendMask = 0x00FFFFFFu;  // join word: count in bits 0-23, resume queue in 24-31

// Placement hint (semantics-free, like EPAQ's queue choice P:990): a table may
// mark tasks "heavy" (e.g. a mergesort subtree whose merges are large) so the
// scheduler never keeps two of them in one warp.
template <class T>
__device__ __forceinline__ bool task_is_heavy(uint32_t fn, const uint32_t* d) {
    if constexpr (T::kHasHeavy) return T::heavy(fn, d);
    else return false;
}
template <class T>
__device__ __forceinline__ bool parent_is_heavy(uint32_t child_fn, const uint32_t* child_d) {
    if constexpr (T::kHasHeavy) return T::heavy_parent(child_fn, child_d);
    else return false;
}
template <class T, class = void>
struct gen_children_of { static constexpr bool value = false; };
template <class T>
struct gen_children_of<T, decltype((void)T::kGenChildren, void())> { static constexpr bool value = T::kGenChildren; };

// a word idle warps poll while they probe steal victims (e.g. mergesort's GPU-wide assist board: nonzero while a
// slot is open); lane 31 reads it instead of a victim's deque word, and a failed steal round that saw it set goes
// to T::help_idle at once
template <class T, class = void>
struct idle_word_of { static constexpr bool value = false; };
template <class T>
struct idle_word_of<T, decltype((void)T::kIdleWord, void())> { static constexpr bool value = T::kIdleWord; };

template <class T, class = void>
struct assist_of { static constexpr bool value = false; };
template <class T>
struct assist_of<T, decltype((void)T::kAssist, void())> { static constexpr bool value = T::kAssist; };

#ifndef GTAP_FSTACK
#define GTAP_FSTACK 256
#endif
// own free-stack depth per warp: GTAP_FSTACK unless the table sets kFreeStack
template <class T, class = void>
struct free_stack_of { static constexpr int value = GTAP_FSTACK; };
template <class T>
struct free_stack_of<T, decltype((void)T::kFreeStack, void())> { static constexpr int value = T::kFreeStack; };

template <class T, class = void>
struct stats_smem_of { static constexpr bool value = false; };
template <class T>
struct stats_smem_of<T, decltype((void)T::kStatsSmem, void())> { static constexpr bool value = T::kStatsSmem; };

template <class T, class = void>
struct num_queues_of { static constexpr int value = 1; };
template <class T>
struct num_queues_of<T, decltype((void)T::kNumQueues, void())> { static constexpr int value = T::kNumQueues; };

// per-queue owner state lives in registers; q is warp-uniform, the loops unroll to selects
template <int NQ>
__device__ __forceinline__ uint32_t qget(const uint32_t (&a)[NQ], uint32_t q) {
    uint32_t v = a[0];
#pragma unroll
    for (int i = 1; i < NQ; ++i) if (q == (uint32_t)i) v = a[i];
    return v;
}
template <int NQ>
__device__ __forceinline__ void qset(uint32_t (&a)[NQ], uint32_t q, uint32_t v) {
#pragma unroll
    for (int i = 0; i < NQ; ++i) if (q == (uint32_t)i) a[i] = v;
}

// per-warp LIFO stack of the warp's own surplus freed records (0: every surplus free goes to the
// home free ring, reused FIFO). A record freed and reused soon is still in L2; the FIFO ring hands
// out the coldest record, so with a live set larger than L2 the next spawn's stores and the join
// RMWs on it went to DRAM (fib(40), ncu: 45 % of the join atomics missed L2).
template <int MAXC, int FS = GTAP_FSTACK>
struct WarpSmem {
    unsigned long long st[12];  // per-warp statistics (lane 0, shared atomics: no registers held across the loop)
    uint32_t kept[32];          // keep-for-next-cycle set
    uint32_t fbuf[32];          // records freed this cycle (reused first)
    uint32_t abuf[32 * MAXC];   // records drawn from the free ring / bump region
    uint32_t cbuf[32 * MAXC];   // child IDs spawned this cycle, spawn order (generic path)
    uint32_t pbuf[32];          // parents made runnable this cycle (generic path)
    uint8_t cqb[32 * MAXC];     // queue of each cbuf entry (EPAQ)
    uint8_t pqb[32];            // queue of each pbuf entry (EPAQ)
    uint32_t fstack[FS > 0 ? FS : 1];  // own freed records, LIFO (L2-hot reuse)
};

template <class T>
__host__ __device__ constexpr size_t block_extra_bytes() {
    return (sizeof(typename T::BlockExtra) + 127) / 128 * 128;
}

#ifdef GTAP_CYC_HIST
// diagnostic build only: per busy cycle, hist[n] += 1 (n = tasks run, 1..32); hist[33] += cycles with n < 32 whose
// private parts were empty while a public part of the own deque held tasks; hist[34] += those public tasks
static __device__ unsigned long long gtap_cyc_hist[40];
#endif

template <class T>
__global__ void __launch_bounds__(T::kMaxThreads, T::kMinBlocks) thread_sched_kernel(KParams p, typename T::Args args) {
    using namespace dev;
    constexpr int MAXC = T::kMaxChildren;
    constexpr int NQ = num_queues_of<T>::value;
    constexpr bool kGeneric = T::kHasHeavy || NQ > 1;  // placement through smem lists
    constexpr bool kGen = gen_children_of<T>::value;  // children described by a generator (N-Queens)
    using Out = TOut<kGen ? 1 : MAXC>;
    extern __shared__ __align__(16) unsigned char smem_raw[];

    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t wib = threadIdx.x >> 5;
    const uint32_t w = blockIdx.x * (blockDim.x >> 5) + wib;
    // dynamic smem: [per-block table scratch (e.g. TMA merge slot)] [per-warp scheduler buffers]
    typename T::BlockExtra* bx = reinterpret_cast<typename T::BlockExtra*>(smem_raw);
    if (threadIdx.x == 0) T::block_init(bx);
    __syncthreads();
    if (w >= p.W) return;  // whole warp
    constexpr int FS = free_stack_of<T>::value;
    WarpSmem<MAXC, FS>& sm = reinterpret_cast<WarpSmem<MAXC, FS>*>(smem_raw + block_extra_bytes<T>())[wib];

    const uint32_t M = 1u << p.logM, mmask = M - 1u;
    const uint32_t Q = p.qmask + 1u, qmask = p.qmask;
    // deque (w, q) is number w * p.nq + q (p.nq >= NQ: the workspace may hold more queues)
    const uint32_t dq0 = w * p.nq;
    uint32_t* myfring = p.fring + ((size_t)w << p.logM);
    const uint32_t base_id = w << p.logM;
    const uint32_t lt = lanemask_lt();

    // owner-local deque / pool state (warp-uniform, in registers)
    uint32_t tail[NQ], split[NQ], sdone[NQ];
#pragma unroll
    for (int i = 0; i < NQ; ++i) tail[i] = split[i] = sdone[i] = 0;
    uint32_t qc = 0;  // queue of the tasks in hand (EPAQ round-robin position)
    uint32_t bump = 0, fhead = 0, fsp = 0;   // fsp: own free-stack depth (warp-uniform)
    uint32_t nkept = 0;
    uint32_t pub_hint = 0;   // own public part (queue 0) seen at the last publication check (thread-level, NQ == 1)
    uint32_t rng = hash32(p.seed * 0x9E3779B97F4A7C15ull + (unsigned long long)w * 32u + lane);
    uint32_t backoff = 32;
    // per-warp statistics (lane 0 counts): 32-bit registers folded into the warp's 64-bit shared-memory
    // counters every 2^16 loop iterations (at most 2^7 per counter per iteration: no overflow) and at exit;
    // tables with kStatsSmem add straight into shared memory (12 register counters cost the mergesort
    // kernel spills at its 128-register cap)
    constexpr bool kStSmem = stats_smem_of<T>::value;
    enum { kStTasks, kStInv, kStPops, kStKept, kStSok, kStSfail, kStStolen, kStPush, kStCyc, kStIdle, kStRfree,
           kStAssist, kStN };
    uint32_t streg[kStSmem ? 1 : kStN];
#pragma unroll
    for (int k = 0; k < (kStSmem ? 1 : kStN); ++k) streg[k] = 0u;
    if (lane < (uint32_t)kStN) sm.st[lane] = 0ull;
    __syncwarp();
    auto stat = [&](int k, uint32_t v) {
        if constexpr (kStSmem) atomicAdd(&sm.st[k], (unsigned long long)v); else streg[k] += v;
    };
    auto stflush = [&]() {   // lane 0
        if constexpr (!kStSmem) {
#pragma unroll
            for (int k = 0; k < kStN; ++k) { sm.st[k] += streg[k]; streg[k] = 0u; }
        }
    };
    auto stget = [&](int k) -> unsigned long long { return sm.st[k]; };
    const unsigned long long t0 = globaltimer();
    const bool wd_on = p.watchdog_ns != 0ull;
    uint32_t cyc_u = 0;  // warp-uniform loop-iteration counter (statistics flush, watchdog)
    bool failed = false;

    // ---- entry: roots r = w, w + W, ... go to this warp's queue 0
    {
        uint32_t mine = p.nroots > w ? (p.nroots - w + p.W - 1) / p.W : 0;
        if (mine > M || mine > Q) {
            if (lane == 0) raise_error(p.ctl, GTAP_E_POOL_EXHAUSTED);
            mine = 0;
        }
        uint32_t* ring0 = p.ring + (size_t)dq0 * Q;
        for (uint32_t i = lane; i < mine; i += 32) {
            const uint32_t r = w + i * p.W;
            const RootSpec rs = p.roots[r];
            const uint32_t id = base_id + i;
            TaskRec* rec = p.rec + id;
            st_v4(rec, make_uint4(0u, 0u, make_meta(rs.fn, 0, 0, 0), kRootFlag | r));
            st_v4(&rec->d[0], make_uint4(rs.d[0], rs.d[1], rs.d[2], rs.d[3]));
            GTAP_CK(ck_alloc(p, id); ck_publish(p, id));
            ring0[i & qmask] = id;
        }
        bump = mine;
        tail[0] = mine;
        if (lane == 0) stat(kStTasks, mine);
        __syncwarp();
    }

    while (true) {
        if (((++cyc_u) & 0xFFFFu) == 0u && lane == 0) stflush();
        if constexpr (assist_of<T>::value) T::help(args, lane, bx);  // join the block's open assist, if any
        // ================= (1) acquire =================
        uint32_t n = nkept;
        uint32_t my = (lane < n) ? (sm.kept[lane] & ~kHeavyBit) : kNone;
        // lane q holds the own S word of queue q (used for reclaim and the publication check)
        unsigned long long S_lane = 0;
        uint32_t done_seen = 0;
        if (lane < (uint32_t)NQ) S_lane = ld_relaxed(&p.dq[dq0 + lane].S);
        if (lane == 31) done_seen = ld_relaxed(&p.ctl->done);
        if (lane == 0) stat(kStKept, n);
        // LIFO pop from a private part, round-robin over the queues from qc: no atomics (owner only)
        if (n < 32) {
#pragma unroll
            for (int k = 0; k < NQ; ++k) {
                const uint32_t q = (qc + (uint32_t)k) % (uint32_t)NQ;
                // kept tasks are of queue qc: only top them up from qc itself
                if (k > 0 && n > 0) break;
                const uint32_t tq = qget(tail, q);
                const uint32_t priv = tq - qget(split, q);
                if (priv > 0) {
                    const uint32_t c = min(32u - n, priv);
                    uint32_t* ringq = p.ring + (size_t)(dq0 + q) * Q;
                    if (lane >= n && lane < n + c) my = ld_relaxed(&ringq[(tq - 1u - (lane - n)) & qmask]);
                    qset(tail, q, tq - c);
                    n += c;
                    qc = q;
                    if (lane == 0) stat(kStPops, c);
                    break;
                }
            }
        }
#ifndef GTAP_RECLAIM_PARTIAL
#define GTAP_RECLAIM_PARTIAL 1
#endif
        // a partly filled cycle with an empty private part takes back tasks of its own public part that no thief
        // has claimed since they were published (fib(40): 14 % of the cycles, ~9 public tasks each; 10.64 ->
        // 10.13 ms); not for tables that publish on purpose (heavy hints, EPAQ, warp assists)
        if (GTAP_RECLAIM_PARTIAL && !kGeneric && !assist_of<T>::value && n > 0u && n < 32u && pub_hint != 0u && tail[0] == split[0]) {
            const unsigned long long sq = __shfl_sync(0xffffffffu, S_lane, 0);
            uint32_t got = 0, s_new = 0;
            if (lane == 0) {
                unsigned long long s = sq;
                for (int it = 0; it < 4; ++it) {
                    const uint32_t h = (uint32_t)s, sp = (uint32_t)(s >> 32);
                    const uint32_t avail = sp - h;
                    if (avail == 0u || avail > Q) break;
                    const uint32_t c = min(32u - n, avail);
                    const unsigned long long nw = ((unsigned long long)(sp - c) << 32) | h;
                    const unsigned long long o = atom_cas_relaxed(&p.dq[dq0].S, s, nw);
                    if (o == s) { got = c; s_new = sp - c; break; }
                    s = o;
                }
            }
            got = __shfl_sync(0xffffffffu, got, 0);
            if (got) {
                s_new = __shfl_sync(0xffffffffu, s_new, 0);
                split[0] = s_new;
                tail[0] = s_new;
                uint32_t* ring0 = p.ring + (size_t)dq0 * Q;
                if (lane >= n && lane < n + got) my = ld_relaxed(&ring0[(s_new + got - 1u - (lane - n)) & qmask]);
                n += got;
                if (lane == 0) stat(kStPops, got);
            }
            pub_hint = 0;
        }
        // reclaim from an own public part (only when nothing else to run)
        if (n == 0) {
#pragma unroll
            for (int k = 0; k < NQ; ++k) {
                const uint32_t q = (qc + (uint32_t)k) % (uint32_t)NQ;
                const unsigned long long sq = __shfl_sync(0xffffffffu, S_lane, q);
                uint32_t got = 0, s_new = 0;
                if (lane == 0) {
                    unsigned long long s = sq;
                    for (int it = 0; it < 8; ++it) {
                        const uint32_t h = (uint32_t)s, sp = (uint32_t)(s >> 32);
                        const uint32_t avail = sp - h;
                        if (avail == 0u || avail > Q) break;
                        // a small public part (top-of-tree / heavy tasks) is shared: take half (>= 1)
                        const uint32_t c = avail <= 4u ? max(1u, avail >> 1) : min(32u, avail);
                        const unsigned long long nw = ((unsigned long long)(sp - c) << 32) | h;
                        const unsigned long long o = atom_cas_relaxed(&p.dq[dq0 + q].S, s, nw);
                        if (o == s) { got = c; s_new = sp - c; break; }
                        s = o;
                    }
                }
                got = __shfl_sync(0xffffffffu, got, 0);
                s_new = __shfl_sync(0xffffffffu, s_new, 0);
                if (got) {
                    qset(split, q, s_new);
                    qset(tail, q, s_new);
                    uint32_t* ringq = p.ring + (size_t)(dq0 + q) * Q;
                    if (lane < got) my = ld_relaxed(&ringq[(s_new + got - 1u - lane) & qmask]);
                    n = got;
                    qc = q;
                    if (lane == 0) stat(kStPops, got);
                    break;
                }
            }
        }
        // an open GPU-wide assist (warp-assist tables) goes before stealing: its requester's task
        // is on the critical path, and when one is open the deques are mostly empty
        if constexpr (assist_of<T>::value) {
            if (n == 0 && T::help_idle(args, lane, bx)) { backoff = 32; continue; }
        }
        // steal: probe 32 random (victim, queue) pairs in parallel, claim from the fullest
        if (n == 0 && p.W > 1) {
            // a long-idle warp probes once per wake-up (keeps idle L2 traffic off busy workers)
            const uint32_t rounds = backoff >= 4096u ? 1u : p.steal_rounds;
            bool board = false;
            for (uint32_t round = 0; round < rounds && n == 0; ++round) {
                const uint32_t v = pick_victim(p.W, w, lane, xorshift32(rng), p.ctl, p.policy);
                const uint32_t vq = (qc + lane) % (uint32_t)NQ;  // EPAQ: round-robin from the own position
                const uint32_t vd = v * p.nq + vq;
                uint32_t avail = 0, polled = 0;
                if (idle_word_of<T>::value && lane == 31u) {
                    if constexpr (idle_word_of<T>::value) {
                        const uint32_t* pw = T::idle_word(args);
                        polled = pw ? ld_relaxed(pw) : 0u;
                    }
                } else {
                    const unsigned long long sv = ld_relaxed(&p.dq[vd].S);
                    avail = (uint32_t)(sv >> 32) - (uint32_t)sv;
                    if (avail > Q) avail = 0;
                }
                // warp arg-max over (avail, lane)
                uint32_t best = (min(avail, (1u << 26)) << 5) | lane;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
                if ((best >> 5) == 0) {
                    if (lane == 0) stat(kStSfail, 1);
                    if (idle_word_of<T>::value && __shfl_sync(0xffffffffu, polled, 31) != 0u) { board = true; break; }
                    continue;
                }
                const uint32_t bl = best & 31u;
                const uint32_t vdq = __shfl_sync(0xffffffffu, vd, bl);
                const uint32_t vqq = __shfl_sync(0xffffffffu, vq, bl);
                DequeMeta* vm = p.dq + vdq;
                uint32_t got = 0, h0 = 0;
                if (lane == 0) {
                    if (atom_cas_relaxed(&vm->lock, 0u, 1u) == 0u) {  // try-lock
                        unsigned long long s = ld_relaxed(&vm->S);
                        for (int it = 0; it < 8; ++it) {
                            const uint32_t h = (uint32_t)s, sp = (uint32_t)(s >> 32);
                            const uint32_t a = sp - h;
                            if (a == 0u || a > Q) break;
                            // claim up to steal_max; half of a small public part
                            const uint32_t c = a <= 4u ? (a + 1u) >> 1 : min(p.steal_max, a);
                            const unsigned long long nw = ((unsigned long long)sp << 32) | (uint32_t)(h + c);
                            const unsigned long long o = atom_cas_acquire(&vm->S, s, nw);
                            if (o == s) { got = c; h0 = h; break; }
                            s = o;
                        }
                        if (got == 0u) st_relaxed(&vm->lock, 0u);
                    }
                }
                got = __shfl_sync(0xffffffffu, got, 0);
                h0 = __shfl_sync(0xffffffffu, h0, 0);
                if (got) {
                    // advance the read prefix only after loading the stolen IDs
                    if (lane < got) my = ld_relaxed(&p.ring[(size_t)vdq * Q + ((h0 + lane) & qmask)]);
                    __syncwarp();
                    if (lane == 0) {
                        red_add_release(&vm->steal_done, got);
                        st_relaxed(&vm->lock, 0u);
                        stat(kStSok, 1);
                        stat(kStStolen, got);
                    }
                    n = got;
                    qc = vqq;
                } else if (lane == 0) {
                    stat(kStSfail, 1);
                }
            }
            if constexpr (assist_of<T>::value && idle_word_of<T>::value) {
                if (n == 0 && board && T::help_idle(args, lane, bx)) { backoff = 32; continue; }
            }
        }
        done_seen = __shfl_sync(0xffffffffu, done_seen, 31);
        if (n == 0) {
            // idle: termination check + watchdog + backoff
            if (lane == 0) stat(kStIdle, 1);
            uint32_t d = 0;
            if (lane == 0) d = ld_relaxed(&p.ctl->done);
            d = __shfl_sync(0xffffffffu, d, 0);
            if (d) break;
            if (p.watchdog_ns && lane == 0 && globaltimer() - t0 > p.watchdog_ns) raise_error(p.ctl, GTAP_E_TIMEOUT);
            if constexpr (assist_of<T>::value) {
                if (T::help_idle(args, lane, bx)) { backoff = 32; continue; }  // helped an open assist
            }
            nanosleep(backoff);
            backoff = min(backoff * 2u, p.idle_backoff);
            continue;
        }
        backoff = 32;
        if (lane == 0) { stat(kStCyc, 1); stat(kStInv, n); }
#ifdef GTAP_CYC_HIST
        {
            const unsigned long long s0 = __shfl_sync(0xffffffffu, S_lane, 0);
            const uint32_t pub = (uint32_t)(s0 >> 32) - (uint32_t)s0;
            if (lane == 0) {
                atomicAdd(&gtap_cyc_hist[n], 1ull);
                if (n < 32u && tail[0] == split[0] && pub > 0u && pub <= Q) {
                    atomicAdd(&gtap_cyc_hist[33], 1ull);
                    atomicAdd(&gtap_cyc_hist[34], (unsigned long long)pub);
                }
            }
        }
#endif

        // ================= (2) execute, one task per lane =================
        Out o;
        o.init();
        uint32_t parent = kNone, ord = 0, myfn = 0;
        uint32_t mydata[kDataWords] = {0, 0, 0, 0};
        if (my != kNone) {
            uint4 h, dv;
            ld_relaxed_v8(p.rec + my, h, dv);   // header + payload: one 256-bit request
            const uint32_t d[kDataWords] = {dv.x, dv.y, dv.z, dv.w};
            if (T::kHasHeavy) { mydata[0] = dv.x; mydata[1] = dv.y; mydata[2] = dv.z; mydata[3] = dv.w; }
            parent = h.w;
            ord = meta_ord(h.z);
            myfn = meta_fn(h.z);
            GTAP_CK(ck_dispatch(p, my, meta_state(h.z)));
            T::exec(args, meta_fn(h.z), meta_state(h.z), d, o, bx);
            if (o.action == 0u) o.err = GTAP_E_BAD_STATE;
            if (NQ > 1 && !kGen) {  // queue(expr) out of range is a usage error
                if (o.action == Out::kSuspend && o.next_queue >= (uint32_t)NQ) o.err = GTAP_E_INVAL;
#pragma unroll
                for (int c = 0; c < MAXC; ++c)
                    if ((uint32_t)c < o.nchild && o.cq[c] >= (uint32_t)NQ) o.err = GTAP_E_INVAL;
            }
            if (kGen && o.nchild > (uint32_t)MAXC) o.err = GTAP_E_CHILD_LIMIT;
            // GTAP_MAX_CHILD_TASKS: the run's limit (config.max_child_tasks, <= the table's bound)
            if (p.max_child && o.nchild > p.max_child) o.err = GTAP_E_CHILD_LIMIT;
        }
        if constexpr (assist_of<T>::value) {
            // (2b) warp assist: lanes whose body deferred a heavy leaf routine get the whole warp,
            // one request at a time (a B200 choice; the task graph and
            // the result are unchanged). One fence + warp sync after the requests, so the
            // requesting lanes' join releases below cover every lane's stores.
            uint32_t req = __ballot_sync(0xffffffffu, my != kNone && o.assist != 0u && o.err == 0u);
            const bool any_assist = req != 0u;
#ifndef GTAP_ASSIST_PUBLISH
#define GTAP_ASSIST_PUBLISH 2   // 0 (off) / 2 / 8: mergesort 2^24 1.310 / 1.281 / 1.285 ms; Cilksort 5.07 -> 4.27 ms
#endif
            if (GTAP_ASSIST_PUBLISH && (uint32_t)__popc(req) >= (uint32_t)GTAP_ASSIST_PUBLISH) {
                // a long assist phase (several warp-wide bodies back to back): publish the private parts first,
                // so that idle warps can steal those tasks meanwhile instead of waiting for this cycle to end
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const uint32_t priv = tail[q] - split[q];
                    if (priv && lane == 0) red_add_release(&p.dq[dq0 + q].S, (unsigned long long)priv << 32);
                    split[q] = tail[q];
                }
            }
            while (req) {
                const uint32_t src = (uint32_t)__ffs(req) - 1u;
                req &= req - 1u;
                uint32_t ap[kDataWords];
#pragma unroll
                for (int k = 0; k < kDataWords; ++k) ap[k] = __shfl_sync(0xffffffffu, o.ap[k], src);
                const bool aok = T::assist(args, ap, lane, bx);
                const uint32_t okm = __ballot_sync(0xffffffffu, aok);
                if (lane == src && okm != 0xffffffffu) o.err = GTAP_E_BAD_STATE;
                if (lane == 0) stat(kStAssist, 1);
            }
            if (any_assist) {
                __threadfence();
                __syncwarp();
            }
        }
        __syncwarp();
        uint32_t err = o.err;

        // ================= (3a) free + allocate =================
        const bool fin = (o.action == Out::kFinish);
        const uint32_t fball = __ballot_sync(0xffffffffu, fin);
        const uint32_t F = __popc(fball);
        if (fin) sm.fbuf[__popc(fball & lt)] = my;
        GTAP_CK(if (fin) ck_free(p, my); __syncwarp());
        const uint32_t nc = (err == 0u) ? o.nchild : 0u;
        // exclusive prefix of the child counts: one ballot per bit of nc (nc <= MAXC)
        uint32_t excl = 0, T_total = 0;
#pragma unroll
        for (int bit = 0; (1 << bit) <= MAXC; ++bit) {
            const uint32_t bb = __ballot_sync(0xffffffffu, (nc >> bit) & 1u);
            excl += (uint32_t)__popc(bb & lt) << bit;
            T_total += (uint32_t)__popc(bb) << bit;
        }
        const uint32_t fromF = min(F, T_total);
        uint32_t need = T_total - fromF;
        uint32_t fromRing = 0;
        // own stack first (most recently freed on top)
        uint32_t abase = 0;
        if (FS > 0 && need > 0u && fsp > 0u) {
            abase = min(need, fsp);
            for (uint32_t i = lane; i < abase; i += 32u) sm.abuf[i] = sm.fstack[fsp - 1u - i];
            fsp -= abase;
            need -= abase;
        }
        while (need > 0u) {  // drain the own free ring, 32 entries per round
            const uint32_t want = min(need, 32u);
            uint32_t e = 0;
            if (lane < want) e = ld_relaxed(&myfring[(fhead + lane) & mmask]);
            const uint32_t valid = __ballot_sync(0xffffffffu, e != 0u);
            const uint32_t k = min((uint32_t)(__ffs(~valid) - 1), want);  // contiguous prefix
            if (lane < k) {
                sm.abuf[abase + fromRing + lane] = e - 1u;
                st_relaxed(&myfring[(fhead + lane) & mmask], 0u);
            }
            fhead += k;
            fromRing += k;
            need -= k;
            if (k < want) break;
        }
        if (need > 0u) {
            if (bump + need > M) {
                if (lane == 0) raise_error(p.ctl, GTAP_E_POOL_EXHAUSTED);
                failed = true;
            } else {
                for (uint32_t i = lane; i < need; i += 32) sm.abuf[abase + fromRing + i] = base_id + bump + i;
                bump += need;
            }
        }
        __syncwarp();
        if (failed) break;
        if (lane == 0) stat(kStTasks, T_total);

        // ================= (3b) spawn: write child records =================
        uint32_t cid[MAXC];
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
            cid[c] = kNone;
            if ((uint32_t)c < nc) {
                const uint32_t g = excl + c;
                cid[c] = (g < fromF) ? sm.fbuf[g] : sm.abuf[g - fromF];
                TaskRec* cr = p.rec + cid[c];
                GTAP_CK(ck_alloc(p, cid[c]); ck_publish(p, cid[c]));
                uint32_t cfn, cq, cd[kDataWords];
                if constexpr (kGen) {
                    T::gen_child(o.gen, o.gmask, (uint32_t)c, cfn, cq, cd);
                } else {
                    cfn = o.cfn[c]; cq = o.cq[c];
                    cd[0] = o.cd[c][0]; cd[1] = o.cd[c][1]; cd[2] = o.cd[c][2]; cd[3] = o.cd[c][3];
                }
                st_v8(cr, make_uint4(0u, 0u, make_meta(cfn, 0, c, cq), T::kTaskwait ? my : kNone),
                      make_uint4(cd[0], cd[1], cd[2], cd[3]));   // the child record: one 256-bit store
                if constexpr (kGeneric) {
                    sm.cbuf[g] = cid[c] | (task_is_heavy<T>(cfn, cd) ? kHeavyBit : 0u);
                    sm.cqb[g] = (uint8_t)cq;
                }
            }
        }
        // suspend: store the resumption state and the join counter; the taskwait
        // queue(expr) rides in the top byte of the join word (EPAQ)
        uint32_t resume_id = kNone, resume_q = 0;
        if (o.action == Out::kSuspend) {
            GTAP_CK(ck_suspend(p, my, nc));
            st_v4(p.rec + my, make_uint4(nc | (o.next_queue << 24), 0u, make_meta(myfn, o.next_state, ord, 0), parent));
            if (nc == 0u) {  // empty join: runnable at once
                resume_id = my | (task_is_heavy<T>(myfn, mydata) ? kHeavyBit : 0u);
                resume_q = o.next_queue;
            }
        }
        // finish: copy the result into the parent's slot (copy-at-finish, R8)
        if (!T::kJoinReduceAdd && fin && err == 0u && parent != kNone && !is_root_link(parent) && o.has_result)
            st_relaxed(reinterpret_cast<int32_t*>(&p.rec[parent].d[2 + ord]), o.result);
        __syncwarp();

        // ================= (3c) join: last child re-enqueues the parent =================
        // the join RMW is issued here and its result consumed after the surplus-free atomics below,
        // so the two round trips overlap (the freed records are not the parent's)
        const bool jn = fin && err == 0u && parent != kNone && !is_root_link(parent);
        unsigned long long jold = 0;
        if (jn) {
            GTAP_CK(ck_join(p, parent));
            if constexpr (T::kJoinReduceAdd) {
                // one relaxed 64-bit RMW: pending -= 1 and acc += result (the count never
                // underflows, so adding 0xFFFFFFFF carries exactly once into acc: add result - 1)
                const unsigned long long inc =
                    ((unsigned long long)(uint32_t)(o.result - 1) << 32) | 0xFFFFFFFFull;
                jold = atom_add_relaxed_u64(&p.rec[parent], inc);
            } else {
                jold = (uint32_t)atom_add_acq_rel(&p.rec[parent].pending, -1);
            }
        }
        // surplus freed records go back to their home worker's free ring
        if (F > T_total) {
            bool mine_free = lane < F - T_total;
            uint32_t fid = mine_free ? sm.fbuf[T_total + lane] : 0u;
            const bool remote = mine_free && (fid >> p.logM) != w;
            if (FS > 0) {   // own records onto the own stack while it has room
                const uint32_t ob = __ballot_sync(0xffffffffu, mine_free && !remote);
                const uint32_t room = (uint32_t)FS - fsp;
                const uint32_t rk = (uint32_t)__popc(ob & lt);
                if (mine_free && !remote && rk < room) {
                    sm.fstack[fsp + rk] = fid;
                    mine_free = false;
                }
                fsp += min((uint32_t)__popc(ob), room);
            }
            const uint32_t mask = __ballot_sync(0xffffffffu, mine_free);
            if (mine_free) {
                const uint32_t home = fid >> p.logM;
                const uint32_t grp = __match_any_sync(mask, home);
                const uint32_t leader = __ffs(grp) - 1u;
                uint32_t base = 0;
                if (lane == leader) base = atom_add_relaxed(&p.fm[home].tail, (uint32_t)__popc(grp));
                base = __shfl_sync(grp, base, leader);
                const uint32_t slot = base + __popc(grp & lt);
                st_relaxed(&p.fring[((size_t)home << p.logM) + (slot & mmask)], fid + 1u);
            }
            const uint32_t rf = __ballot_sync(0xffffffffu, remote);
            if (lane == 0) stat(kStRfree, (uint32_t)__popc(rf));
        }
        __syncwarp();
        if (fin && err == 0u) {
            if (jn) {
                const uint32_t pend_old = (uint32_t)jold;
                const bool last = (pend_old & kPendMask) == 1u;
                if constexpr (T::kJoinReduceAdd) {
                    if (last) {  // the continuation reads the sum as load_result(0) + load_result(1)
                        const uint32_t sum = (uint32_t)(jold >> 32) + (uint32_t)o.result;
                        st_v2(&p.rec[parent].d[2], sum, 0u);
                    }
                }
                if (last) {
                    resume_id = parent | (parent_is_heavy<T>(myfn, mydata) ? kHeavyBit : 0u);
                    resume_q = pend_old >> 24;
                }
            } else if (is_root_link(parent)) {
                const uint32_t r = parent & ~kRootFlag;
                p.root_results[r] = o.has_result ? (long long)o.result : 0ll;
                if (T::kTaskwait) {
                    if (atom_add_acq_rel(&p.ctl->roots_left, 0xFFFFFFFFu) == 1u) st_release(&p.ctl->done, 1u);
                }
            }
        }
        GTAP_CK(if (resume_id != kNone) ck_publish(p, resume_id & ~kHeavyBit));
        {
            const uint32_t eb = __ballot_sync(0xffffffffu, err != 0u);
            if (eb && lane == (uint32_t)__ffs(eb) - 1u) raise_error(p.ctl, err);
        }
        if (!T::kTaskwait) {
            // outstanding-task counter (SPEC S:321 reading): +children -finished, one atomic per warp-cycle
            const long long delta = (long long)T_total - (long long)F;
            if (lane == 0 && delta != 0) {
                const long long old = atom_add_acq_rel(&p.ctl->outstanding, delta);
                if (old + delta == 0) st_release(&p.ctl->done, 1u);
            }
        }

        // ================= (3d) distribute: keep <= 32, push the rest =================
        const uint32_t rball = __ballot_sync(0xffffffffu, resume_id != kNone);
        const uint32_t P = __popc(rball);
        const uint32_t R = P + T_total;
        uint32_t keep = 0, pushc = 0;
        uint32_t pushq[NQ];      // pushed per queue (uniform)
        uint32_t heavy_q = 0;    // bit q: a heavy task was pushed to queue q
#pragma unroll
        for (int i = 0; i < NQ; ++i) pushq[i] = 0;
        if constexpr (!kGeneric) {
            // runnable list = [resumed parents in lane order, children in spawn order]; the first 32
            // are kept, entry e >= 32 goes to ring slot tail + e - 32: every lane places its own
            keep = min(R, 32u);
            pushc = R - keep;
            pushq[0] = pushc;
            if (pushc && tail[0] + pushc - sdone[0] > Q) {
                if (lane == 0) sdone[0] = ld_acquire(&p.dq[dq0].steal_done);
                sdone[0] = __shfl_sync(0xffffffffu, sdone[0], 0);
                __syncwarp();  // lane 0's acquire orders every lane's ring overwrites after the thieves' reads
                if (tail[0] + pushc - sdone[0] > Q) {
                    if (lane == 0) raise_error(p.ctl, GTAP_E_QUEUE_OVERFLOW);
                    break;
                }
            }
            uint32_t* ring0 = p.ring + (size_t)dq0 * Q;
            if (resume_id != kNone) sm.kept[__popc(rball & lt)] = resume_id;
#pragma unroll
            for (int c = 0; c < MAXC; ++c) {
                if ((uint32_t)c < nc) {
                    const uint32_t e = P + excl + c;
                    if (e < 32u) sm.kept[e] = cid[c];
                    else ring0[(tail[0] + (e - 32u)) & qmask] = cid[c];
                }
            }
        } else {
            // generic placement (heavy hints and/or EPAQ): the kept set holds up to 32 light tasks of
            // ONE queue class in list order (resumed parents first, then children); every
            // other task goes to the tail of its own queue
            if (resume_id != kNone) {
                sm.pbuf[__popc(rball & lt)] = resume_id;
                sm.pqb[__popc(rball & lt)] = (uint8_t)resume_q;
            }
            __syncwarp();
            // EPAQ: the class of the next cycle is the next queue in round-robin order;
            // the kept set holds this cycle's new tasks of that class, so every class -- including
            // continuations, which free records -- is visited every NQ cycles
            uint32_t qk = NQ > 1 ? (qc + 1u) % (uint32_t)NQ : 0u;
            if (NQ > 1 && (p.policy & kPolQueueStay)) {
                // P:177-178 read literally: stay on the class in use while this cycle produced runnable tasks
                // of it, else the next class (round robin from it) that did
                uint32_t has = 0;
                for (uint32_t base = 0; base < R; base += 32) {
                    const uint32_t i = base + lane;
                    uint32_t id = kNone, qi = 0;
                    if (i < R) {
                        id = (i < P) ? sm.pbuf[i] : sm.cbuf[i - P];
                        qi = (i < P) ? sm.pqb[i] : sm.cqb[i - P];
                    }
                    has |= __reduce_or_sync(0xffffffffu, (i < R && !(id & kHeavyBit)) ? 1u << qi : 0u);
                }
                qk = qc;
#pragma unroll
                for (int k = 0; k < NQ; ++k) {
                    const uint32_t q = (qc + (uint32_t)k) % (uint32_t)NQ;
                    if ((has >> q) & 1u) { qk = q; break; }
                }
            }
            // pass 1: count pushes per queue (capacity check before any ring write)
            for (uint32_t base = 0; base < R; base += 32) {
                const uint32_t i = base + lane;
                uint32_t id = kNone, qi = 0;
                if (i < R) {
                    id = (i < P) ? sm.pbuf[i] : sm.cbuf[i - P];
                    qi = NQ > 1 ? ((i < P) ? sm.pqb[i] : sm.cqb[i - P]) : 0u;
                }
                const bool hv = (i < R) && (id & kHeavyBit);
                const bool cand = (i < R) && !hv && qi == qk;
                const uint32_t cb = __ballot_sync(0xffffffffu, cand);
                const bool k = cand && (keep + __popc(cb & lt)) < 32u;
                keep += min(__popc(cb), 32u - min(keep, 32u));
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const uint32_t pb = __ballot_sync(0xffffffffu, i < R && !k && qi == (uint32_t)q);
                    pushq[q] += __popc(pb);
                    if (__ballot_sync(0xffffffffu, i < R && !k && hv && qi == (uint32_t)q)) heavy_q |= 1u << q;
                }
            }
            bool overflow = false;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                if (pushq[q] && tail[q] + pushq[q] - sdone[q] > Q) {
                    if (lane == 0) sdone[q] = ld_acquire(&p.dq[dq0 + q].steal_done);
                    sdone[q] = __shfl_sync(0xffffffffu, sdone[q], 0);
                    __syncwarp();  // lane 0's acquire orders every lane's ring overwrites after the thieves' reads
                    if (tail[q] + pushq[q] - sdone[q] > Q) overflow = true;
                }
            }
            if (overflow) {
                if (lane == 0) raise_error(p.ctl, GTAP_E_QUEUE_OVERFLOW);
                break;
            }
            // pass 2: place
            uint32_t kk = 0;
            uint32_t pc[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) pc[q] = 0;
            for (uint32_t base = 0; base < R; base += 32) {
                const uint32_t i = base + lane;
                uint32_t id = kNone, qi = 0;
                if (i < R) {
                    id = (i < P) ? sm.pbuf[i] : sm.cbuf[i - P];
                    qi = NQ > 1 ? ((i < P) ? sm.pqb[i] : sm.cqb[i - P]) : 0u;
                }
                const bool hv = (i < R) && (id & kHeavyBit);
                const bool cand = (i < R) && !hv && qi == qk;
                const uint32_t cb = __ballot_sync(0xffffffffu, cand);
                const uint32_t rank = kk + __popc(cb & lt);
                const bool k = cand && rank < 32u;
                if (k) sm.kept[rank] = id;
                kk += min(__popc(cb), 32u - min(kk, 32u));
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const uint32_t pb = __ballot_sync(0xffffffffu, i < R && !k && qi == (uint32_t)q);
                    if (i < R && !k && qi == (uint32_t)q) {
                        uint32_t* ringq = p.ring + (size_t)(dq0 + q) * Q;
                        ringq[(tail[q] + pc[q] + __popc(pb & lt)) & qmask] = id & ~kHeavyBit;
                    }
                    pc[q] += __popc(pb);
                }
            }
            pushc = 0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) pushc += pushq[q];
            qc = qk;  // next cycle runs the kept class (or pops from it first)
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < NQ; ++q) tail[q] += pushq[q];
        nkept = keep;
        if (lane == 0) stat(kStPush, pushc);
        // publish the oldest half of a private part when thieves drained its public part,
        // or all of it when heavy tasks were just pushed there
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const unsigned long long sq = __shfl_sync(0xffffffffu, S_lane, q);
            if (lane == 0) {
                const uint32_t h = (uint32_t)sq;
                const uint32_t priv = tail[q] - split[q];
                const bool hvq = (heavy_q >> q) & 1u;
                if ((hvq && priv) || (h == split[q] && priv >= 2u)) {
                    const uint32_t k = hvq ? priv : (priv >> 1);
                    split[q] += k;
                    red_add_release(&p.dq[dq0 + q].S, (unsigned long long)k << 32);
                }
                if (q == 0) pub_hint = split[0] - h;
            }
            split[q] = __shfl_sync(0xffffffffu, split[q], 0);
            if (q == 0) pub_hint = __shfl_sync(0xffffffffu, pub_hint, 0);
        }
        __syncwarp();
        if (done_seen) break;  // error raised elsewhere (completion implies no tasks left)
        if ((cyc_u & 4095u) == 0u && wd_on) {
            uint32_t tmo = 0;
            if (lane == 0 && globaltimer() - t0 > p.watchdog_ns) { raise_error(p.ctl, GTAP_E_TIMEOUT); tmo = 1; }
            if (__shfl_sync(0xffffffffu, tmo, 0)) break;
        }
    }

    // ---- exit: fold per-warp counters into the control block
    if (lane == 0) {
        stflush();
        unsigned long long* s = p.ctl->stats;
        atomicAdd(&s[ST_TASKS], stget(kStTasks));
        atomicAdd(&s[ST_INVOC], stget(kStInv));
        atomicAdd(&s[ST_POPS], stget(kStPops));
        atomicAdd(&s[ST_KEPT], stget(kStKept));
        atomicAdd(&s[ST_STEALS_OK], stget(kStSok));
        atomicAdd(&s[ST_STEALS_FAILED], stget(kStSfail));
        atomicAdd(&s[ST_STOLEN], stget(kStStolen));
        atomicAdd(&s[ST_PUSHES], stget(kStPush));
        atomicAdd(&s[ST_CYCLES], stget(kStCyc));
        atomicAdd(&s[ST_IDLE], stget(kStIdle));
        atomicAdd(&s[ST_REMOTE_FREES], stget(kStRfree));
        if (stget(kStAssist)) atomicAdd(&s[ST_ASSISTS], stget(kStAssist));
        atomicMax(&s[ST_MAX_POOL], (unsigned long long)bump);
    }
}

}  // namespace gtap
