// sched_block.cuh -- block-level persistent scheduler ("block-cooperative"
// mode, §4.1; deque §4.3.1; API §5.1.3).
//
// One worker = one thread block. Warp 0 is the queue leader ("a
// designated leader thread performs queue operations, and each pop/steal
// retrieves at most one task"): it takes the kept task or pops one task from
// the block's own deque, else steals one (probing 32 random victims in
// parallel, one per lane), and broadcasts the record through shared memory.
// All threads then run the task body data-parallel (threadIdx/blockDim,
// __syncthreads, shared memory: P:1081-1082). Spawns made by individual
// threads ("performed by the thread that reaches the pragma") are
// staged in shared memory (reading R13) and published by warp 0 after the
// body, or mid-body through flush() for tables without taskwait.
//
// The deque is the same split ring as the thread-level one (DESIGN.md
// "Deque") with claims of exactly one task, i.e. a fixed-capacity Chase-Lev
// deque whose owner end is private until published.
#pragma once
#include "gtap.h"
#include "gtap_internal.cuh"

namespace gtap {

// Batch pop (B200 choice): a leader that pops from its private part takes up to
// T::kPopBatch tasks (at most half of the private part, so publication still has work to hand to
// thieves) and loads their records with one lane each -- one ring round trip and one record round
// trip per batch instead of per task; the block then runs them one at a time in LIFO order, as
// single pops would. Tables without kPopBatch pop one task at a time (measured: SpMV and the
// block-level trees are slower with batches, BFS faster with 4).
// keep the newest child for the block's next task (default) or push every child (kKeepChild = false)
template <class T, class = void>
struct keep_child_of { static constexpr bool value = true; };
template <class T>
struct keep_child_of<T, decltype((void)T::kKeepChild, void())> { static constexpr bool value = T::kKeepChild; };

template <class T, class = void>
struct pop_oldest_of { static constexpr bool value = false; };
template <class T>
struct pop_oldest_of<T, decltype((void)T::kPopOldest, void())> { static constexpr bool value = T::kPopOldest; };

template <class T, class = void>
struct pop_batch_of { static constexpr int value = 0; };
template <class T>
struct pop_batch_of<T, decltype((void)T::kPopBatch, void())> { static constexpr int value = T::kPopBatch; };

// depth of the block's shared-memory free stack (default 256; small blocks packed 32 per SM need less smem)
template <class T, class = void>
struct bfstack_of { static constexpr uint32_t value = 256; };
template <class T>
struct bfstack_of<T, decltype((void)T::kBlockFreeStack, void())> { static constexpr uint32_t value = T::kBlockFreeStack; };

// multi-task cycles (tables without taskwait): a cycle runs up to kMultiTask tasks of a popped batch at once,
// T::exec_multi (e.g. BFS on one-warp blocks: groups of lanes expand several small vertices side by side)
template <class T, class = void>
struct multi_task_of { static constexpr int value = 1; };
template <class T>
struct multi_task_of<T, decltype((void)T::kMultiTask, void())> { static constexpr int value = T::kMultiTask; };

struct ChildSpec {
    uint32_t fn;
    uint32_t d[kDataWords];
};

template <class T>
struct BlockSmem {
    // task of a cycle (kNone: none, kExit: leave), double-buffered by cycle parity: warp 0 writes the next
    // cycle's word while the other warps may still read this cycle's (an idle cycle has no second barrier)
    uint32_t task_id[2];
    uint32_t fn, state, parent, ord;
    uint32_t d[kDataWords];
    uint32_t nspawn;          // staged children (smem atomic)
    uint32_t action;          // 1 finish, 2 suspend
    uint32_t next_state;
    uint32_t has_result;
    int32_t result;
    uint32_t err;
    ChildSpec spawns[T::kSpawnCap];
    typename T::Scratch scratch;
    // records of this block's own pool freed here, reused first (no global atomics)
    uint32_t fstack[bfstack_of<T>::value];
    uint32_t nfree;
    // the kept child is dispatched from its staged spec (no record reload)
    ChildSpec kept_spec;
    uint32_t kept_parent, kept_ord, kept_fresh;
    // batch pop: up to kPopBatch tasks taken from the private part at once, records loaded in parallel
    uint4 bq_h[pop_batch_of<T>::value > 0 ? pop_batch_of<T>::value : 1];
    uint4 bq_d[pop_batch_of<T>::value > 0 ? pop_batch_of<T>::value : 1];
    uint32_t bq_id[pop_batch_of<T>::value > 0 ? pop_batch_of<T>::value : 1];
    // multi-task cycle: the cycle's tasks (mt_n of them; task 0 is also in fn/state/d above)
    uint32_t mt_n;
    uint32_t mt_fn[multi_task_of<T>::value];   // fn | state << 8
    uint32_t mt_id[multi_task_of<T>::value];
    uint32_t mt_d[multi_task_of<T>::value][kDataWords];
};

// Leader-side (warp 0) persistent state.
struct BLeader {
    uint32_t tail, split, sdone, bump, fhead, kept, rng, backoff;
    uint32_t bq_n, bq_i;           // batch-popped tasks held in smem, next to run
    uint32_t local_dec;            // finished no-taskwait tasks not yet subtracted from ctl->outstanding
    unsigned long long S_pref;     // own deque word, loaded at acquire time, used at finalize
    unsigned long long st[ST_COUNT];
};

template <class T>
struct BCtx;
template <class T>
__device__ void block_flush(BlockSmem<T>& sm, const KParams& p, BLeader& L, uint32_t w, uint32_t headroom);

template <class T>
struct BCtx {
    BlockSmem<T>& sm;
    const KParams& p;
    BLeader& L;
    uint32_t w;
    __device__ __forceinline__ BCtx(BlockSmem<T>& s, const KParams& pp, BLeader& l, uint32_t ww)
        : sm(s), p(pp), L(l), w(ww) {}
    // uniform: publish staged spawns if fewer than `headroom` staging slots remain (no-taskwait tables only)
    __device__ __forceinline__ void flush(uint32_t headroom) { block_flush<T>(sm, p, L, w, headroom); }
    // called by any subset of threads (the ones that reach the spawn)
    __device__ __forceinline__ void spawn(uint32_t fn, uint32_t d0, uint32_t d1 = 0, uint32_t d2 = 0, uint32_t d3 = 0) {
        const uint32_t i = atomicAdd(&sm.nspawn, 1u);
        if (i < (uint32_t)T::kSpawnCap) {
            ChildSpec& c = sm.spawns[i];
            c.fn = fn; c.d[0] = d0; c.d[1] = d1; c.d[2] = d2; c.d[3] = d3;
        } else {
            atomicCAS(&sm.err, 0u, (uint32_t)GTAP_E_CHILD_LIMIT);
        }
    }
    // single-thread (thread 0) or uniform calls
    __device__ __forceinline__ void finish(int32_t r) { sm.action = 1; sm.has_result = 1; sm.result = r; }
    __device__ __forceinline__ void finish_void() { sm.action = 1; }
    __device__ __forceinline__ void suspend(uint32_t next) { sm.action = 2; sm.next_state = next; }
    __device__ __forceinline__ void bad_state() { sm.action = 1; sm.err = GTAP_E_BAD_STATE; }
};

// warp 0: draw `cnt` (<= 32) record IDs from the own pool into out[] (lane i gets out[i]).
// Returns false (and raises) on exhaustion.
template <class SM>
__device__ __forceinline__ bool block_alloc(const KParams& p, BLeader& L, SM& sm, uint32_t w, uint32_t lane,
                                            uint32_t cnt, uint32_t& id_out) {
    using namespace dev;
    const uint32_t M = 1u << p.logM, mmask = M - 1u;
    // 1) this block's shared-memory free stack
    const uint32_t nf = sm.nfree;
    const uint32_t fs = min(nf, cnt);
    if (lane < fs) id_out = sm.fstack[nf - 1u - lane];
    __syncwarp();
    if (lane == 0) sm.nfree = nf - fs;
    if (fs == cnt) { __syncwarp(); return true; }
    // 2) the own free ring (records freed by other blocks)
    uint32_t* myfring = p.fring + ((size_t)w << p.logM);
    const uint32_t want = cnt - fs;
    uint32_t e = 0;
    if (lane < want) e = ld_relaxed(&myfring[(L.fhead + lane) & mmask]);
    const uint32_t valid = __ballot_sync(0xffffffffu, e != 0u);
    const uint32_t k = min((uint32_t)(__ffs(~valid) - 1), want);
    if (lane < k) st_relaxed(&myfring[(L.fhead + lane) & mmask], 0u);
    const uint32_t src = lane - fs;  // lane fs + i takes ring entry i
    const uint32_t er = __shfl_sync(0xffffffffu, e, src & 31u);
    if (lane >= fs && lane < fs + k) id_out = er - 1u;
    L.fhead += k;
    const uint32_t rest = want - k;
    if (rest) {
        if (L.bump + rest > M) {
            if (lane == 0) raise_error(p.ctl, GTAP_E_POOL_EXHAUSTED);
            return false;
        }
        if (lane >= fs + k && lane < cnt) id_out = (w << p.logM) + L.bump + (lane - fs - k);
        L.bump += rest;
    }
    __syncwarp();
    return true;
}

// warp 0, lane 0: free one record -- to the block's smem stack when it is ours, else to its
// home block's free ring.
template <class SM>
__device__ __forceinline__ void block_free1(const KParams& p, SM& sm, uint32_t w, uint32_t id) {
    using namespace dev;
    if ((id >> p.logM) == w && sm.nfree < (uint32_t)(sizeof(sm.fstack) / sizeof(sm.fstack[0]))) {
        sm.fstack[sm.nfree++] = id;
        return;
    }
    const uint32_t home = id >> p.logM;
    const uint32_t slot = atom_add_relaxed(&p.fm[home].tail, 1u);
    st_relaxed(&p.fring[((size_t)home << p.logM) + (slot & ((1u << p.logM) - 1u))], id + 1u);
}

// warp 0: free record `id` (lane-predicated `doit`) to its home free ring.
__device__ __forceinline__ void block_free(const KParams& p, uint32_t lane, bool doit, uint32_t id) {
    using namespace dev;
    const uint32_t mask = __ballot_sync(0xffffffffu, doit);
    if (!doit) return;
    const uint32_t home = id >> p.logM;
    const uint32_t grp = __match_any_sync(mask, home);
    const uint32_t leader = __ffs(grp) - 1u;
    uint32_t base = 0;
    if (lane == leader) base = atom_add_relaxed(&p.fm[home].tail, (uint32_t)__popc(grp));
    base = __shfl_sync(grp, base, leader);
    const uint32_t slot = base + __popc(grp & lanemask_lt());
    st_relaxed(&p.fring[((size_t)home << p.logM) + (slot & ((1u << p.logM) - 1u))], id + 1u);
}

// warp 0: move staged children [0, cnt) into records and onto the deque.
// keep_last: keep the newest child for the next cycle instead of pushing it.
template <class T>
__device__ bool block_publish_spawns(const KParams& p, BLeader& L, BlockSmem<T>& sm, uint32_t w, uint32_t lane,
                                     uint32_t cnt, uint32_t parent_id, bool keep_last, bool count_outstanding) {
    using namespace dev;
    const uint32_t Q = p.qmask + 1u;
    uint32_t* ring = p.ring + (size_t)w * Q;
    if (cnt == 0) return true;
    if (!T::kTaskwait && count_outstanding) {
        // outstanding += children before any of them can be published (termination, R6); the
        // publication's release orders this relaxed add before any thief can run a child
        if (lane == 0) red_add_relaxed(reinterpret_cast<unsigned long long*>(&p.ctl->outstanding), cnt);
    }
    uint32_t pushc = keep_last ? cnt - 1u : cnt;
    if (pushc && L.tail + pushc - L.sdone > Q) {
        if (lane == 0) L.sdone = ld_acquire(&p.dq[w].steal_done);
        L.sdone = __shfl_sync(0xffffffffu, L.sdone, 0);
        __syncwarp();  // lane 0's acquire orders every lane's ring overwrites after the thieves' reads
        if (L.tail + pushc - L.sdone > Q) {
            if (lane == 0) raise_error(p.ctl, GTAP_E_QUEUE_OVERFLOW);
            return false;
        }
    }
    for (uint32_t b = 0; b < cnt; b += 32) {
        const uint32_t c = min(32u, cnt - b);
        uint32_t id = kNone;
        if (!block_alloc(p, L, sm, w, lane, c, id)) return false;
        if (lane < c) {
            const ChildSpec cs = sm.spawns[b + lane];
            TaskRec* r = p.rec + id;
            GTAP_CK(ck_alloc(p, id); ck_publish(p, id));
            st_v8(r, make_uint4(0u, 0u, make_meta(cs.fn, 0, b + lane, 0), parent_id),
                  make_uint4(cs.d[0], cs.d[1], cs.d[2], cs.d[3]));   // one 256-bit store per child record
            const uint32_t i = b + lane;
            if (keep_last && i == cnt - 1u) {  // lane-local; broadcast below
                L.kept = id;
                sm.kept_spec = cs;
                sm.kept_parent = parent_id;
                sm.kept_ord = i;
                sm.kept_fresh = 1u;
            } else {
                ring[(L.tail + i) & p.qmask] = id;
            }
        }
        if (keep_last && cnt - 1u >= b && cnt - 1u < b + c) {
            L.kept = __shfl_sync(0xffffffffu, L.kept, (cnt - 1u) - b);
        }
    }
    L.tail += pushc;
    if (lane == 0) L.st[ST_TASKS] += cnt, L.st[ST_PUSHES] += pushc;
    return true;
}

// warp 0: publish half of the private part if thieves drained the public part.
__device__ __forceinline__ void block_maybe_publish(const KParams& p, BLeader& L, uint32_t w, uint32_t lane,
                                                    bool use_pref = false) {
    using namespace dev;
    if (lane == 0) {
        const unsigned long long s = use_pref ? L.S_pref : ld_relaxed(&p.dq[w].S);
        const uint32_t priv = L.tail - L.split;
        if ((uint32_t)s == L.split && priv >= 2u) {
            const uint32_t k = priv >> 1;
            L.split += k;
            red_add_release(&p.dq[w].S, (unsigned long long)k << 32);
        }
    }
    L.split = __shfl_sync(0xffffffffu, L.split, 0);
}

template <class T>
__global__ void __launch_bounds__(T::kMaxThreads, T::kMinBlocks) block_sched_kernel(KParams p, typename T::Args args) {
    using namespace dev;
    __shared__ BlockSmem<T> sm;
    constexpr int kPB = pop_batch_of<T>::value;
    static_assert(kPB <= 32, "one lane per batched pop");
    constexpr int kMT = multi_task_of<T>::value;
    static_assert(kMT == 1 || (!T::kTaskwait && kPB >= kMT), "multi-task cycles: tables without taskwait, batch pops");
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t w = blockIdx.x;
    if (w >= p.W) return;
    const uint32_t Q = p.qmask + 1u, qmask = p.qmask;
    uint32_t* ring = p.ring + (size_t)w * Q;
    DequeMeta* mydq = p.dq + w;
    BLeader L;
    BCtx<T> ctx(sm, p, L, w);
    const unsigned long long t0 = globaltimer();

    if (warp == 0) {
        L.tail = L.split = L.sdone = L.bump = L.fhead = 0;
        L.local_dec = 0;
        L.S_pref = 0;
        L.kept = kNone;
        L.bq_n = L.bq_i = 0;
        L.backoff = 64;
        L.rng = hash32(p.seed * 0x9E3779B97F4A7C15ull + (unsigned long long)w * 32u + lane);
#pragma unroll
        for (int i = 0; i < ST_COUNT; ++i) L.st[i] = 0;
        // entry: roots w, w + W, ... onto this block's deque
        uint32_t mine = p.nroots > w ? (p.nroots - w + p.W - 1) / p.W : 0;
        if (mine > (1u << p.logM) || mine > Q) {
            if (lane == 0) raise_error(p.ctl, GTAP_E_POOL_EXHAUSTED);
            mine = 0;
        }
        for (uint32_t i = lane; i < mine; i += 32) {
            const uint32_t r = w + i * p.W;
            const RootSpec rs = p.roots[r];
            const uint32_t id = (w << p.logM) + i;
            TaskRec* rec = p.rec + id;
            st_v4(rec, make_uint4(0u, 0u, make_meta(rs.fn, 0, 0, 0), kRootFlag | r));
            st_v4(&rec->d[0], make_uint4(rs.d[0], rs.d[1], rs.d[2], rs.d[3]));
            GTAP_CK(ck_alloc(p, id); ck_publish(p, id));
            ring[i & qmask] = id;
        }
        L.bump = mine;
        L.tail = mine;
        if (lane == 0) L.st[ST_TASKS] += mine;
        __syncwarp();
    }
    if (tid == 0) { sm.nfree = 0; sm.kept_fresh = 0; }
    uint32_t par = 0;   // cycle parity (every thread passes the acquire barrier once per cycle)
    __syncthreads();

    while (true) {
        // ================= warp 0: acquire one task =================
        if (warp == 0) {
            uint32_t id = kNone;
            bool from_spec = false;
            int32_t from_bq = -1;   // slot of a batch-popped task
            if (L.kept != kNone) {
                id = L.kept;
                L.kept = kNone;
                from_spec = sm.kept_fresh != 0u;
                if (lane == 0) ++L.st[ST_KEPT];
            } else if (kPB > 0 && L.bq_i < L.bq_n) {   // next task of the popped batch
                from_bq = (int32_t)L.bq_i;
                id = sm.bq_id[L.bq_i];
                ++L.bq_i;
            } else if (kPB > 1 && L.tail - L.split >= 2u) {   // batch pop, private part
                const uint32_t c = min((uint32_t)kPB, (L.tail - L.split) >> 1);
                if (lane < c) {
                    uint32_t bid;
                    if constexpr (pop_oldest_of<T>::value) {
                        // the c OLDEST private tasks (bottom of the private part); the c newest move into
                        // their slots (c <= half the private part: no overlap; thieves never read past split)
                        bid = ld_relaxed(&ring[(L.split + lane) & qmask]);
                        const uint32_t top = ld_relaxed(&ring[(L.tail - 1u - lane) & qmask]);
                        ring[(L.split + lane) & qmask] = top;
                    } else {
                        bid = ld_relaxed(&ring[(L.tail - 1u - lane) & qmask]);
                    }
                    sm.bq_id[lane] = bid;
                    uint4 bh, bd4;
                    ld_relaxed_v8(p.rec + bid, bh, bd4);   // one 256-bit request per record
                    sm.bq_h[lane] = bh;
                    sm.bq_d[lane] = bd4;
                }
                __syncwarp();
                L.tail -= c;
                L.bq_n = c;
                L.bq_i = 1;
                from_bq = 0;
                id = sm.bq_id[0];
                if (lane == 0) L.st[ST_POPS] += c;
            } else if (L.tail != L.split) {  // LIFO pop, private part
                L.tail -= 1u;
                if (lane == 0) id = ld_relaxed(&ring[L.tail & qmask]);
                id = __shfl_sync(0xffffffffu, id, 0);
                if (lane == 0) ++L.st[ST_POPS];
            } else {
                // reclaim one from the own public part
                uint32_t got = kNone;
                if (lane == 0) {
                    unsigned long long s = ld_relaxed(&mydq->S);
                    for (int it = 0; it < 8; ++it) {
                        const uint32_t h = (uint32_t)s, sp = (uint32_t)(s >> 32);
                        if (sp == h || sp - h > Q) break;
                        const unsigned long long nw = ((unsigned long long)(sp - 1u) << 32) | h;
                        const unsigned long long o = atom_cas_relaxed(&mydq->S, s, nw);
                        if (o == s) { got = ld_relaxed(&ring[(sp - 1u) & qmask]); L.split = sp - 1u; break; }
                        s = o;
                    }
                }
                L.split = __shfl_sync(0xffffffffu, L.split, 0);
                L.tail = L.split;
                id = __shfl_sync(0xffffffffu, got, 0);
                if (id != kNone && lane == 0) ++L.st[ST_POPS];
                // steal one from the fullest of 32 random victims
                const uint32_t rounds = L.backoff >= 4096u ? 1u : p.steal_rounds;
                for (uint32_t round = 0; id == kNone && round < rounds && p.W > 1; ++round) {
                    const uint32_t v = pick_victim(p.W, w, lane, xorshift32(L.rng), p.ctl, p.policy);
                    const unsigned long long sv = ld_relaxed(&p.dq[v].S);
                    uint32_t avail = (uint32_t)(sv >> 32) - (uint32_t)sv;
                    if (avail > Q) avail = 0;
                    uint32_t best = (min(avail, (1u << 26)) << 5) | lane;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
                    if ((best >> 5) == 0) { if (lane == 0) ++L.st[ST_STEALS_FAILED]; continue; }
                    const uint32_t victim = __shfl_sync(0xffffffffu, v, best & 31u);
                    DequeMeta* vdq = p.dq + victim;
                    // claim c tasks from the head: 1 or, with steal_max > 1, up to half of a
                    // public part of >= 2 (the thief runs one and keeps c - 1 in its own deque)
                    uint32_t got = 0, h0 = 0;
                    if (lane == 0 && atom_cas_relaxed(&vdq->lock, 0u, 1u) == 0u) {
                        unsigned long long s = ld_relaxed(&vdq->S);
                        const uint32_t room = Q - (L.tail - L.sdone);  // own ring space for the extras
                        for (int it = 0; it < 8; ++it) {
                            const uint32_t h = (uint32_t)s, sp = (uint32_t)(s >> 32);
                            const uint32_t avail = sp - h;
                            if (avail == 0u || avail > Q) break;
                            const uint32_t c = min(max(1u, min(p.steal_max, avail >> 1)), room + 1u);
                            const unsigned long long nw = ((unsigned long long)sp << 32) | (uint32_t)(h + c);
                            const unsigned long long o = atom_cas_acquire(&vdq->S, s, nw);
                            if (o == s) { got = c; h0 = h; break; }
                            s = o;
                        }
                        if (got == 0u) st_relaxed(&vdq->lock, 0u);
                    }
                    got = __shfl_sync(0xffffffffu, got, 0);
                    uint32_t sidl = kNone;
                    if (got) {
                        h0 = __shfl_sync(0xffffffffu, h0, 0);
                        if (lane < got) sidl = ld_relaxed(&p.ring[(size_t)victim * Q + ((h0 + lane) & qmask)]);
                        __syncwarp();
                        if (lane == 0) {  // advance the read prefix only after loading the IDs
                            red_add_release(&vdq->steal_done, got);
                            st_relaxed(&vdq->lock, 0u);
                        }
                        if (got > 1u) {  // extras onto the own private part
                            if (lane >= 1u && lane < got) ring[(L.tail + lane - 1u) & qmask] = sidl;
                            L.tail += got - 1u;
                        }
                    }
                    id = __shfl_sync(0xffffffffu, sidl, 0);
                    if (lane == 0) { if (id != kNone) { ++L.st[ST_STEALS_OK]; L.st[ST_STOLEN] += got; } else ++L.st[ST_STEALS_FAILED]; }
                }
            }
            if (id != kNone) {
                __syncwarp();   // every lane read kept_fresh / the batch slots above before lane 0 rewrites them
                if (lane == 0) {
                    L.S_pref = ld_relaxed(&mydq->S);  // consumed at finalize (publication check)
                    if (from_spec) {  // a child this block just spawned: its record is not re-read
                        const ChildSpec cs = sm.kept_spec;
                        sm.fn = cs.fn; sm.state = 0; sm.ord = sm.kept_ord; sm.parent = sm.kept_parent;
                        sm.d[0] = cs.d[0]; sm.d[1] = cs.d[1]; sm.d[2] = cs.d[2]; sm.d[3] = cs.d[3];
                    } else if (from_bq >= 0) {   // record loaded with its batch
                        const uint4 h = sm.bq_h[from_bq];
                        const uint4 dv = sm.bq_d[from_bq];
                        sm.fn = meta_fn(h.z); sm.state = meta_state(h.z); sm.ord = meta_ord(h.z);
                        sm.parent = h.w;
                        sm.d[0] = dv.x; sm.d[1] = dv.y; sm.d[2] = dv.z; sm.d[3] = dv.w;
                    } else {
                        uint4 h, dv;
                        ld_relaxed_v8(p.rec + id, h, dv);   // one 256-bit request per record
                        sm.fn = meta_fn(h.z); sm.state = meta_state(h.z); sm.ord = meta_ord(h.z);
                        sm.parent = h.w;
                        sm.d[0] = dv.x; sm.d[1] = dv.y; sm.d[2] = dv.z; sm.d[3] = dv.w;
                    }
                    sm.kept_fresh = 0;
                    GTAP_CK(ck_dispatch(p, id, sm.state));
                    if constexpr (kMT > 1) {
                        // more tasks of the popped batch run in this cycle (one ring / record round trip for all)
                        uint32_t k = 1;
                        sm.mt_fn[0] = sm.fn | (sm.state << 8); sm.mt_id[0] = id;   // fn | state << 8
                        sm.mt_d[0][0] = sm.d[0]; sm.mt_d[0][1] = sm.d[1]; sm.mt_d[0][2] = sm.d[2]; sm.mt_d[0][3] = sm.d[3];
                        if (from_bq >= 0) {
                            while (k < (uint32_t)kMT && L.bq_i < L.bq_n) {
                                const uint32_t b = L.bq_i++;
                                const uint4 h = sm.bq_h[b];
                                const uint4 dv = sm.bq_d[b];
                                sm.mt_fn[k] = meta_fn(h.z) | (meta_state(h.z) << 8); sm.mt_id[k] = sm.bq_id[b];
                                sm.mt_d[k][0] = dv.x; sm.mt_d[k][1] = dv.y; sm.mt_d[k][2] = dv.z; sm.mt_d[k][3] = dv.w;
                                GTAP_CK(ck_dispatch(p, sm.bq_id[b], 0u));
                                ++k;
                            }
                        }
                        sm.mt_n = k;
                        L.st[ST_INVOC] += k - 1u;
                    }
                    sm.nspawn = 0; sm.action = 0; sm.has_result = 0; sm.err = 0;
                    ++L.st[ST_CYCLES];
                    ++L.st[ST_INVOC];
                }
                if constexpr (kMT > 1) L.bq_i = __shfl_sync(0xffffffffu, L.bq_i, 0);
                L.backoff = 64;
            } else {
                if (lane == 0) ++L.st[ST_IDLE];
                uint32_t d = 0;
                if (lane == 0) {
                    if (!T::kTaskwait && L.local_dec) {  // flush deferred finishes (termination, R6)
                        const long long dec = (long long)L.local_dec;
                        L.local_dec = 0;
                        if (atom_add_acq_rel(&p.ctl->outstanding, -dec) == dec) st_release(&p.ctl->done, 1u);
                    }
                    d = ld_relaxed(&p.ctl->done);
                    if (!d && p.watchdog_ns && globaltimer() - t0 > p.watchdog_ns) raise_error(p.ctl, GTAP_E_TIMEOUT);
                }
                d = __shfl_sync(0xffffffffu, d, 0);
                if (d) id = kExit;
                if (!d) {
                    nanosleep(L.backoff);
                    L.backoff = min(L.backoff * 2u, p.idle_backoff);
                }
            }
            if (lane == 0) sm.task_id[par] = id;
        }
        __syncthreads();
        const uint32_t my = sm.task_id[par];
        par ^= 1u;
        if (my == kExit) break;
        if (my == kNone) continue;

        // ================= all threads: run the task body =================
#ifdef GTAP_TRACE
        const unsigned long long tr0 = dev::globaltimer();
#endif
        if constexpr (kMT > 1) {
            T::exec_multi(args, ctx, sm.mt_n, sm.mt_fn, sm.mt_d);
        } else {
            const uint32_t d[kDataWords] = {sm.d[0], sm.d[1], sm.d[2], sm.d[3]};
            T::exec_block(args, ctx, sm.fn, sm.state, d);
        }
        __syncthreads();
#ifdef GTAP_TRACE
        if (tid == 0) trace_rec(tr0, w | (sm.state << 24), sm.d[0], sm.d[1]);
#endif

        // ================= warp 0: spawn / join / finish =================
        if (warp == 0) {
            uint32_t err = sm.err ? sm.err : (sm.action == 0 ? (uint32_t)GTAP_E_BAD_STATE : 0u);
            // GTAP_MAX_CHILD_TASKS: the run's limit on spawns per invocation (tables without taskwait
            // publish mid-body through flush(); their limit is checked per staging round)
            if (err == 0u && p.max_child && sm.nspawn > p.max_child) err = GTAP_E_CHILD_LIMIT;
            const uint32_t staged = min(sm.nspawn, (uint32_t)T::kSpawnCap);
            bool ok = (err == 0u);
            if (!ok && lane == 0) raise_error(p.ctl, err);
            const bool fin = (sm.action == 1);
            const uint32_t total_children = staged;
            if (ok && !T::kTaskwait && lane == 0) {
                // +children must reach the counter before they are published; this task's -1 may be
                // deferred (the counter then only stays positive longer): fold it into the +children
                // when there are children, else batch it locally (flushed every 64 tasks or when idle)
                const uint32_t nfin = kMT > 1 ? sm.mt_n : 1u;
                if (staged) {
                    const long long delta = (long long)staged - (long long)nfin - (long long)L.local_dec;
                    L.local_dec = 0;
                    if (delta > 0) red_add_relaxed(reinterpret_cast<unsigned long long*>(&p.ctl->outstanding),
                                                   (unsigned long long)delta);
                    else if (delta < 0 && atom_add_acq_rel(&p.ctl->outstanding, delta) == -delta)
                        st_release(&p.ctl->done, 1u);
                } else if ((L.local_dec += nfin) >= 64u) {
                    const long long dec = (long long)L.local_dec;
                    L.local_dec = 0;
                    if (atom_add_acq_rel(&p.ctl->outstanding, -dec) == dec) st_release(&p.ctl->done, 1u);
                }
            }
            if (ok) {
                // a resumed parent takes the kept slot later; the kept child is then pushed
                ok = block_publish_spawns<T>(p, L, sm, w, lane, staged, T::kTaskwait ? my : kNone, keep_child_of<T>::value,
                                             false);
            }
            if (ok) {
                if (sm.action == 2) {
                    // suspend: resumption state + join counter
                    GTAP_CK(if (lane == 0) ck_suspend(p, my, total_children));
                    if (lane == 0) st_v4(p.rec + my, make_uint4(total_children, 0u, make_meta(sm.fn, sm.next_state, sm.ord, 0), sm.parent));
                    if (total_children == 0u) {
                        GTAP_CK(if (lane == 0) ck_publish(p, my));
                        if (L.kept != kNone) {  // keep the continuation, push the kept child instead
                            if (lane == 0) ring[L.tail & qmask] = L.kept;
                            L.tail += 1u;
                        }
                        L.kept = my;
                        if (lane == 0) sm.kept_fresh = 0u;  // a continuation: reload its record
                    }
                } else if (fin) {
                    const uint32_t parent = sm.parent;
                    if (parent != kNone && !is_root_link(parent) && sm.has_result && lane == 0)
                        st_relaxed(reinterpret_cast<int32_t*>(&p.rec[parent].d[2 + sm.ord]), sm.result);
                    GTAP_CK(if (lane == 0) ck_free(p, my));
                    if (lane == 0) block_free1(p, sm, w, my);
                    if constexpr (kMT > 1) {
                        if (lane == 0) {
                            for (uint32_t k = 1; k < sm.mt_n; ++k) {
                                GTAP_CK(ck_free(p, sm.mt_id[k]));
                                block_free1(p, sm, w, sm.mt_id[k]);
                            }
                        }
                    }
                    __syncwarp();
                    uint32_t resume = kNone;
                    if (lane == 0) {
                        if (parent != kNone && !is_root_link(parent)) {
                            GTAP_CK(ck_join(p, parent));
                            if (atom_add_acq_rel(&p.rec[parent].pending, -1) == 1) resume = parent;
                        } else if (is_root_link(parent)) {
                            p.root_results[parent & ~kRootFlag] = sm.has_result ? (long long)sm.result : 0ll;
                            if (T::kTaskwait && atom_add_acq_rel(&p.ctl->roots_left, 0xFFFFFFFFu) == 1u)
                                st_release(&p.ctl->done, 1u);
                        }
                    }
                    GTAP_CK(if (lane == 0 && resume != kNone) ck_publish(p, resume));
                    resume = __shfl_sync(0xffffffffu, resume, 0);
                    if (resume != kNone) {
                        if (L.kept != kNone) {
                            if (lane == 0) ring[L.tail & qmask] = L.kept;
                            L.tail += 1u;
                        }
                        L.kept = resume;
                        if (lane == 0) sm.kept_fresh = 0u;
                    }
                }
                block_maybe_publish(p, L, w, lane, true);
            }
            __syncwarp();
        }
        // (next iteration's acquire runs in warp 0; other warps wait at the barrier above)
    }

    if (warp == 0 && lane == 0) {
        unsigned long long* s = p.ctl->stats;
        for (int i = 0; i < ST_COUNT; ++i)
            if (i != ST_MAX_POOL && L.st[i]) atomicAdd(&s[i], L.st[i]);
        atomicMax(&s[ST_MAX_POOL], (unsigned long long)L.bump);
    }
}

// Mid-body flush for tables without taskwait: publish staged spawns when the
// staging buffer could overflow in the next chunk. Must be called uniformly
// by all threads of the block.
template <class T>
__device__ void block_flush(BlockSmem<T>& sm, const KParams& p, BLeader& L, uint32_t w,
                                            uint32_t headroom) {
    static_assert(!T::kTaskwait, "mid-body flush would publish children before the join count is set");
    __syncthreads();
    const uint32_t staged = sm.nspawn;
    if (staged + headroom > (uint32_t)T::kSpawnCap) {
        if ((threadIdx.x >> 5) == 0) {
            const uint32_t lane = threadIdx.x & 31u;
            block_publish_spawns<T>(p, L, sm, w, lane, min(staged, (uint32_t)T::kSpawnCap), kNone, false, true);
            block_maybe_publish(p, L, w, lane);
        }
        __syncthreads();
        if (threadIdx.x == 0) sm.nspawn = 0;
        __syncthreads();
    }
}

}  // namespace gtap
