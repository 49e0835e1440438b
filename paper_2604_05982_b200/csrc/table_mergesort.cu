// table_mergesort.cu -- cutoff mergesort task table (thread-level).
//
// PAPER.md P:153-165 (Prog. cutoff mergesort) with the state machine of
// P:59-74:  case 0: if (right - left <= CUTOFF) { sequential_sort; return; }
//                   mid = (left + right) / 2; fork [left, mid), [mid, right);
//                   store_state(1); return;
//           case 1: merge(data, left, mid, right); return;
// Readings: half-open ranges, mid = l + (r - l) / 2 (R14);
// sequential_sort = insertion sort, merge = two-pointer stable merge (R15).
//
// B200 layout choice (not in the paper): ping-pong buffers by depth. A task
// at depth e leaves its sorted range in buf(e) = (e even ? keys : scratch):
// a leaf sorts keys[l, r) into buf(e); an internal task merges its two
// children's ranges from buf(e + 1) into buf(e). Every key is read and
// written exactly once per tree level (8 B/key/level, no copy-back), and the
// root (depth 0) ends in `keys`. The output is the unique sorted permutation
// either way. Payload: d[0] = l, d[1] = r, d[2] = depth.
#include <climits>
#include <type_traits>

#include "table_common.cuh"
#include "warp_sort.cuh"
#include "warp_merge.cuh"

namespace gtap {

constexpr int kMsMaxCutoff = 256;


// One thread merges src[l, m) and src[m, r) into dst[l, r) (thread-executed
// task; the paper's merge is "largely sequential and executed by a
// single thread-level worker"). Two independent dependency chains run
// interleaved: the front chain emits the ceil(n/2) smallest keys (ties: left
// run first), the back chain the floor(n/2) largest (ties: right run last), so
// the output equals the plain two-pointer stable merge. In long stretches
// where no run can end, each chain reads its runs through 4-key register
// windows refilled 4 keys ahead (no bounds checks, no sentinels) with L1
// prefetches 512 B further out; near the run ends a checked scalar step is used.
__device__ __noinline__ void ms_merge(const int32_t* __restrict__ src, int32_t* __restrict__ dst, uint32_t l,
                                      uint32_t m, uint32_t r) {
    const uint32_t n = r - l;
    const uint32_t nf = (n + 1u) >> 1, nb = n - nf;
    uint32_t ia = l, ib = m, kf = l;          // front chain
    int32_t ja = (int32_t)m - 1, jb = (int32_t)r - 1;  // back chain (inclusive tails)
    uint32_t kb = r - 1u;
    uint32_t done = 0;                         // paired steps done (front and back each)
    while (done < nb) {
        // unchecked steps available: every window refill index stays inside its run
        int64_t S = (int64_t)min(min(m - ia, r - ib), min((uint32_t)(ja - (int32_t)l + 1), (uint32_t)(jb - (int32_t)m + 1))) - 5;
        S = min(S, (int64_t)(nb - done));
        if (S >= 16) {
            int32_t a0 = src[ia], a1 = src[ia + 1], a2 = src[ia + 2], a3 = src[ia + 3];
            int32_t b0 = src[ib], b1 = src[ib + 1], b2 = src[ib + 2], b3 = src[ib + 3];
            int32_t c0 = src[ja], c1 = src[ja - 1], c2 = src[ja - 2], c3 = src[ja - 3];
            int32_t e0 = src[jb], e1 = src[jb - 1], e2 = src[jb - 2], e3 = src[jb - 3];
            const uint32_t steps = (uint32_t)S;
            for (uint32_t t = 0; t < steps; ++t) {
                if ((t & 7u) == 0u) {
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(src + min(ia + 128u, m - 1u)));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(src + min(ib + 128u, r - 1u)));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(src + max(ja - 128, (int32_t)l)));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(src + max(jb - 128, (int32_t)m)));
                }
                if (b0 < a0) {  // front: right run only if strictly smaller
                    dst[kf] = b0; b0 = b1; b1 = b2; b2 = b3; b3 = src[ib + 4]; ++ib;
                } else {
                    dst[kf] = a0; a0 = a1; a1 = a2; a2 = a3; a3 = src[ia + 4]; ++ia;
                }
                ++kf;
                if (c0 > e0) {  // back: left run only if strictly larger
                    dst[kb] = c0; c0 = c1; c1 = c2; c2 = c3; c3 = src[ja - 4]; --ja;
                } else {
                    dst[kb] = e0; e0 = e1; e1 = e2; e2 = e3; e3 = src[jb - 4]; --jb;
                }
                --kb;
            }
            done += steps;
        } else {
            // checked scalar step for each chain
            const bool takeB = ib < r && (ia >= m || src[ib] < src[ia]);
            dst[kf++] = takeB ? src[ib++] : src[ia++];
            const bool takeA = ja >= (int32_t)l && (jb < (int32_t)m || src[ja] > src[jb]);
            dst[kb--] = takeA ? src[ja--] : src[jb--];
            ++done;
        }
    }
    if (nf > nb) {
        const bool takeB = ib < r && (ia >= m || src[ib] < src[ia]);
        dst[kf] = takeB ? src[ib] : src[ia];
    }
}


// ---------------------------------------------------------------------------
// TMA-staged single-thread merge (B200 path for large merges).
//
// Calibration on B200 (profiles/r01_calib_single_thread.txt): one thread
// streaming 4-byte global loads sustains only ~13.5 ns per load even when the
// loads are independent and L2-resident, while shared-memory loads cost ~15 ns
// dependent and far less pipelined. So the thread that runs a large merge
// streams its two runs (from both ends) through shared memory with 1-D bulk
// TMA copies (cp.async.bulk, mbarrier completion), and streams its two output
// halves back with bulk stores: the thread then only issues one bulk copy per
// 512 keys per stream and merges out of shared memory. One 24 KB merge slot
// per block; a lane claims it with a shared-memory CAS, other lanes use
// ms_merge. Partial chunks at the ends of the output range are written with
// plain stores (a bulk store must not touch a neighbouring task's keys).
namespace tma {
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* mb, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mb, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mb, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P;\n"
        "GTAP_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra GTAP_WAIT_%=;\n}" ::"r"(sa(mb)), "r"(parity) : "memory");
}
__device__ __forceinline__ void g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* mb) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
                 "l"(src), "r"(bytes), "r"(sa(mb)) : "memory");
}
__device__ __forceinline__ void s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sa(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void wait_read(uint32_t n) {  // <= n most recent bulk groups may still read smem
    if (n == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    else if (n == 1) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    else if (n == 2) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
    else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
}
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
}  // namespace tma

__device__ __forceinline__ int32_t lds(uint32_t a) {
    int32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts(uint32_t a, int32_t v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

#ifdef GTAP_MS_PROBE_STATS
__device__ long long gtap_ms_probe[8];
extern "C" int gtap_ms_probe_read(long long* h) {
    cudaMemcpyFromSymbol(h, gtap_ms_probe, sizeof(long long) * 8);
    long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(gtap_ms_probe, z, sizeof(z));
    return 0;
}
#endif

#ifndef GTAP_MS_CHAINS
#define GTAP_MS_CHAINS 4
#endif
constexpr int kChains = GTAP_MS_CHAINS;      // independent merge chains interleaved in one thread
constexpr int kIn = 256;                     // keys per input chunk (1 KB bulk load)
constexpr int kOut = 128;                    // keys per output chunk (512 B bulk store)
constexpr int kRing = 512;                   // keys per ring (2 input chunks / 4 output chunks), 2 KB
constexpr uint32_t kRingMaskB = kRing * 4u - 1u;
constexpr uint32_t kTmaMin = 8192;           // merges at least this long take the TMA path
constexpr uint32_t kNoChunk = 0x80000000u;
#ifdef GTAP_MS_TRACE
// diagnostic build only: one record per merge / leaf / assist / chunk:
// {t0, t1, size << 32 | l, smid << 8 | kind}; kinds: 0 lane merge, 1 TMA merge, 2 leaf sort,
// 3 warp assist, 4 block assist (requester), 5 GPU-wide assist (requester), 6 GPU-wide chunk, 7 block chunk
constexpr uint32_t kMsTraceCap = 1u << 20;
__device__ ulonglong4 gtap_ms_trace[kMsTraceCap];
__device__ uint32_t gtap_ms_trace_n;
extern "C" int gtap_ms_trace_read(void* host, uint32_t* n) {
    cudaMemcpyFromSymbol(n, gtap_ms_trace_n, 4);
    cudaMemcpyFromSymbol(host, gtap_ms_trace, sizeof(ulonglong4) * (*n < kMsTraceCap ? *n : kMsTraceCap));
    const uint32_t z = 0;
    cudaMemcpyToSymbol(gtap_ms_trace_n, &z, 4);
    return 0;
}
__device__ __forceinline__ void ms_trace(unsigned long long t0, uint32_t size, uint32_t l, uint32_t kind) {
    const uint32_t i = atomicAdd(&gtap_ms_trace_n, 1u);
    if (i < kMsTraceCap) {
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        gtap_ms_trace[i] = make_ulonglong4(t0, dev::globaltimer(), ((unsigned long long)size << 32) | l,
                                           ((unsigned long long)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) << 32) | ((unsigned long long)smid << 8) | kind);
    }
}
#define MS_T0 const unsigned long long ms_t0 = dev::globaltimer()
#define MS_TRACE(size, l, kind) ms_trace(ms_t0, (size), (l), (kind))
#define MS_TRACE_LANE0(size, l, kind) do { if (lane == 0) ms_trace(ms_t0, (size), (l), (kind)); } while (0)
#else
#define MS_T0 do {} while (0)
#define MS_TRACE(size, l, kind) do {} while (0)
#define MS_TRACE_LANE0(size, l, kind) do {} while (0)
#endif

struct MergeSlot {                           // placed 2 KB-aligned inside the block's dynamic smem
    int32_t in[2 * kChains][kRing];          // per chain: A ring, B ring
    int32_t out[kChains][kRing];             // per chain: output ring
    unsigned long long mbar[2 * kChains][2];
    uint32_t par[2 * kChains];               // mbarrier parity bits per input ring
};
// warp-assist merge tiles (GTAP_MERGE_WARP): per warp, one smem ring per input run
#ifndef GTAP_MS_WT
#define GTAP_MS_WT 256
#endif
#ifndef GTAP_MS_WR
#define GTAP_MS_WR 1024
#endif
constexpr int kWT = GTAP_MS_WT;              // outputs per tile
constexpr int kVT = kWT / 32;                // outputs per lane per tile
constexpr int kWR = GTAP_MS_WR;              // keys per ring
constexpr uint32_t kTopChunk = kWT / 2;      // cp.async top-up granule
// window issued >= 2 tiles before it is read (wait_group 1): top-ups trail pa + kWR by < kTopChunk
// keys and a tile consumes <= kWT keys of a run
static_assert(kWR >= 3 * kWT + (int)kTopChunk - 1, "ring too small for wait_group 1");
static_assert((kWR & (kWR - 1)) == 0 && kWT % 64 == 0, "ring: power of two; tile: multiple of 64");
struct WarpTiles {
    int32_t a[kWR];
    int32_t b[kWR];
};
constexpr int kMsWarps = 4;                  // kMaxThreads / 32
struct MergeSlotHolder {                     // BlockExtra of merge_mode thread: 2 KB of slack to align the slot
    unsigned char raw[sizeof(MergeSlot) + 2048];
    uint32_t busy;
    __device__ __forceinline__ MergeSlot* slot() {
        const uint32_t a = tma::sa(raw);
        return reinterpret_cast<MergeSlot*>(raw + ((2048u - (a & 2047u)) & 2047u));
    }
};
static_assert(sizeof(WarpTiles) == sizeof(wm3::WM3Rings), "the two merge cores share the per-warp rings");
struct WarpAssistHolder {                    // BlockExtra of merge_mode warp: per-warp rings + block board
    // per-warp rings, R * 4-aligned (wm3) inside raw; the bulk-copy merge core's buffers and barriers
    unsigned char raw[sizeof(WarpTiles) * kMsWarps + sizeof(wm3::WM3Rings::ring[0])];
    wm3::WM3Aux aux[kMsWarps];
    // block assist board (merges >= kBlockAssistMin): one open merge per block
    struct Board {
        uint32_t state;               // 0 free, 1 being set up, 2 open
        uint32_t l, m, r, depth;
        uint32_t next;                // next chunk to claim (>= nchunks: closed)
        uint32_t nchunks, done;
    } board;
    __device__ __forceinline__ WarpTiles* tiles(uint32_t warp) {
        constexpr uint32_t kAl = sizeof(wm3::WM3Rings::ring[0]);   // one ring: the wrap alignment of wm3
        const uint32_t a = tma::sa(raw);
        return reinterpret_cast<WarpTiles*>(raw + ((kAl - (a & (kAl - 1u))) & (kAl - 1u))) + warp;
    }
    __device__ __forceinline__ wm3::WM3Tiles wtiles(uint32_t warp) {
        return wm3::WM3Tiles{reinterpret_cast<wm3::WM3Rings*>(tiles(warp)), &aux[warp]};
    }
};

__device__ __forceinline__ bool mbar_try(uint32_t mb, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}"
        : "=r"(ok) : "r"(mb), "r"(parity) : "memory");
    return ok != 0;
}

// Input run streamed through a 2-chunk ring. Up streams hold the resident window
// [chunk(pos)*kIn, rhi); down streams (rlo, ...] mirrored with rhi = lowest resident key.
struct InS {
    const int32_t* g;
    uint32_t ring;        // smem byte address (2 KB aligned)
    uint32_t mb;          // smem byte address of 2 mbarriers
    int32_t pos, lo, hi;  // head, run [lo, hi)
    int32_t edge;         // up: resident end (exclusive); down: lowest resident key
    uint32_t pend;        // chunk in flight or kNoChunk
    uint32_t par;
    int32_t nt;
};
__device__ __forceinline__ void in_issue(InS& s, int32_t c) {
    const int32_t b0 = c * kIn;
    const uint32_t bytes = (uint32_t)min(kIn, s.nt - b0) * 4u;
    const uint32_t sl = (uint32_t)c & 1u;
    tma::fence_smem();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s.mb + 8u * sl), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(s.ring + sl * (kIn * 4u)), "l"(s.g + b0), "r"(bytes), "r"(s.mb + 8u * sl) : "memory");
    s.pend = (uint32_t)c;
}
__device__ __forceinline__ bool in_poll(InS& s, bool block) {  // true if the pending chunk landed
    const uint32_t sl = s.pend & 1u;
    const uint32_t ph = (s.par >> sl) & 1u;
    if (block) {
        while (!mbar_try(s.mb + 8u * sl, ph)) {}
    } else if (!mbar_try(s.mb + 8u * sl, ph)) {
        return false;
    }
    s.par ^= 1u << sl;
    s.pend = kNoChunk;
    return true;
}
__device__ __forceinline__ void in_start(InS& s, bool up) {
    s.pend = kNoChunk;
    if (s.lo >= s.hi) { s.edge = up ? s.hi : s.lo; return; }
    const int32_t c = s.pos / kIn;
    in_issue(s, c);
    in_poll(s, true);
    s.edge = up ? (c + 1) * kIn : c * kIn;
}
// keep the window full: land a pending chunk, issue the next one into the free slot
// (issue first: a head that left the window gets its chunk requested and waited here)
__device__ __forceinline__ void in_maint(InS& s, bool up) {
    if (up) {
        if (s.pend == kNoChunk && s.edge < s.hi && s.edge - s.pos <= kIn) in_issue(s, s.edge / kIn);
        if (s.pend != kNoChunk && in_poll(s, s.pos + 1 >= s.edge)) s.edge += kIn;
    } else {
        if (s.pend == kNoChunk && s.edge > s.lo && s.pos - s.edge < kIn) in_issue(s, s.edge / kIn - 1);
        if (s.pend != kNoChunk && in_poll(s, s.pos - 1 < s.edge)) s.edge -= kIn;
    }
}
__device__ __forceinline__ int32_t in_safe(const InS& s, bool up) {
    return up ? min(s.edge, s.hi) - 1 - s.pos : s.pos - max(s.edge, s.lo);
}
__device__ __forceinline__ uint32_t in_addr(const InS& s, int32_t p) {
    return s.ring + (((uint32_t)p * 4u) & kRingMaskB);
}

// Output range streamed through a 4-chunk ring; completed chunks leave by bulk store
// (or plain stores for a chunk that is only partly inside [lo, hi)).
struct OutS {
    int32_t* g;
    uint32_t ring;
    int32_t pos, lo, hi;  // next position, range
    int32_t fl;           // next chunk to flush
    int32_t wend;         // up: writable end (exclusive); down: lowest writable key
    uint32_t gid[4];
};
__device__ __forceinline__ void out_flush(OutS& o, int32_t c, uint32_t& gc) {
    const int32_t b0 = c * kOut;
    const int32_t cs = max(b0, o.lo), ce = min(b0 + kOut, o.hi);
    const uint32_t sb = o.ring + ((uint32_t)(c & 3)) * (kOut * 4u);
    if (cs == b0 && ce == b0 + kOut) {
        tma::fence_smem();
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o.g + b0), "r"(sb),
                     "r"(kOut * 4u) : "memory");
        tma::commit();
        o.gid[c & 3] = ++gc;
    } else {
        for (int32_t i = cs; i < ce; ++i) o.g[i] = lds(sb + 4u * (uint32_t)(i - b0));
    }
}
__device__ __forceinline__ void out_claim(OutS& o, int32_t c, uint32_t gc) {  // slot of chunk c free to write
    const uint32_t gid = o.gid[c & 3];
    if (gid) { tma::wait_read(min(gc - gid, 3u)); o.gid[c & 3] = 0; }
}
__device__ __forceinline__ void out_start(OutS& o, bool up, uint32_t gc) {
    o.gid[0] = o.gid[1] = o.gid[2] = o.gid[3] = 0;
    if (up) { o.pos = o.lo; o.fl = o.lo / kOut; o.wend = (o.fl + 1) * kOut; }
    else    { o.pos = o.hi - 1; o.fl = o.hi > 0 ? (o.hi - 1) / kOut : 0; o.wend = o.fl * kOut; }
    (void)gc;
}
__device__ __forceinline__ void out_maint(OutS& o, bool up, uint32_t& gc) {
    if (up) {
        while (o.fl * kOut < o.hi && ((o.fl + 1) * kOut <= o.pos || o.pos == o.hi)) { out_flush(o, o.fl, gc); ++o.fl; }
        while (o.wend < o.hi && o.wend / kOut < o.fl + 3) { out_claim(o, o.wend / kOut, gc); o.wend += kOut; }
    } else {
        while (o.fl >= 0 && (o.fl + 1) * kOut > o.lo && (o.fl * kOut > o.pos || o.pos < o.lo)) {
            out_flush(o, o.fl, gc);
            --o.fl;
        }
        while (o.wend > o.lo && o.wend / kOut - 1 > o.fl - 3) { out_claim(o, o.wend / kOut - 1, gc); o.wend -= kOut; }
    }
}
__device__ __forceinline__ int32_t out_safe(const OutS& o, bool up) {
    return up ? min(o.wend, o.hi) - o.pos : o.pos - max(o.wend, o.lo) + 1;
}

struct Chain {
    InS A, B;
    OutS O;
    int32_t left;
};

// one checked step (exhausted runs read as 64-bit sentinels), used when a run is at its last key
__device__ __forceinline__ void chain_step_checked(Chain& ch, bool up) {
    InS& A = ch.A;
    InS& B = ch.B;
    if (up) {
        const long long a = A.pos < A.hi ? (long long)lds(in_addr(A, A.pos)) : 0x7fffffffffffffffll;
        const long long b = B.pos < B.hi ? (long long)lds(in_addr(B, B.pos)) : 0x7fffffffffffffffll;
        const bool tb = b < a;
        sts(ch.O.ring + (((uint32_t)ch.O.pos * 4u) & kRingMaskB), (int32_t)(tb ? b : a));
        ++ch.O.pos;
        if (tb) ++B.pos; else ++A.pos;
    } else {
        const long long a = A.pos >= A.lo ? (long long)lds(in_addr(A, A.pos)) : (long long)0x8000000000000000ull;
        const long long b = B.pos >= B.lo ? (long long)lds(in_addr(B, B.pos)) : (long long)0x8000000000000000ull;
        const bool ta = a > b;  // stable: left run only if strictly larger
        sts(ch.O.ring + (((uint32_t)ch.O.pos * 4u) & kRingMaskB), (int32_t)(ta ? a : b));
        --ch.O.pos;
        if (ta) --A.pos; else --B.pos;
    }
    --ch.left;
}

// stable merge-path split: number of A keys among the first t outputs of merge(A, B)
__device__ __forceinline__ uint32_t merge_path(const int32_t* src, uint32_t l, uint32_t m, uint32_t r, uint32_t t) {
    uint32_t lo = t > (r - m) ? t - (r - m) : 0u, hi = min(t, m - l);
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (src[l + mid] <= src[m + (t - mid - 1)]) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Stable merge of src[l, m) and src[m, r) into dst[l, r) by ONE thread through
// the block's merge slot (nt = array length, a multiple of 4; 16-B aligned).
// The output is cut by merge-path searches into kChains/2 independent
// sub-merges, each produced from both ends (an ascending and a descending
// chain), so kChains dependency chains interleave in the hot loop. Between
// stretches every stream is maintained (bulk loads landed/issued, output
// chunks flushed by bulk store, output slots reclaimed); a stretch is as long
// as every chain can go without reaching a window edge or a run end.
// Returns false if the merge stopped making progress (a bug surfaced as GTAP_E_BAD_STATE).
__device__ __noinline__ bool ms_merge_tma(const int32_t* src, int32_t* dst, uint32_t l, uint32_t m, uint32_t r,
                                          uint32_t nt, MergeSlotHolder* H) {
    bool ok = true;
    MergeSlot* S = H->slot();
    tma::fence_global();  // children's generic-proxy writes (acquired at the join) -> async-proxy reads
    constexpr int kSub = kChains / 2;
    const uint32_t n = r - l;
    uint32_t cut_a[kSub + 1], cut_t[kSub + 1];
#pragma unroll
    for (int q = 0; q <= kSub; ++q) {
        const uint32_t t = (uint32_t)(((unsigned long long)n * q) / kSub);
        cut_t[q] = t;
        cut_a[q] = (q == 0) ? 0u : (q == kSub ? m - l : merge_path(src, l, m, r, t));
    }
    Chain ch[kChains];
    uint32_t gc = 0;
#pragma unroll
    for (int k = 0; k < kChains; ++k) {
        const int q = k >> 1;
        const bool up = (k & 1) == 0;
        Chain& c = ch[k];
        const int32_t alo = (int32_t)(l + cut_a[q]), ahi = (int32_t)(l + cut_a[q + 1]);
        const int32_t blo = (int32_t)(m + cut_t[q] - cut_a[q]), bhi = (int32_t)(m + cut_t[q + 1] - cut_a[q + 1]);
        const int32_t olo = (int32_t)(l + cut_t[q]), ohi = (int32_t)(l + cut_t[q + 1]);
        const int32_t nq = ohi - olo, nf = (nq + 1) >> 1;
        c.A.g = c.B.g = src;
        c.A.nt = c.B.nt = (int32_t)nt;
        c.A.ring = tma::sa(&S->in[2 * k][0]);
        c.B.ring = tma::sa(&S->in[2 * k + 1][0]);
        c.A.mb = tma::sa(&S->mbar[2 * k][0]);
        c.B.mb = tma::sa(&S->mbar[2 * k + 1][0]);
        c.A.par = S->par[2 * k];
        c.B.par = S->par[2 * k + 1];
        c.A.lo = alo; c.A.hi = ahi; c.B.lo = blo; c.B.hi = bhi;
        c.A.pos = up ? alo : ahi - 1;
        c.B.pos = up ? blo : bhi - 1;
        c.O.g = dst;
        c.O.ring = tma::sa(&S->out[k][0]);
        c.O.lo = up ? olo : olo + nf;
        c.O.hi = up ? olo + nf : ohi;
        c.left = c.O.hi - c.O.lo;
        in_start(c.A, up);
        in_start(c.B, up);
        out_start(c.O, up, gc);
    }
#ifdef GTAP_MS_PROBE_STATS
    long long t_hot = 0, t_all0 = clock64(), n_str = 0, n_fast = 0, n_chk = 0;
#endif
    uint32_t stall = 0;
    while (true) {
        int32_t steps = 0x7fffffff;
        int32_t work = 0, done_any = 0;
#pragma unroll
        for (int k = 0; k < kChains; ++k) {
            work |= ch[k].left;
            done_any |= (ch[k].left == 0);
        }
        if (work == 0) break;
#pragma unroll
        for (int k = 0; k < kChains; ++k) {
            const bool up = (k & 1) == 0;
            Chain& c = ch[k];
            in_maint(c.A, up);
            in_maint(c.B, up);
            out_maint(c.O, up, gc);
            steps = min(steps, min(min(in_safe(c.A, up), in_safe(c.B, up)), min(out_safe(c.O, up), c.left)));
        }
        if (steps <= 0 || done_any) {
            // an edge (run end, ring wrap, window edge) or the last keys: one checked step on
            // every chain that can write (heads are resident after in_maint)
            bool moved = false;
#pragma unroll
            for (int k = 0; k < kChains; ++k) {
                const bool up = (k & 1) == 0;
                if (ch[k].left > 0 && out_safe(ch[k].O, up) > 0) {
                    chain_step_checked(ch[k], up);
                    moved = true;
#ifdef GTAP_MS_PROBE_STATS
                    ++n_chk;
#endif
                }
            }
            if (!moved && ++stall > (1u << 24)) {  // no chain could move for a long time: a bug, not a hang
                ok = false;
                break;
            }
            continue;
        }
        stall = 0;
        // hot loop: `steps` unchecked steps on every chain; heads and outputs move through ring byte
        // addresses (IADD + LOP3 each): per key 1 compare, 1 min/max, 1 st.shared, 2 ld.shared
#ifdef GTAP_MS_PROBE_STATS
        const long long th0 = clock64();
        ++n_str; n_fast += steps;
#endif
        // tagged smem byte addresses: every ring is 2 KB and 2 KB-aligned, so a head moves by
        // addr = ring | ((addr + 4) & mask): one IADD + one LOP3, and ld/st.shared use it directly
        uint32_t ao[kChains], bo[kChains], oo[kChains];
        int32_t av[kChains], bv[kChains];
        int32_t da[kChains], db[kChains];
#pragma unroll
        for (int k = 0; k < kChains; ++k) {
            ao[k] = ch[k].A.ring | (((uint32_t)ch[k].A.pos * 4u) & kRingMaskB);
            bo[k] = ch[k].B.ring | (((uint32_t)ch[k].B.pos * 4u) & kRingMaskB);
            oo[k] = ch[k].O.ring | (((uint32_t)ch[k].O.pos * 4u) & kRingMaskB);
            av[k] = lds(ao[k]);
            bv[k] = lds(bo[k]);
            da[k] = db[k] = 0;
            ch[k].left -= steps;
        }
#pragma unroll 4
        for (int32_t st = 0; st < steps; ++st) {
#pragma unroll
            for (int k = 0; k < kChains; ++k) {
                const uint32_t ra = ch[k].A.ring, rb = ch[k].B.ring, ro = ch[k].O.ring;
                if ((k & 1) == 0) {  // ascending chain: right run only if strictly smaller
                    const uint32_t d = bv[k] < av[k] ? 4u : 0u;
#ifndef GTAP_MS_PROBE_NOSTORE
                    sts(oo[k], min(av[k], bv[k]));
#endif
                    oo[k] = ro | ((oo[k] + 4u) & kRingMaskB);
                    ao[k] = ra | ((ao[k] + 4u - d) & kRingMaskB);
                    bo[k] = rb | ((bo[k] + d) & kRingMaskB);
                    db[k] += (int32_t)d;
                } else {             // descending chain: left run only if strictly larger
                    const uint32_t d = av[k] > bv[k] ? 4u : 0u;
#ifndef GTAP_MS_PROBE_NOSTORE
                    sts(oo[k], max(av[k], bv[k]));
#endif
                    oo[k] = ro | ((oo[k] - 4u) & kRingMaskB);
                    ao[k] = ra | ((ao[k] - d) & kRingMaskB);
                    bo[k] = rb | ((bo[k] - 4u + d) & kRingMaskB);
                    da[k] += (int32_t)d;
                }
                av[k] = lds(ao[k]);
                bv[k] = lds(bo[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < kChains; ++k) {
            // up: B moved db/4 keys, A the rest; down: A moved da/4 keys, B the rest
            if ((k & 1) == 0) {
                ch[k].B.pos += db[k] / 4;
                ch[k].A.pos += steps - db[k] / 4;
                ch[k].O.pos += steps;
            } else {
                ch[k].A.pos -= da[k] / 4;
                ch[k].B.pos -= steps - da[k] / 4;
                ch[k].O.pos -= steps;
            }
        }
#ifdef GTAP_MS_PROBE_STATS
        t_hot += clock64() - th0 + (long long)(av[0] & 0);
#endif
    }
#ifdef GTAP_MS_PROBE_STATS
    if (n >= gtap_ms_probe[7]) {  // keep the stats of the largest merge
        gtap_ms_probe[7] = n;
        gtap_ms_probe[0] = clock64() - t_all0; gtap_ms_probe[1] = t_hot; gtap_ms_probe[2] = n_str;
        gtap_ms_probe[3] = n_fast; gtap_ms_probe[4] = n_chk;
    }
#endif
#pragma unroll
    for (int k = 0; k < kChains; ++k) {
        const bool up = (k & 1) == 0;
        out_maint(ch[k].O, up, gc);  // flush the final (partial) chunks
        if (ch[k].A.pend != kNoChunk) in_poll(ch[k].A, true);
        if (ch[k].B.pend != kNoChunk) in_poll(ch[k].B, true);
        S->par[2 * k] = ch[k].A.par;
        S->par[2 * k + 1] = ch[k].B.par;
    }
    tma::wait_all();
    tma::fence_global();  // async-proxy writes complete before the join's release
    return ok;
}

// ---------------------------------------------------------------------------
// Warp-assisted merge (B200 design): a heavy merge
// task's body is run by all 32 lanes of its warp after the cycle's bodies (the
// other lanes' own tasks have run by then). The output is produced in tiles of
// kWT keys. Each input run streams through a per-warp shared-memory ring of kWR
// keys, kept topped up by 4-byte cp.async copies in 128-key chunks (one commit
// group per tile; top-ups trail pa + kWR by < 128 keys and a tile consumes
// <= kWT keys of a run, so the window a tile reads was issued >= 2 tiles
// earlier and `wait_group 1` suffices). Per tile, lane k finds the
// start of its kVT outputs by a stable merge-path search in the rings and merges
// them serially from shared memory; the run consumption of the tile is the last
// active lane's position. Ties take the left run first (search and serial step
// alike), so the output is the stable two-pointer merge.
namespace wm {
__device__ __forceinline__ void cp4(const int32_t* sdst, const int32_t* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(tma::sa(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// lanes copy src[from, to) into ring positions (global index & (kWR - 1)): whole kTopChunk-key
// chunks (no tail) while they fit, the rest only at the run's end. Returns the new `from`.
__device__ __forceinline__ uint32_t topup(int32_t* ring, const int32_t* src, uint32_t from, uint32_t to,
                                          uint32_t end, uint32_t lane) {
    while (from + kTopChunk <= to) {
#pragma unroll
        for (uint32_t k = 0; k < kTopChunk / 32u; ++k) {
            const uint32_t i = from + lane + 32u * k;
            cp4(ring + (i & (kWR - 1u)), src + i);
        }
        from += kTopChunk;
    }
    if (to == end) {
        for (uint32_t i = from + lane; i < to; i += 32u) cp4(ring + (i & (kWR - 1u)), src + i);
        from = to;
    }
    return from;
}
}  // namespace wm

// all 32 lanes: stable merge of src[a0, m) and src[b0, r) into dst[o0, o0 + (m - a0) + (r - b0))
__device__ __noinline__ void warp_merge(const int32_t* __restrict__ src, int32_t* __restrict__ dst, uint32_t a0,
                                        uint32_t m, uint32_t b0, uint32_t r, uint32_t o0, uint32_t lane,
                                        WarpTiles* T) {
    int32_t* RA = T->a;
    int32_t* RB = T->b;
    const uint32_t l = a0, oend = o0 + (m - a0) + (r - b0);
    uint32_t pa = a0, pb = b0, out = o0;              // next key of each run, next output
    uint32_t la = wm::topup(RA, src, l, min(m, l + (uint32_t)kWR), m, lane);   // loaded (issued) up to
    uint32_t lb = wm::topup(RB, src, b0, min(r, b0 + (uint32_t)kWR), r, lane);
    wm::commit();
    wm::commit();
    wm::commit();
    while (out < oend) {
        const uint32_t tile = min((uint32_t)kWT, oend - out);
        wm::wait<1>();  // the window was issued >= 2 tiles ago (see kTopChunk)
        __syncwarp();
        const uint32_t na = min(tile, m - pa), nb = min(tile, r - pb);
        // the tile's kWT outputs by one bitonic half-cleaner + merge network over registers:
        // element e = k * 32 + lane of A[pa, pa + kWT) ++ reverse(B[pb, pb + kWT)) (runs padded with
        // +inf past na / nb); c[e] = min(A[e], B[kWT-1-e]) is bitonic and holds the kWT smallest keys,
        // and A[e] is taken iff A[e] <= B[kWT-1-e] (ties: left run first), so the count of taken A
        // keys is the stable merge-path split of the tile; log2(kWT) compare stages sort c.
        // Every smem access and the global stores are lane-contiguous (no search, no serial chain).
        int32_t x[kVT];
        uint32_t ca = 0;
#pragma unroll
        for (int k = 0; k < kVT; ++k) {
            const uint32_t e = (uint32_t)k * 32u + lane, j = (uint32_t)kWT - 1u - e;
            const bool ha = e < na, hb = j < nb;
            const int32_t va = ha ? RA[(pa + e) & (kWR - 1u)] : INT_MAX;
            const int32_t vb = hb ? RB[(pb + j) & (kWR - 1u)] : INT_MAX;
            const bool takeA = ha && (!hb || va <= vb);
            x[k] = takeA ? va : vb;
            ca += (uint32_t)__popc(__ballot_sync(0xffffffffu, takeA));
        }
#pragma unroll
        for (uint32_t stride = (uint32_t)kWT >> 1; stride > 0u; stride >>= 1) {
            if (stride >= 32u) {
#pragma unroll
                for (int k = 0; k < kVT; ++k) {
                    const int kk = k ^ (int)(stride >> 5);
                    if (kk > k) {
                        const int32_t u = x[k], v = x[kk];
                        x[k] = min(u, v);
                        x[kk] = max(u, v);
                    }
                }
            } else {
                const bool lower = (lane & stride) == 0u;
#pragma unroll
                for (int k = 0; k < kVT; ++k) {
                    const int32_t p = __shfl_xor_sync(0xffffffffu, x[k], stride);
                    x[k] = lower ? min(x[k], p) : max(x[k], p);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < kVT; ++k) {
            const uint32_t e = (uint32_t)k * 32u + lane;
            if (e < tile) dst[out + e] = x[k];
        }
        __syncwarp();                                  // ring reads done before the top-up
        pa += ca;
        pb += tile - ca;
        out += tile;
        la = wm::topup(RA, src, la, min(m, pa + (uint32_t)kWR), m, lane);
        lb = wm::topup(RB, src, lb, min(r, pb + (uint32_t)kWR), r, lane);
        wm::commit();
    }
    wm::wait<0>();
    __threadfence();  // every lane's stores before the requesting lane's join release
    __syncwarp();
}

// all 32 lanes: stable merge-path splits (A keys among the first t outputs of merge(src[l, m), src[m, r)))
// over global memory, 32 probes per step (a ~33-way search: ~5 dependent round trips for 2^23 keys);
// both splits of a chunk [t0, t1) in lockstep (one dependent round trip per step for the pair)
__device__ __noinline__ uint2 warp_split2(const int32_t* src, uint32_t l, uint32_t m, uint32_t r, uint32_t t0,
                                          uint32_t t1, uint32_t lane) {
    uint32_t lo0 = t0 > (r - m) ? t0 - (r - m) : 0u, hi0 = min(t0, m - l);
    uint32_t lo1 = t1 > (r - m) ? t1 - (r - m) : 0u, hi1 = min(t1, m - l);
    {
        // first round: 32 probes s apart around the proportional guess t * |A| / (|A| + |B|) (a
        // random merge's split lies within a few sqrt(t) of it); a bracket found there leaves ~s
        // positions (1-2 further rounds instead of ~4), a miss still halves nothing worse than before
        const unsigned long long na = m - l, nn = r - l;
        const uint32_t g0 = (uint32_t)((t0 * na) / nn), g1 = (uint32_t)((t1 * na) / nn);
        const uint32_t s = max(32u, 1u << ((33u - (uint32_t)__clz(max(t1, 1u))) / 2u)) >> 2;  // ~sqrt(t1) / 4
        uint32_t q0 = g0 + lane * s, q1 = g1 + lane * s;
        q0 = q0 >= 15u * s ? q0 - 15u * s : 0u;
        q1 = q1 >= 15u * s ? q1 - 15u * s : 0u;
        q0 = min(max(q0, lo0), hi0 > 0u ? hi0 - 1u : 0u);
        q1 = min(max(q1, lo1), hi1 > 0u ? hi1 - 1u : 0u);
        const bool a0 = hi0 - lo0 > 32u && __ldcg(src + l + q0) <= __ldcg(src + m + (t0 - q0 - 1u));
        const bool a1 = hi1 - lo1 > 32u && __ldcg(src + l + q1) <= __ldcg(src + m + (t1 - q1 - 1u));
        // predicate true below the split, false from it on: the ballot is a prefix of lanes
        const uint32_t c0 = (uint32_t)__popc(__ballot_sync(0xffffffffu, a0));
        const uint32_t c1 = (uint32_t)__popc(__ballot_sync(0xffffffffu, a1));
        const uint32_t ql0 = __shfl_sync(0xffffffffu, q0, (c0 + 31u) & 31u), qh0 = __shfl_sync(0xffffffffu, q0, c0 & 31u);
        const uint32_t ql1 = __shfl_sync(0xffffffffu, q1, (c1 + 31u) & 31u), qh1 = __shfl_sync(0xffffffffu, q1, c1 & 31u);
        if (hi0 - lo0 > 32u) { if (c0 > 0u) lo0 = max(lo0, ql0 + 1u); if (c0 < 32u) hi0 = min(hi0, qh0); }
        if (hi1 - lo1 > 32u) { if (c1 > 0u) lo1 = max(lo1, ql1 + 1u); if (c1 < 32u) hi1 = min(hi1, qh1); }
    }
    while (hi0 - lo0 > 32u || hi1 - lo1 > 32u) {
        const uint32_t w0 = hi0 - lo0, w1 = hi1 - lo1;
        const uint32_t q0 = lo0 + (uint32_t)(((unsigned long long)(lane + 1u) * w0) / 33u);
        const uint32_t q1 = lo1 + (uint32_t)(((unsigned long long)(lane + 1u) * w1) / 33u);
        const bool a0 = w0 > 32u && __ldcg(src + l + q0) <= __ldcg(src + m + (t0 - q0 - 1u));
        const bool a1 = w1 > 32u && __ldcg(src + l + q1) <= __ldcg(src + m + (t1 - q1 - 1u));
        const uint32_t c0 = (uint32_t)__popc(__ballot_sync(0xffffffffu, a0));
        const uint32_t c1 = (uint32_t)__popc(__ballot_sync(0xffffffffu, a1));
        const uint32_t ql0 = __shfl_sync(0xffffffffu, q0, (c0 + 31u) & 31u), qh0 = __shfl_sync(0xffffffffu, q0, c0 & 31u);
        const uint32_t ql1 = __shfl_sync(0xffffffffu, q1, (c1 + 31u) & 31u), qh1 = __shfl_sync(0xffffffffu, q1, c1 & 31u);
        if (w0 > 32u) { if (c0 > 0u) lo0 = ql0 + 1u; if (c0 < 32u) hi0 = qh0; }
        if (w1 > 32u) { if (c1 > 0u) lo1 = ql1 + 1u; if (c1 < 32u) hi1 = qh1; }
    }
    const uint32_t q0 = lo0 + lane, q1 = lo1 + lane;
    const bool a0 = q0 < hi0 && __ldcg(src + l + q0) <= __ldcg(src + m + (t0 - q0 - 1u));
    const bool a1 = q1 < hi1 && __ldcg(src + l + q1) <= __ldcg(src + m + (t1 - q1 - 1u));
    return make_uint2(lo0 + (uint32_t)__popc(__ballot_sync(0xffffffffu, a0)),
                      lo1 + (uint32_t)__popc(__ballot_sync(0xffffffffu, a1)));
}

#ifndef GTAP_MS_BLOCK_MIN
#define GTAP_MS_BLOCK_MIN (1u << 17)
#endif
#ifndef GTAP_MS_BCHUNK
#define GTAP_MS_BCHUNK (1u << 16)
#endif
constexpr uint32_t kBlockAssistMin = GTAP_MS_BLOCK_MIN;  // merges this long are shared by the block's warps
constexpr uint32_t kChunk = GTAP_MS_BCHUNK;      // output keys per claimed chunk (block board)

// GPU-wide assist board (GTAP_MERGE_WARP, merges >= kGlobalAssistMin): any idle warp of the grid
// claims kGChunk-key output chunks of an open slot. Slot protocol (all words in global memory):
// requester CAS state 0 -> 1, writes the parameters, fence, next = 0, fence, state = 2 (release),
// open += 1; a claim is atomicAdd(next) followed by a fence and the parameter reads, so a claim that
// lands after a reopen sees the new parameters; closing sets next = 2^31 (late claims fail) before
// state = 0. A helper fences its chunk's stores before done += 1; the requester waits for
// done == nchunks and fences before its join release.
constexpr uint32_t kGSlots = 1024;
#ifndef GTAP_MS_GLOBAL_MIN
#define GTAP_MS_GLOBAL_MIN 32768   // 8192 / 16384 / 32768 / 65536: 1.57 / 1.43 / 1.41 / 1.46 ms at 2^24
#endif
#ifndef GTAP_MS_GCHUNK
#define GTAP_MS_GCHUNK 4096   // 2048 / 3072 / 4096 / 6144: 1.51 / 1.46 / 1.44 / 1.50 ms at 2^24
#endif
#ifndef GTAP_MS_KEEP_GLOBAL
#define GTAP_MS_KEEP_GLOBAL 1   // 0: 1.40 ms, 1: 1.38 ms at 2^24
#endif
constexpr uint32_t kGlobalAssistMin = GTAP_MS_GLOBAL_MIN;
constexpr uint32_t kGChunk = GTAP_MS_GCHUNK;
// chunk c of an n-key merge: output range [c * kGChunk, min(n, (c + 1) * kGChunk)) (uniform chunks; a
// tail of shorter chunks measured slower: 1024 / 2048-key tails 1.51 / 1.47 ms vs 1.45 at 2^24)
#ifndef GTAP_MS_GCH_TOP
#define GTAP_MS_GCH_TOP 2   // 0 / 2 / 4 / 8: 1.312 / 1.306 / 1.310 / 1.319 ms at 2^24; merges of >= n_array / GTAP_MS_GCH_TOP keys: one chunk per warp share (0: off)
#endif
__device__ __forceinline__ uint32_t gch_count(uint32_t n, uint32_t n_all) {
    uint32_t c = (n + kGChunk - 1u) / kGChunk;
#if GTAP_MS_GCH_TOP
    // the top levels' merges run (nearly) alone on the GPU: a merge of n of the array's n_all keys is cut into its
    // share n W / n_all of the grid's W warps (one chunk per warp, 2^24 keys: 2368 chunks of ~7085 keys), so the
    // fixed cost of a chunk (split search, ring fill, store drain: ~10 us) is paid once per warp and level
    // instead of in 1.73 rounds of 4096-key chunks
    const uint32_t W = gridDim.x * (blockDim.x >> 5);
    if ((unsigned long long)n * GTAP_MS_GCH_TOP >= n_all) {
        const uint32_t cw = (uint32_t)(((unsigned long long)n * W + n_all - 1u) / n_all);
        c = max(1u, min(c, cw));
    }
#endif
    (void)n_all;
    return c;
}
// chunk c of the nch chunks of an n-key merge: the kGChunk grid when nch = ceil(n / kGChunk), else the output
// range [c n / nch, (c + 1) n / nch), inner bounds rounded down to a multiple of 4 (16-B aligned bulk stores)
__device__ __forceinline__ uint2 gch_range(uint32_t n, uint32_t c, uint32_t nch) {
    if (nch == (n + kGChunk - 1u) / kGChunk) return make_uint2(c * kGChunk, min(n, c * kGChunk + kGChunk));
    const uint32_t o0 = c == 0u ? 0u : (uint32_t)(((unsigned long long)c * n / nch) & ~3ull);
    const uint32_t o1 = c + 1u >= nch ? n : (uint32_t)(((unsigned long long)(c + 1u) * n / nch) & ~3ull);
    return make_uint2(o0, o1);
}
struct __align__(128) GSlot {
    uint32_t state, next, done, nchunks;
    uint32_t l, m, r, depth;
    uint32_t pad[24];
};
struct GBoard {
    uint32_t open;                               // slots in state 2
    uint32_t hint;                               // last slot opened
    uint32_t pad[30];
    uint32_t bits[kGSlots / 32];                 // slots with unclaimed chunks (set at open, cleared by the last claim)
    GSlot slot[kGSlots];
};

// merges up to this many keys run as one bitonic network when the bulk-copy core is available (larger ones:
// the core); without it, up to kBitonicMax
#ifndef GTAP_MS_BITONIC_MAX
#define GTAP_MS_BITONIC_MAX 512
#endif
constexpr uint32_t kMsBitonicMax = GTAP_MS_BITONIC_MAX;

#ifndef GTAP_MS_WARP_MINB
#define GTAP_MS_WARP_MINB 4
#endif

struct MsArgs {
    int32_t* keys;
    int32_t* scratch;
    uint32_t cutoff;
    uint32_t n;         // array length (TMA path needs n % 4 == 0 and 16-B aligned buffers)
    uint32_t mode;      // GTAP_MERGE_THREAD (0) or GTAP_MERGE_WARP (1)
    uint32_t bulk;      // 1: n % 4 == 0 and 16-B aligned buffers -> tiled merges by the bulk-copy core (wm3)
    GBoard* gb;         // GPU-wide assist board (table-owned, reset before each run)
};

// MODE: GTAP_MERGE_THREAD (0, one-lane bodies, TMA merge slot) or GTAP_MERGE_WARP (1, warp assist)
template <uint32_t MODE>
struct MergesortTable {
    static constexpr uint32_t kKind = GTAP_WORKER_THREAD;
    static constexpr int kMaxChildren = 2;
    static constexpr bool kTaskwait = true;
    static constexpr uint32_t kNumFn = 1;
    static constexpr bool kJoinReduceAdd = false;  // see TaskRec
    // placement hint: subtrees whose merges take the TMA path are spread over warps (never two
    // in one warp's kept set, where they would share issue slots and the block's merge slot)
    static constexpr bool kHasHeavy = true;
#ifndef GTAP_MS_HEAVY_MIN
#define GTAP_MS_HEAVY_MIN 8192   // warp mode placement hint (4096 / 8192 / 16384 / 32768: 1.255 / 1.26 / 1.31 / 1.31 ms)
#endif
    static constexpr uint32_t kHeavyMin = MODE == 1u ? GTAP_MS_HEAVY_MIN : kTmaMin;
    __device__ __forceinline__ static bool heavy(uint32_t, const uint32_t* d) { return d[1] - d[0] >= kHeavyMin; }
    __device__ __forceinline__ static bool heavy_parent(uint32_t, const uint32_t* d) {
#if GTAP_MS_KEEP_GLOBAL
        // a resumed parent whose merge goes to the GPU-wide board stays in the kept set: every idle warp
        // helps that merge anyway, and a push + publish + reclaim would add round trips to the top levels'
        // critical path (join -> slot open)
        if (MODE == 1u && 2u * (d[1] - d[0]) >= kGlobalAssistMin) return false;
#endif
        return 2u * (d[1] - d[0]) >= kHeavyMin;
    }
    static constexpr int kMaxThreads = 128;                    // __launch_bounds__
    static constexpr int kMinBlocks = MODE == 1u ? GTAP_MS_WARP_MINB : 4;
    static constexpr bool kAssist = MODE == 1u;                // leaf and merge bodies: warp assist
    static constexpr bool kStatsSmem = true;   // scheduler statistics in smem: frees 24 registers (no spills at 128)
    static constexpr int kFreeStack = 0;   // own free stack off: measured 2-3 % slower here (few live records, smem-heavy blocks)
#ifndef GTAP_MS_ASSIST_MIN
#define GTAP_MS_ASSIST_MIN 0
#endif
    static constexpr uint32_t kAssistMin = GTAP_MS_ASSIST_MIN;
    using Args = MsArgs;
    // all 32 lanes: stable merge of src[a0, m) and src[b0, r) into dst[o0, ...) by this warp -- the bulk-copy
    // core (wm3, warp_merge.cuh) when the arrays allow 16-B bulk copies, else the cp.async bitonic tiles
    __device__ __forceinline__ static void merge_tiles(const Args& a, const int32_t* src, int32_t* dst, uint32_t a0,
                                                       uint32_t m, uint32_t b0, uint32_t r, uint32_t o0, uint32_t lane,
                                                       WarpAssistHolder* H) {
        const uint32_t warp = threadIdx.x >> 5;
        if (a.bulk) wm3::merge(src, dst, a0, m, b0, r, o0, a.n, lane, H->wtiles(warp));
        else warp_merge(src, dst, a0, m, b0, r, o0, lane, H->tiles(warp));
    }
    // warp assist: ap = {l, r, depth}; all 32 lanes
    __device__ __forceinline__ static bool assist(const Args& a, const uint32_t (&ap)[kDataWords], uint32_t lane,
                                                  WarpAssistHolder* H) {
        static_assert(kMaxThreads / 32 <= kMsWarps, "one WarpTiles per warp");
        const uint32_t l = ap[0], r = ap[1], depth = ap[2];
        MS_T0;
        if (ap[3] == 1u) {  // sequential_sort of a leaf, by the warp
            warp_leaf_sort(a.keys, buf(a, depth), l, r, lane);
            MS_TRACE_LANE0(r - l, l, 2u);
            return true;
        }
        const uint32_t m = l + (r - l) / 2u;
        if (r - l <= (a.bulk ? kMsBitonicMax : kBitonicMax)) {
            const int32_t* src = buf(a, depth + 1u);
            warp_merge_small(src + l, m - l, src + m, r - m, buf(a, depth) + l, lane);
            MS_TRACE_LANE0(r - l, l, 3u);
            return true;
        }
        if (r - l >= kGlobalAssistMin && a.gb != nullptr && global_assist(a, l, m, r, depth, lane, H)) {
            MS_TRACE_LANE0(r - l, l, 5u);
            return true;
        }
        if (r - l >= kBlockAssistMin) {
            // block assist: open the board, merge chunks alongside the block's other warps (they
            // join at the top of their scheduler loops), wait until every chunk is done
            volatile WarpAssistHolder::Board& B = H->board;
            uint32_t got = 0;
            if (lane == 0) got = (atomicCAS(&H->board.state, 0u, 1u) == 0u) ? 1u : 0u;
            if (__shfl_sync(0xffffffffu, got, 0)) {
                const uint32_t nch = (r - l + kChunk - 1u) / kChunk;
                if (lane == 0) {
                    B.l = l; B.m = m; B.r = r; B.depth = depth; B.nchunks = nch; B.done = 0u;
                    __threadfence_block();
                    atomicExch(&H->board.next, 0u);   // claims from here on see the parameters above
                    __threadfence_block();
                    B.state = 2u;
                }
                __syncwarp();
                help_chunks(a, H, lane);
                if (lane == 0) {
                    while (B.done < nch) __nanosleep(128);
                    atomicExch(&H->board.next, 0x80000000u);  // late claims see a closed board
                    __threadfence_block();
                    B.state = 0u;
                }
                __syncwarp();
                __threadfence();  // helpers fenced their stores before counting; order them before our release
                __syncwarp();
                MS_TRACE_LANE0(r - l, l, 4u);
                return true;
            }
        }
        merge_tiles(a, buf(a, depth + 1u), buf(a, depth), l, m, m, r, l, lane, H);
        MS_TRACE_LANE0(r - l, l, 3u);
        return true;
    }

    // claim and merge chunks of the block's open board until none is left (all 32 lanes)
    __device__ __noinline__ static void help_chunks(const Args& a, WarpAssistHolder* H, uint32_t lane) {
        volatile WarpAssistHolder::Board& B = H->board;
        while (true) {
            uint32_t c = 0;
            if (lane == 0) c = atomicAdd(&H->board.next, 1u);
            c = __shfl_sync(0xffffffffu, c, 0);
            __threadfence_block();
            const uint32_t nch = B.nchunks;                // read after the claim (see assist)
            if (c >= nch) break;
            const uint32_t l = B.l, m = B.m, r = B.r, depth = B.depth;
            const int32_t* src = buf(a, depth + 1u);
            const uint32_t n = r - l, o0 = c * kChunk, o1 = min(n, o0 + kChunk);
            MS_T0;
            const uint2 sp = warp_split2(src, l, m, r, o0, o1, lane);
            const uint32_t i0 = sp.x, i1 = sp.y;
            merge_tiles(a, src, buf(a, depth), l + i0, l + i1, m + (o0 - i0), m + (o1 - i1), l + o0, lane, H);
            if (lane == 0) atomicAdd(&H->board.done, 1u);  // warp_merge fenced the chunk's stores
            MS_TRACE_LANE0(o1 - o0, l + o0, 7u);
        }
    }

    // claim and merge chunks of global slot S until none is left (all 32 lanes)
    __device__ __noinline__ static void gchunks(const Args& a, GSlot* S, uint32_t lane, WarpAssistHolder* H) {
        using namespace dev;
        const uint32_t si = (uint32_t)(S - a.gb->slot);
        while (true) {
            uint32_t c = 0;
            // the acquire claim orders the parameter loads after it (the requester fenced them
            // before next = 0); nchunks and {l, m, r, depth} are then read in one round trip
            uint32_t nch = 0;
            uint4 prm = make_uint4(0u, 0u, 0u, 0u);
            if (lane == 0) {
                c = atom_add_acquire(&S->next, 1u);
                nch = ld_relaxed(&S->nchunks);
                prm = ld_relaxed_v4(&S->l);
            }
            c = __shfl_sync(0xffffffffu, c, 0);
            nch = __shfl_sync(0xffffffffu, nch, 0);   // read after the claim (see GBoard)
            if (c >= nch) break;
            if (c == nch - 1u && lane == 0) atomicAnd(&a.gb->bits[si >> 5], ~(1u << (si & 31u)));  // all claimed
            const uint32_t l = __shfl_sync(0xffffffffu, prm.x, 0), m = __shfl_sync(0xffffffffu, prm.y, 0),
                           r = __shfl_sync(0xffffffffu, prm.z, 0), depth = __shfl_sync(0xffffffffu, prm.w, 0);
            const int32_t* src = buf(a, depth + 1u);
            const uint2 orng = gch_range(r - l, c, nch);
            const uint32_t o0 = orng.x, o1 = orng.y;
            MS_T0;
            const uint2 sp = warp_split2(src, l, m, r, o0, o1, lane);
            MS_TRACE_LANE0(o1 - o0, l + o0, 8u);   // trace build: the split search alone (kind 8)
            const uint32_t i0 = sp.x, i1 = sp.y;
            merge_tiles(a, src, buf(a, depth), l + i0, l + i1, m + (o0 - i0), m + (o1 - i1), l + o0, lane, H);
            if (lane == 0) atom_add_relaxed(&S->done, 1u);   // warp_merge fenced the chunk's stores
            MS_TRACE_LANE0(o1 - o0, l + o0, 6u);
        }
    }

    // find an open global slot with unclaimed chunks and work on it; false if none (all 32 lanes)
    __device__ __noinline__ static bool help_global_once(const Args& a, uint32_t lane, WarpAssistHolder* H) {
        using namespace dev;
        GBoard* gb = a.gb;
        uint32_t open = 0, hint = 0;
        if (lane == 0) { open = ld_relaxed(&gb->open); hint = ld_relaxed(&gb->hint); }
        if (__shfl_sync(0xffffffffu, open, 0) == 0u) return false;
        hint = __shfl_sync(0xffffffffu, hint, 0);
        static_assert(kGSlots / 32 == 32, "one bitmap word per lane");
        // lane k reads bitmap word (k + rot): open slots with unclaimed chunks; rotate by the hint so
        // helpers spread over the open slots
        const uint32_t wi = (lane + (hint >> 5)) & 31u;
        const uint32_t word = ld_relaxed(&gb->bits[wi]);
        const uint32_t bal = __ballot_sync(0xffffffffu, word != 0u);
        if (bal == 0u) return false;
        const uint32_t src_lane = (uint32_t)__ffs(bal) - 1u;
        const uint32_t wsel = __shfl_sync(0xffffffffu, word, src_lane);
        const uint32_t wix = __shfl_sync(0xffffffffu, wi, src_lane);
        // a set bit chosen by a per-warp rotation
        const uint32_t rot = (hint + (blockIdx.x * 4u + (threadIdx.x >> 5)) * 7u) & 31u;
        const uint32_t rotw = (wsel >> rot) | (rot ? (wsel << (32u - rot)) : 0u);
        const uint32_t bit = ((uint32_t)__ffs(rotw) - 1u + rot) & 31u;
        gchunks(a, gb->slot + wix * 32u + bit, lane, H);
        return true;
    }

    // requester side (all 32 lanes); false if no slot was free (the caller merges another way)
    __device__ __noinline__ static bool global_assist(const Args& a, uint32_t l, uint32_t m, uint32_t r,
                                                      uint32_t depth, uint32_t lane, WarpAssistHolder* H) {
        using namespace dev;
        GBoard* gb = a.gb;
        uint32_t sidx = kNone;
        const uint32_t h = (l >> 15) * 0x9E3779B1u;
        for (uint32_t base = 0; base < 128u && sidx == kNone; base += 32u) {
            const uint32_t cand = (h + base + lane) & (kGSlots - 1u);
            uint32_t bal = __ballot_sync(0xffffffffu, ld_relaxed(&gb->slot[cand].state) == 0u);
            while (bal) {
                const uint32_t k = (uint32_t)__ffs(bal) - 1u;
                bal &= bal - 1u;
                uint32_t ok = 0;
                if (lane == k) ok = atom_cas_relaxed(&gb->slot[cand].state, 0u, 1u) == 0u ? 1u : 0u;
                if (__shfl_sync(0xffffffffu, ok, k)) { sidx = __shfl_sync(0xffffffffu, cand, k); break; }
            }
        }
        if (sidx == kNone) return false;
        GSlot* S = gb->slot + sidx;
        const uint32_t nch = gch_count(r - l, a.n);
        if (lane == 0) {
            st_relaxed(&S->l, l); st_relaxed(&S->m, m); st_relaxed(&S->r, r); st_relaxed(&S->depth, depth);
            st_relaxed(&S->nchunks, nch); st_relaxed(&S->done, 0u);
            // the release RMW publishes the parameters to every claim (an acquire RMW on next) that follows it;
            // the release store orders the reset before the slot shows as open
            atom_exch_release(&S->next, 0u);
            st_release(&S->state, 2u);
            atomicOr(&gb->bits[sidx >> 5], 1u << (sidx & 31u));
            red_add_relaxed(&gb->open, 1u);
            st_relaxed(&gb->hint, sidx);
        }
        __syncwarp();
        gchunks(a, S, lane, H);
        while (true) {   // wait for the helpers (helping other open slots meanwhile measured slower: 1.38 vs
                         // 1.32 ms, the requester then closes its own slot late)
            uint32_t dn = 0;
            if (lane == 0) dn = ld_relaxed(&S->done);
            if (__shfl_sync(0xffffffffu, dn, 0) >= nch) break;
            if (lane == 0) nanosleep(256);
            __syncwarp();
        }
        if (lane == 0) {
            atom_exch_relaxed(&S->next, 0x80000000u);
            red_add_relaxed(&gb->open, 0xFFFFFFFFu);
            st_release(&S->state, 0u);   // orders the close (late claims fail) before the slot shows as free
        }
        __syncwarp();
        __threadfence();
        __syncwarp();
        return true;
    }

    // scheduler hook: idle warps poll the board's open-slot count while probing steal victims (sched_thread.cuh
    // idle_word_of), so a slot opened during a steal round is seen one round trip later
    static constexpr bool kIdleWord = MODE == 1u;
    __device__ __forceinline__ static const uint32_t* idle_word(const Args& a) {
        return a.gb ? &a.gb->open : nullptr;
    }
    // scheduler hook, idle path (all 32 lanes): help an open GPU-wide assist
    __device__ __forceinline__ static bool help_idle(const Args& a, uint32_t lane, WarpAssistHolder* H) {
        if (a.gb == nullptr) return false;
        return help_global_once(a, lane, H);
    }

    // scheduler hook, top of every cycle (all 32 lanes): join an open board of this block
    __device__ __forceinline__ static void help(const Args& a, uint32_t lane, WarpAssistHolder* H) {
        if (reinterpret_cast<volatile uint32_t&>(H->board.state) == 2u)
            help_chunks(a, H, lane);
    }
    using BlockExtra = std::conditional_t<MODE == 1u, WarpAssistHolder, MergeSlotHolder>;
    __device__ __forceinline__ static void block_init(BlockExtra* H) {
        if constexpr (MODE == 1u) {
            H->board.state = 0;
            H->board.next = 0x80000000u;
            H->board.nchunks = 0;
            H->board.done = 0;
            for (uint32_t w = 0; w < (uint32_t)kMsWarps; ++w) wm3::init_one(&H->aux[w]);
        } else {
            MergeSlot* S = H->slot();
            for (int k = 0; k < 2 * kChains; ++k) {
                for (int j = 0; j < 2; ++j) tma::mbar_init(&S->mbar[k][j], 1);
                S->par[k] = 0;
            }
            H->busy = 0;
            tma::fence_smem();
        }
    }

    __device__ __forceinline__ static int32_t* buf(const Args& a, uint32_t depth) {
        return (depth & 1u) ? a.scratch : a.keys;
    }

    // sequential_sort: insertion sort of src[l, r) into dst[l, r).
    __device__ __noinline__ static void leaf_sort(const int32_t* __restrict__ src, int32_t* __restrict__ dst,
                                                  uint32_t l, uint32_t r) {
        int32_t t[kMsMaxCutoff];
        const uint32_t n = r - l;
        for (uint32_t i = 0; i < n; ++i) {
            const int32_t v = src[l + i];
            int32_t j = (int32_t)i - 1;
            while (j >= 0 && t[j] > v) {
                t[j + 1] = t[j];
                --j;
            }
            t[j + 1] = v;
        }
        for (uint32_t i = 0; i < n; ++i) dst[l + i] = t[i];
    }

    // merge: stable merge of src[l, m) and src[m, r) into dst[l, r).
    __device__ __forceinline__ static bool merge(const Args& a, const int32_t* src, int32_t* dst, uint32_t l,
                                                 uint32_t m, uint32_t r, MergeSlotHolder* S) {
        const bool tma_ok = (r - l) >= kTmaMin && (a.n & 3u) == 0u &&
                            ((reinterpret_cast<uintptr_t>(a.keys) | reinterpret_cast<uintptr_t>(a.scratch)) & 15u) == 0u;
        MS_T0;
        bool ok = true;
        uint32_t used = 0;
        if (tma_ok && atomicCAS(&S->busy, 0u, 1u) == 0u) {
            ok = ms_merge_tma(src, dst, l, m, r, a.n, S);
            atomicExch(&S->busy, 0u);
            used = 1;
        } else {
            ms_merge(src, dst, l, m, r);
        }
        MS_TRACE(r - l, l, used);
        (void)used;
        return ok;
    }

    __device__ __forceinline__ static void exec(const Args& a, uint32_t fn, uint32_t state,
                                                const uint32_t (&d)[kDataWords], TOut<kMaxChildren>& o,
                                                BlockExtra* S) {
        if (fn != 0u) { o.bad_state(); return; }
        const uint32_t l = d[0], r = d[1], depth = d[2];
        switch (state) {
            case 0:
                if (r - l <= a.cutoff) {
                    if constexpr (MODE == 1u) {               // by the whole warp (bitonic, registers)
                        o.request_assist(l, r, depth, 1u);
                    } else {
                        MS_T0;
                        leaf_sort(a.keys, buf(a, depth), l, r);
                        MS_TRACE(r - l, l, 2u);
                    }
                    o.finish_void();
                    return;
                } else {
                    const uint32_t m = l + (r - l) / 2u;
                    o.spawn(0, 0u, l, m, depth + 1u);         // fork [l, m)
                    o.spawn(1, 0u, m, r, depth + 1u);         // fork [m, r)
                    o.suspend(1);                             // join
                    return;
                }
            case 1: {
                const uint32_t m = l + (r - l) / 2u;
                if constexpr (MODE == 1u) {
                    if (r - l >= kAssistMin) {                // merge(l, m, r) by the whole warp
                        o.request_assist(l, r, depth, 0u);
                        o.finish_void();
                        return;
                    }
                    ms_merge(buf(a, depth + 1u), buf(a, depth), l, m, r);
                } else {
                    if (!merge(a, buf(a, depth + 1u), buf(a, depth), l, m, r, S)) { o.bad_state(); return; }
                }
                o.finish_void();
                return;
            }
            default:
                o.bad_state();
        }
    }
};

// a root {l, r} must lie inside keys[0, n): the kernel reads and writes [l, r) of keys and scratch
static int validate_ms(const gtap_task_table* t, uint32_t fn, const uint32_t* d) {
    MsArgs a;
    std::memcpy(&a, t->args, sizeof(a));
    return (fn == 0u && d[0] <= d[1] && d[1] <= a.n && d[2] == 0u) ? 0 : -1;
}

}  // namespace gtap

extern "C" const gtap_task_table* gtap_table_mergesort_ex(int32_t* keys, int32_t* scratch, uint64_t n, int32_t cutoff,
                                                         uint32_t merge_mode) {
    if (((!keys || !scratch) && n > 0) || cutoff < 1 || cutoff > gtap::kMsMaxCutoff || n >= (1ull << 31)) return nullptr;
    if (merge_mode > 1u) return nullptr;
    gtap::GBoard* gb = nullptr;
    if (merge_mode == 1u && cudaMalloc(&gb, sizeof(gtap::GBoard)) != cudaSuccess) return nullptr;
    const uint32_t bulk = (n % 4u == 0u) && (((uintptr_t)keys | (uintptr_t)scratch) & 15u) == 0u ? 1u : 0u;
    gtap::MsArgs a{keys, scratch, (uint32_t)cutoff, (uint32_t)n, merge_mode, bulk, gb};
    gtap_task_table* t = merge_mode == 1u
        ? gtap::make_table<gtap::MergesortTable<1u>>("mergesort_warp", a, &gtap::validate_ms)
        : gtap::make_table<gtap::MergesortTable<0u>>("mergesort", a, &gtap::validate_ms);
    if (!t) { cudaFree(gb); return nullptr; }
    if (gb) {
        t->dev_scratch = gb;
        t->prepare = [](const gtap_task_table* tt, cudaStream_t s) {
            return gtap::zero_async(tt->dev_scratch, sizeof(gtap::GBoard), s);
        };
    }
    return t;
}

extern "C" const gtap_task_table* gtap_table_mergesort(int32_t* keys, int32_t* scratch, uint64_t n, int32_t cutoff) {
    return gtap_table_mergesort_ex(keys, scratch, n, cutoff, 1u);
}
