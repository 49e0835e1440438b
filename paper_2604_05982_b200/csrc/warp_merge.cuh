// warp_merge.cuh -- the warp-level merge core of the warp-assisted mergesort bodies (B200 design,
// DESIGN.md "Warp assist"; the paper's merge, P:69 / P:163, is a sequential two-pointer merge: this
// produces exactly its output, the stable merge, ties from the left run first).
//
// One warp merges src[a0, m) and src[b0, r) into dst[o0, ...) in tiles of T = 32 * VT outputs:
//   * each input run streams through a per-warp shared-memory ring of NS chunks of C keys, filled by
//     1-D bulk copies (cp.async.bulk, one lane issues, one mbarrier per ring slot): up to NS * C keys
//     of look-ahead per run for a handful of instructions per KB;
//   * per tile, lane k finds the start of its VT outputs [k * VT, k * VT + VT) by a stable merge-path
//     binary search over the two resident windows, then merges them serially out of shared memory
//     (one compare and one select-addressed shared load per output, no divergence; interior tiles,
//     where both windows hold T keys, need no bounds checks) into a per-warp output buffer (VT odd:
//     the lanes' stores are VT words apart, conflict-free);
//   * the buffer leaves by ONE 1-D bulk store per tile (cp.async.bulk.global.shared::cta); tiles are
//     cut so that every tile after the first starts 16-B aligned in dst, and the at most 3 + 3 keys at
//     the ends of the output range go by plain stores.
// The chunks a tile reads are waited for (mbarrier parity per slot, persistent across calls in
// WM3Tiles::par) before the tile; every chunk issued is waited for before the call returns, and the
// bulk stores are complete (and fenced to the generic proxy) before it returns.
// Requires 16-B aligned src / dst arrays whose length n4 is a multiple of 4 (bulk granularity);
// chunks are C-key (2 KB) aligned in the array and may read keys outside [a0, m) / [b0, r) (never used).
#pragma once
#include <climits>
#include <cstdint>

namespace gtap {
namespace wm3 {

#ifndef GTAP_MS_VT
#define GTAP_MS_VT 13   // 9 / 11 / 13 / 15 / 17 / 19: 1.337 / 1.29 / 1.26 / 1.29 / 1.30 / 1.30 ms at 2^24
#endif
constexpr int VT = GTAP_MS_VT;                // outputs per lane per tile (odd: conflict-free output buffer)
constexpr int T = 32 * VT;                    // outputs per tile (a multiple of 4)
#ifndef GTAP_MS_C
#define GTAP_MS_C 512   // 256 x 4 / 512 x 2 / 128 x 8 (keys per chunk x chunks per ring): 1.26 / 1.24 / 1.31-1.34 ms
#endif
constexpr int C = GTAP_MS_C;                  // keys per bulk chunk (2 KB)
#ifndef GTAP_MS_NS
#define GTAP_MS_NS 2
#endif
constexpr int NS = GTAP_MS_NS;                // chunks per ring
constexpr int R = C * NS;                     // keys per ring
static_assert((VT & 1) == 1, "VT odd");
static_assert(T + C - 1 <= R, "a tile's window (T keys at any offset) must fit NS chunks");
static_assert((R & (R - 1)) == 0, "ring length: power of two");

// per warp: the two rings (placed R * 4-aligned: a ring byte address wraps with one LOP3) ...
struct WM3Rings {
    int32_t ring[2][R];                       // A ring, B ring (slot s of a ring = keys [s * C, s * C + C))
};
// ... and the rest
struct __align__(16) WM3Aux {
    int32_t out[T + 8];                       // output staging; global key g of a tile sits at (g & 3) + (g - out)
    unsigned long long mbar[2][NS];
    uint32_t par[2];                          // completed-phase parity bit per slot (uniform, persistent)
};
struct WM3Tiles {                             // what a warp passes around
    WM3Rings* rings;
    WM3Aux* aux;
};

__device__ __forceinline__ uint32_t smaddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int32_t lds(uint32_t a) {
    int32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts(uint32_t a, int32_t v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t mb, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}"
        : "=r"(ok) : "r"(mb), "r"(parity) : "memory");
    return ok != 0;
}

// one-time setup of a warp's barriers by one thread (a block barrier or __syncwarp must follow)
__device__ __forceinline__ void init_one(WM3Aux* S) {
    for (int k = 0; k < 2; ++k) {
        for (int s = 0; s < NS; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smaddr(&S->mbar[k][s])) : "memory");
        S->par[k] = 0u;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// the same by lane 0 of the warp (all lanes call)
__device__ __forceinline__ void init(WM3Aux* S, uint32_t lane) {
    if (lane == 0) {
        for (int k = 0; k < 2; ++k) {
            for (int s = 0; s < NS; ++s)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smaddr(&S->mbar[k][s])) : "memory");
            S->par[k] = 0u;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
}

// streaming state of one input run (uniform across the warp)
struct Run {
    const int32_t* g;     // array base
    uint32_t n4;          // array length (multiple of 4)
    uint32_t issued;      // next chunk index to issue
    uint32_t waited;      // next chunk index to wait for
    uint32_t last;        // last chunk index of the run
    uint32_t ring;        // smem byte address of the ring (R * 4-aligned)
    uint32_t mb;          // smem byte address of the slot mbarriers
    uint32_t par;         // slot parity bits
};

__device__ __forceinline__ void issue(Run& s, uint32_t lane) {
    const uint32_t c = s.issued++;
    if (lane == 0) {
        const uint32_t k0 = c * (uint32_t)C;
        const uint32_t bytes = min((uint32_t)C, s.n4 - k0) * 4u;
        const uint32_t slot = c % (uint32_t)NS;
        const uint32_t mb = s.mb + 8u * slot;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(s.ring + slot * (uint32_t)(C * 4)), "l"(s.g + k0), "r"(bytes), "r"(mb) : "memory");
    }
}
__device__ __forceinline__ void wait_one(Run& s) {
    const uint32_t slot = s.waited % (uint32_t)NS;
    const uint32_t ph = (s.par >> slot) & 1u;
    while (!mbar_try(s.mb + 8u * slot, ph)) {}
    s.par ^= 1u << slot;
    ++s.waited;
}
// issue every chunk the ring has room for: chunk c may reuse its slot once the run head `pos` left chunk c - NS
__device__ __forceinline__ void fill(Run& s, uint32_t pos, uint32_t lane) {
    const uint32_t lim = pos / (uint32_t)C + (uint32_t)NS;
    while (s.issued <= s.last && s.issued < lim) issue(s, lane);
}
__device__ __forceinline__ void start(Run& s, const int32_t* g, uint32_t n4, uint32_t lo, uint32_t hi, uint32_t ring,
                                      uint32_t mb, uint32_t par, uint32_t lane) {
    s.g = g; s.n4 = n4; s.ring = ring; s.mb = mb; s.par = par;
    s.issued = s.waited = lo / (uint32_t)C;
    s.last = hi > lo ? (hi - 1u) / (uint32_t)C : s.issued;
    if (hi <= lo) { s.issued = s.waited = s.last + 1u; return; }   // empty run: nothing to load
    fill(s, lo, lane);
}
// the chunks holding keys [.., upto) have landed
__device__ __forceinline__ void need(Run& s, uint32_t upto) {
    if (upto == 0u) return;
    const uint32_t lastc = (upto - 1u) / (uint32_t)C;
    while (s.waited <= lastc && s.waited < s.issued) wait_one(s);
}
constexpr uint32_t kMask = (uint32_t)(R * 4 - 1);
constexpr int kSearchIters = 32 - __builtin_clz((unsigned)T);   // ceil(log2(T + 1)) halvings cover [0, T]
__device__ __forceinline__ uint32_t addr(uint32_t ring, uint32_t key) { return ring + ((key * 4u) & kMask); }
// advance a ring byte address by one key, wrapping inside its ring: ((t + 4) & mask) | (t & ~mask)
__device__ __forceinline__ uint32_t next(uint32_t t) { return ((t + 4u) & kMask) | (t & ~kMask); }

// all 32 lanes: stable merge of src[a0, m) and src[b0, r) into dst[o0, o0 + (m - a0) + (r - b0));
// n4: length of the array src points into (multiple of 4, 16-B aligned base); dst 16-B aligned
__device__ __noinline__ void merge(const int32_t* __restrict__ src, int32_t* __restrict__ dst, uint32_t a0,
                                   uint32_t m, uint32_t b0, uint32_t r, uint32_t o0, uint32_t n4, uint32_t lane,
                                   WM3Tiles W) {
    asm volatile("fence.proxy.async.global;" ::: "memory");   // producers' generic stores -> bulk-copy reads
    WM3Aux* S = W.aux;
    Run A, B;
    const uint32_t ringA = smaddr(&W.rings->ring[0][0]), ringB = smaddr(&W.rings->ring[1][0]);
    start(A, src, n4, a0, m, ringA, smaddr(&S->mbar[0][0]), S->par[0], lane);
    start(B, src, n4, b0, r, ringB, smaddr(&S->mbar[1][0]), S->par[1], lane);
    const uint32_t ob = smaddr(&S->out[0]);
    uint32_t pa = a0, pb = b0, out = o0;
    const uint32_t oend = o0 + (m - a0) + (r - b0);
    bool pending_store = false;
    while (out < oend) {
        // tile: up to T outputs, the first one shortened so that every later tile starts 16-B aligned
        const uint32_t tile = min((uint32_t)T - (out & 3u), oend - out);
        const uint32_t na = min(tile, m - pa), nb = min(tile, r - pb);
        need(A, pa + na);
        need(B, pb + nb);
        __syncwarp();
        // merge-path split of this lane's diagonal d: the smallest i in [lo, hi] with !(A[i] <= B[d-1-i]);
        // a fixed number of branch-free halvings (ring byte offsets; the rings are R * 4-aligned)
        const uint32_t d = min(lane * (uint32_t)VT, tile);
        uint32_t lo = d > nb ? d - nb : 0u, hi = min(d, na);
        {
            const uint32_t aoff = pa * 4u, boff = (pb + d - 1u) * 4u;
#pragma unroll
            for (int it = 0; it < kSearchIters; ++it) {
                const uint32_t mid = (lo + hi) >> 1;
                const int32_t x = lds(ringA | ((aoff + mid * 4u) & kMask));
                const int32_t y = lds(ringB | ((boff - mid * 4u) & kMask));
                const bool open = lo < hi, le = x <= y;
                lo = (open && le) ? mid + 1u : lo;
                hi = (open && !le) ? mid : hi;
            }
        }
        uint32_t ta = addr(ringA, pa + lo), tb = addr(ringB, pb + d - lo);
        int32_t va = lds(ta), vb = lds(tb);
        // the previous tile's bulk store must have read the buffer before it is overwritten
        if (pending_store) {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
        }
        const uint32_t obase = ob + 4u * ((out & 3u) + d);
        if (tile == (uint32_t)T && na == (uint32_t)T && nb == (uint32_t)T) {
            // interior tile: ai + bi < T keeps both heads inside their windows; no bounds checks
#pragma unroll
            for (int v = 0; v < VT; ++v) {
                const bool takeA = va <= vb;
                sts(obase + 4u * (uint32_t)v, takeA ? va : vb);
                const uint32_t t = next(takeA ? ta : tb);
                ta = takeA ? t : ta;
                tb = takeA ? tb : t;
                const int32_t x = lds(t);
                va = takeA ? x : va;
                vb = takeA ? vb : x;
            }
        } else {
            uint32_t ai = lo, bi = d - lo;
            const uint32_t cnt = min((uint32_t)VT, tile - d);
#pragma unroll
            for (int v = 0; v < VT; ++v) {
                if ((uint32_t)v < cnt) {
                    const bool takeA = bi >= nb || (ai < na && va <= vb);
                    sts(obase + 4u * (uint32_t)v, takeA ? va : vb);
                    ai += takeA ? 1u : 0u;
                    bi += takeA ? 0u : 1u;
                    const uint32_t t = next(takeA ? ta : tb);   // may point past the run: the value is unused
                    ta = takeA ? t : ta;
                    tb = takeA ? tb : t;
                    const int32_t x = lds(t);
                    va = takeA ? x : va;
                    vb = takeA ? vb : x;
                }
            }
        }
        // A keys consumed by the tile: the A head of the lane holding the tile's last output (its offset
        // from pa is < T < R, so the ring position determines it)
        const uint32_t myA = ((ta - ringA) >> 2) & (uint32_t)(R - 1);
        const uint32_t endA = __shfl_sync(0xffffffffu, myA, (tile - 1u) / (uint32_t)VT);
        const uint32_t cA = (endA - pa) & (uint32_t)(R - 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // buffer writes / ring reads -> async proxy
        __syncwarp();
        // out [out, e) sits at buffer [(out & 3), (out & 3) + tile): bulk-store its 16-B aligned middle
        // [g0, g1), the < 4 keys on each side by plain stores
        const uint32_t e = out + tile;
        const uint32_t g0 = min((out + 3u) & ~3u, e), g1 = max(e & ~3u, g0);
        if (g1 > g0) {
            if (lane == 0) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + g0),
                             "r"(ob + 4u * ((out & 3u) + (g0 - out))), "r"((g1 - g0) * 4u) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            pending_store = true;
        }
        if (((out | e) & 3u) != 0u) {   // uniform: only the first / last tile of a range has unaligned ends
            if (lane < g0 - out) dst[out + lane] = lds(ob + 4u * ((out & 3u) + lane));
            else if (lane >= 4u && lane - 4u < e - g1)
                dst[g1 + lane - 4u] = lds(ob + 4u * ((out & 3u) + (g1 - out) + lane - 4u));
        }
        pa += cA;
        pb += tile - cA;
        out += tile;
        __syncwarp();
        fill(A, pa, lane);
        fill(B, pb, lane);
    }
    // drain: every issued chunk must land before its slot or the parity bits are reused
    while (A.waited < A.issued) wait_one(A);
    while (B.waited < B.issued) wait_one(B);
    if (lane == 0) {
        S->par[0] = A.par;
        S->par[1] = B.par;
        if (pending_store) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // bulk stores complete
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __threadfence();   // every lane's stores (and the completed bulk stores) before the requester's join release
    __syncwarp();
}

}  // namespace wm3
}  // namespace gtap
