// table_spmv.cu -- SpMV task table (block-level, no taskwait).
//
// The paper names SpMV as a block-cooperative workload but
// gives no listing; the task program here is reading R20:
//   spmv(lo, hi): if (nnz(lo, hi) > nnz_cut && hi - lo > 1)
//                   spawn spmv on `fanout` equal row sub-ranges   (no taskwait)
//                 else  y[i] = sum_j val[j] * x[col[j]] for i in [lo, hi),
//                       computed cooperatively by the block in fp32.
// Leaf layout (CSR-stream): the block walks the leaf's non-zeros in chunks of
// 8 x blockDim: coalesced col/val loads (streaming, evict-first) and
// independent x gathers (read-only path) land as products in shared memory,
// then warps sum each row's segment by shuffle; a row that runs past a chunk
// carries its partial sum into the next one, so heavy rows (up to 64K nnz)
// need no separate path and no row serialises on one warp.
// Payload: d[0] = lo, d[1] = hi.
#include "table_common.cuh"

namespace gtap {

struct SpmvTable {
    static constexpr uint32_t kKind = GTAP_WORKER_BLOCK;
    static constexpr int kMaxChildren = 32;
    static constexpr bool kTaskwait = false;
    static constexpr uint32_t kNumFn = 2;          // 0: spmv(lo, hi); 1: part(k, R) (a forest root)
    static constexpr bool kJoinReduceAdd = false;  // see TaskRec
#ifndef GTAP_SPMV_MINB
#define GTAP_SPMV_MINB 4
#endif
#ifndef GTAP_SPMV_MAXT
#define GTAP_SPMV_MAXT 256
#endif
    static constexpr int kMaxThreads = GTAP_SPMV_MAXT, kMinBlocks = GTAP_SPMV_MINB;  // __launch_bounds__ (prod[] holds 8 x 256)
    static constexpr int kSpawnCap = 32;
#ifndef GTAP_SPMV_PER
#define GTAP_SPMV_PER 24   // with 256-thread blocks: 6 K non-zeros per chunk (12 / 16 / 20 / 24 / 28 / 32: 0.74 / 0.71 / - / 0.69 / 0.74 / 0.73 ms at the bench shape; 20 and 28 spill)
#endif
    static constexpr int kPer = GTAP_SPMV_PER;  // non-zeros per thread per chunk
    static constexpr int kMaxBlock = 256;   // prod[] sized for blocks up to 256 threads
    static constexpr int kRp = 512;         // row_ptr entries staged per chunk (more rows: global loads)
#ifndef GTAP_SPMV_ROWS_BY_THREAD
#define GTAP_SPMV_ROWS_BY_THREAD 1
#endif
#ifndef GTAP_SPMV_SHORT
#define GTAP_SPMV_SHORT 64
#endif
    static constexpr int kShortSeg = GTAP_SPMV_SHORT;    // in-chunk row segments up to this long: one thread
    static constexpr int kLongCap = kPer * kMaxBlock / (kShortSeg + 1) + 1;  // > segments that fit a chunk
    struct Scratch {
        float prod[kPer * kMaxBlock];
        int32_t rp[kRp + 1];
        uint32_t rcur, rnext;
        float carry, carry_next;
        uint32_t nlong;
        uint32_t longr[kLongCap];
    };
    struct Args {
        const int32_t* row_ptr;
        const int32_t* col;
        const float* val;
        const float* x;
        float* y;
        uint32_t nrows;
        uint32_t nnz_cut;
        uint32_t fanout;
        uint32_t pad;
    };

    // streaming loads for the matrix (read once: do not displace x from L2), read-only path for x
    __device__ __forceinline__ static int32_t ld_col(const int32_t* p) { return __ldcs(p); }
    __device__ __forceinline__ static float ld_val(const float* p) { return __ldcs(p); }
    template <class Ctx>
    __device__ __forceinline__ static void exec_block(const Args& a, Ctx& ctx, uint32_t fn, uint32_t state,
                                                      const uint32_t (&d)[kDataWords]) {
        if (fn > 1u || state != 0u) {
            if (threadIdx.x == 0) ctx.bad_state();
            return;
        }
        uint32_t lo = d[0], hi = d[1];
        if (fn == 1u) {
            // part(k, R, r0, r1): the k-th of R row ranges of [r0, r1) (r1 = 0: all rows) balanced by
            // non-zeros (reading R20): boundary j is the first row whose start offset reaches
            // row_ptr[r0] + floor(j * nnz(r0, r1) / R); every thread runs the same search (uniform
            // loads), then the range is an ordinary spmv(lo, hi) task
            const uint32_t k = d[0], R = d[1], r0 = d[2], r1 = d[3] ? d[3] : a.nrows;
            const long long s0 = __ldg(&a.row_ptr[r0]);
            const unsigned long long nnz = (unsigned long long)(__ldg(&a.row_ptr[r1]) - s0);
            // block-parallel search: every thread probes one of blockDim points per round and
            // __syncthreads_count ranks the boundary (~log_{blockDim+1}(rows) round trips instead of
            // the ~22 of a binary search, twice per root at the start of the run)
            const uint32_t bdim = blockDim.x, tix = threadIdx.x;
            auto bound = [&](uint32_t j) -> uint32_t {
                if (j == 0u) return r0;
                if (j >= R) return r1;
                const long long target = s0 + (long long)((nnz * j) / R);
                uint32_t l = r0, h = r1;   // smallest i in [l, h] with row_ptr[i] >= target
                while (h - l > bdim) {
                    const unsigned long long w = h - l;
                    const uint32_t q = l + (uint32_t)(((unsigned long long)(tix + 1u) * w) / (bdim + 1u));
                    const uint32_t cnt = (uint32_t)__syncthreads_count((long long)__ldg(&a.row_ptr[q]) < target);
                    const uint32_t nl = cnt == 0u ? l : l + (uint32_t)(((unsigned long long)cnt * w) / (bdim + 1u)) + 1u;
                    const uint32_t nh = cnt == bdim ? h : l + (uint32_t)(((unsigned long long)(cnt + 1u) * w) / (bdim + 1u));
                    l = nl;
                    h = nh;
                }
                const uint32_t q = l + tix;
                return l + (uint32_t)__syncthreads_count(q < h && (long long)__ldg(&a.row_ptr[q]) < target);
            };
            lo = bound(k);
            hi = max(lo, bound(k + 1u));
        }
        const int32_t s = __ldg(&a.row_ptr[lo]), e = __ldg(&a.row_ptr[hi]);
        const uint32_t tid = threadIdx.x, bd = blockDim.x;
        if ((uint32_t)(e - s) > a.nnz_cut && hi - lo > 1u) {
            // split: fanout equal row ranges (no taskwait)
            const uint32_t f = min(a.fanout, hi - lo);
            if (tid < f) {
                const uint32_t n = hi - lo;
                const uint32_t b0 = lo + (uint32_t)(((unsigned long long)n * tid) / f);
                const uint32_t b1 = lo + (uint32_t)(((unsigned long long)n * (tid + 1)) / f);
                if (b1 > b0) ctx.spawn(0u, b0, b1);
            }
            if (tid == 0) ctx.finish_void();
            return;
        }
        // ---- leaf: CSR-stream over the leaf's non-zeros [s, e) in chunks of kPer * blockDim ----
        // load phase: every thread issues kPer coalesced (col, val) loads and kPer independent x
        // gathers, products to shared memory; row phase: warps sum each row's segment of the chunk
        // by shuffle; a row that continues past the chunk leaves its partial sum in `carry`
        // (so a 64K-nnz row is just a row that spans many chunks).
        auto& sc = ctx.sm.scratch;
        const uint32_t lane = tid & 31u, warp = tid >> 5, nw = bd >> 5;
        const int32_t CH = kPer * (int32_t)bd;
        if (tid == 0) { sc.rcur = lo; sc.carry = 0.f; }
        __syncthreads();
#ifdef GTAP_SPMV_PIPE
        // software pipeline: chunk c+1's (col, val) loads are issued before chunk c's row phase and
        // its x gathers right after it, so the memory latency overlaps the shared-memory reduction
        int32_t cc[kPer];
        float vv[kPer], pr[kPer];
        if (s < e) {
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int32_t idx = s + (int32_t)tid + k * (int32_t)bd;
                const bool in = idx < min(s + CH, e);
                cc[k] = ld_col(&a.col[in ? idx : s]);
                vv[k] = in ? ld_val(&a.val[idx]) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < kPer; ++k) pr[k] = vv[k] * __ldg(&a.x[cc[k]]);
        }
        for (int32_t c0 = s; c0 < e; c0 += CH) {   // uniform
            const int32_t c1 = min(c0 + CH, e);
            const uint32_t r0 = sc.rcur;
            for (uint32_t i = tid; i <= (uint32_t)kRp; i += bd)
                sc.rp[i] = (r0 + i <= hi) ? __ldg(&a.row_ptr[r0 + i]) : e;
#pragma unroll
            for (int k = 0; k < kPer; ++k) sc.prod[tid + k * bd] = pr[k];
            __syncthreads();
            const bool more = c0 + CH < e;
            if (more) {
                const int32_t n0 = c0 + CH, n1 = min(n0 + CH, e);
#pragma unroll
                for (int k = 0; k < kPer; ++k) {
                    const int32_t idx = n0 + (int32_t)tid + k * (int32_t)bd;
                    const bool in = idx < n1;
                    cc[k] = ld_col(&a.col[in ? idx : n0]);
                    vv[k] = in ? ld_val(&a.val[idx]) : 0.f;
                }
            }
#else
        for (int32_t c0 = s; c0 < e; c0 += CH) {   // uniform
            const int32_t c1 = min(c0 + CH, e);
            const uint32_t r0 = sc.rcur;
            // row_ptr[r0 .. r0 + kRp] staged with the chunk (the row phase then reads smem only)
            for (uint32_t i = tid; i <= (uint32_t)kRp; i += bd)
                sc.rp[i] = (r0 + i <= hi) ? __ldg(&a.row_ptr[r0 + i]) : e;
            int32_t cc[kPer];
            float vv[kPer];
#pragma unroll
            for (int k = 0; k < kPer; ++k) {
                const int32_t idx = c0 + (int32_t)tid + k * (int32_t)bd;
                const bool in = idx < c1;
                cc[k] = ld_col(&a.col[in ? idx : c0]);
                vv[k] = in ? ld_val(&a.val[idx]) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < kPer; ++k) sc.prod[tid + k * bd] = vv[k] * __ldg(&a.x[cc[k]]);
            __syncthreads();
#endif
            const float carry_in = sc.carry;
#if GTAP_SPMV_ROWS_BY_THREAD
            // row phase, pass 1: one thread per row of the chunk; a segment of <= kShortSeg products
            // is summed serially from shared memory (4 interleaved partial sums), longer segments are
            // listed for the warp pass. (Warp-per-row reductions left 4 warps doing ~8 short rows
            // each, one shuffle tree per row.)
            if (tid == 0) sc.nlong = 0u;
            __syncthreads();
            for (uint32_t i = tid;; i += bd) {
                const uint32_t r = r0 + i;
                if (r >= hi) break;
                const int32_t rs = i < (uint32_t)kRp ? sc.rp[i] : __ldg(&a.row_ptr[r]);
                if (rs >= c1) break;                          // rows are sorted by start
                const int32_t re = i < (uint32_t)kRp ? sc.rp[i + 1] : __ldg(&a.row_ptr[r + 1]);
                const int32_t a0 = max(rs, c0), a1 = min(re, c1);
                if (a1 - a0 > kShortSeg) {
                    const uint32_t q = atomicAdd(&sc.nlong, 1u);
                    if (q < (uint32_t)kLongCap) sc.longr[q] = r;
                    continue;
                }
                float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
                int32_t j = a0 - c0;
                const int32_t je = a1 - c0;
                for (; j + 4 <= je; j += 4) {
                    t0 += sc.prod[j]; t1 += sc.prod[j + 1]; t2 += sc.prod[j + 2]; t3 += sc.prod[j + 3];
                }
                for (; j < je; ++j) t0 += sc.prod[j];
                float t = (t0 + t1) + (t2 + t3);
                if (rs < c0) t += carry_in;                   // only r0 can have started earlier
                if (re <= c1) a.y[r] = t;
                if (re >= c1) {                               // the last row touching this chunk
                    sc.rnext = (re > c1) ? r : r + 1u;
                    sc.carry_next = (re > c1) ? t : 0.f;
                }
            }
            __syncthreads();
            // pass 2: long segments, one warp each (strided lanes + shuffle tree)
            const uint32_t nlong = sc.nlong;
            for (uint32_t q = warp; q < nlong; q += nw) {     // warp-uniform
                const uint32_t r = q < (uint32_t)kLongCap ? sc.longr[q] : 0u;
                const uint32_t i = r - r0;
                const int32_t rs = i < (uint32_t)kRp ? sc.rp[i] : __ldg(&a.row_ptr[r]);
                const int32_t re = i < (uint32_t)kRp ? sc.rp[i + 1] : __ldg(&a.row_ptr[r + 1]);
                const int32_t a0 = max(rs, c0), a1 = min(re, c1);
                float t = 0.f;
                for (int32_t j = a0 + (int32_t)lane; j < a1; j += 32) t += sc.prod[j - c0];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                if (rs < c0) t += carry_in;
                if (lane == 0) {
                    if (re <= c1) a.y[r] = t;
                    if (re >= c1) {
                        sc.rnext = (re > c1) ? r : r + 1u;
                        sc.carry_next = (re > c1) ? t : 0.f;
                    }
                }
            }
#else
            for (uint32_t r = r0 + warp; r < hi; r += nw) {   // warp-uniform
                const uint32_t i = r - r0;
                const int32_t rs = i < (uint32_t)kRp ? sc.rp[i] : __ldg(&a.row_ptr[r]);
                if (rs >= c1) break;                          // rows are sorted by start
                const int32_t re = i < (uint32_t)kRp ? sc.rp[i + 1] : __ldg(&a.row_ptr[r + 1]);
                const int32_t a0 = max(rs, c0), a1 = min(re, c1);
                float t = 0.f;
                for (int32_t j = a0 + (int32_t)lane; j < a1; j += 32) t += sc.prod[j - c0];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                if (rs < c0) t += carry_in;                   // only r0 can have started earlier
                if (lane == 0) {
                    if (re <= c1) a.y[r] = t;
                    if (re >= c1) {                           // the last row touching this chunk
                        sc.rnext = (re > c1) ? r : r + 1u;
                        sc.carry_next = (re > c1) ? t : 0.f;
                    }
                }
            }
#endif
#ifdef GTAP_SPMV_PIPE
            if (more) {
#pragma unroll
                for (int k = 0; k < kPer; ++k) pr[k] = vv[k] * __ldg(&a.x[cc[k]]);
            }
#endif
            __syncthreads();
            if (tid == 0) { sc.rcur = sc.rnext; sc.carry = sc.carry_next; }
            __syncthreads();
        }
        // rows that start at the leaf's last non-zero offset (empty rows at the end, or an empty leaf)
        for (uint32_t r = (s < e ? sc.rcur : lo) + tid; r < hi; r += bd)
            if (__ldg(&a.row_ptr[r]) == e) a.y[r] = 0.f;
        if (tid == 0) ctx.finish_void();
    }
};

static int validate_spmv(const gtap_task_table* t, uint32_t fn, const uint32_t* d) {
    SpmvTable::Args a;
    std::memcpy(&a, t->args, sizeof(a));
    if (fn == 1u) {   // part(k, R, r0, r1)
        const uint32_t r1 = d[3] ? d[3] : a.nrows;
        return (d[0] < d[1] && d[2] <= r1 && r1 <= a.nrows) ? 0 : -1;
    }
    return (fn == 0u && d[0] <= d[1] && d[1] <= a.nrows) ? 0 : -1;
}

}  // namespace gtap

extern "C" const gtap_task_table* gtap_table_spmv(const int32_t* row_ptr, const int32_t* col, const float* val,
                                                  const float* x, float* y, uint32_t nrows, uint32_t nnz_cut,
                                                  uint32_t fanout) {
    if (!row_ptr || !col || !val || !x || !y || fanout < 2 || fanout > 32 || nnz_cut == 0) return nullptr;
    gtap::SpmvTable::Args a{row_ptr, col, val, x, y, nrows, nnz_cut, fanout, 0u};
    return gtap::make_table<gtap::SpmvTable>("spmv", a, &gtap::validate_spmv);
}

#ifdef GTAP_TRACE
GTAP_TRACE_READER(spmv)
#endif
