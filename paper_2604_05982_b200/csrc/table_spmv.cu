// table_spmv.cu -- SpMV task table (block-level, no taskwait).
//
// The paper names SpMV as a block-cooperative workload but
// gives no listing; the task program here is reading R20:
//   spmv(lo, hi): if (nnz(lo, hi) > nnz_cut && hi - lo > 1)
//                   spawn spmv on `fanout` equal row sub-ranges   (no taskwait)
//                 else  y[i] = sum_j val[j] * x[col[j]] for i in [lo, hi),
//                       computed cooperatively by the block in fp32.
// Leaf layout: rows with <= kLight non-zeros are processed by 8-lane groups
// (4 rows per warp in flight, lanes stride the row, shuffle reduce); heavier
// rows are queued in shared memory and processed one at a time by the whole
// block (strided, 4-way unrolled, warp + shared-memory reduction), so a
// 64K-nnz row does not serialise on one warp. col/val/row_ptr/x are read-only
// for the run and use the non-coherent read-only path; y is write-only.
// Payload: d[0] = lo, d[1] = hi.
#include "table_common.cuh"

namespace gtap {

struct SpmvTable {
    static constexpr uint32_t kKind = GTAP_WORKER_BLOCK;
    static constexpr int kMaxChildren = 32;
    static constexpr bool kTaskwait = false;
    static constexpr uint32_t kNumFn = 1;
    static constexpr bool kJoinReduceAdd = false;  // see TaskRec
    static constexpr int kMaxThreads = 1024, kMinBlocks = 1;  // __launch_bounds__
    static constexpr int kSpawnCap = 32;
    static constexpr int kMaxHeavy = 256;
    static constexpr int32_t kLight = 256;
    struct Scratch {
        uint32_t nheavy;
        uint32_t heavy[kMaxHeavy];
        float red[32];
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
    // 8 lanes per row; each lane keeps 4 independent (col, val, x) loads in flight per iteration
    __device__ __forceinline__ static float row_group8(const Args& a, int32_t s, int32_t e, uint32_t g) {
        float acc0 = 0.f, acc1 = 0.f;
        int32_t j = s + (int32_t)g;
        for (; j + 24 < e; j += 32) {
            const int32_t c0 = ld_col(&a.col[j]), c1 = ld_col(&a.col[j + 8]);
            const int32_t c2 = ld_col(&a.col[j + 16]), c3 = ld_col(&a.col[j + 24]);
            const float v0 = ld_val(&a.val[j]), v1 = ld_val(&a.val[j + 8]);
            const float v2 = ld_val(&a.val[j + 16]), v3 = ld_val(&a.val[j + 24]);
            const float x0 = __ldg(&a.x[c0]), x1 = __ldg(&a.x[c1]), x2 = __ldg(&a.x[c2]), x3 = __ldg(&a.x[c3]);
            acc0 = fmaf(v0, x0, acc0);
            acc1 = fmaf(v1, x1, acc1);
            acc0 = fmaf(v2, x2, acc0);
            acc1 = fmaf(v3, x3, acc1);
        }
        // tail: up to 3 more strided elements per lane, loads issued together
        int32_t c[3];
        float v[3];
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            const int32_t jj = j + 8 * u;
            c[u] = jj < e ? ld_col(&a.col[jj]) : 0;
            v[u] = jj < e ? ld_val(&a.val[jj]) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 3; ++u)
            if (j + 8 * u < e) acc0 = fmaf(v[u], __ldg(&a.x[c[u]]), acc0);
        return acc0 + acc1;
    }

    template <class Ctx>
    __device__ __forceinline__ static void exec_block(const Args& a, Ctx& ctx, uint32_t fn, uint32_t state,
                                                      const uint32_t (&d)[kDataWords]) {
        if (fn != 0u || state != 0u) {
            if (threadIdx.x == 0) ctx.bad_state();
            return;
        }
        const uint32_t lo = d[0], hi = d[1];
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
        auto& sc = ctx.sm.scratch;
        if (tid == 0) sc.nheavy = 0;
        __syncthreads();
        // light rows: 8-lane groups, each group owns 4 consecutive rows at a time; every lane keeps
        // 4 rows x 2 strided (col, val, x) loads in flight, then the group reduces 4 sums by shuffle
        const uint32_t lane = tid & 31u, g = lane & 7u;
        const uint32_t grp = tid >> 3, ngrp = bd >> 3;
        constexpr uint32_t RPG = 4;
        for (uint32_t base = lo; base < hi; base += ngrp * RPG) {   // uniform trip count
            const uint32_t r0 = base + grp * RPG;
            // row_ptr[r0 .. r0+4] by lanes 0..4 of the group, shared by shuffle
            int32_t rpv = 0;
            if (g <= RPG && r0 + g <= hi) rpv = __ldg(&a.row_ptr[r0 + g]);
            int32_t rs[RPG], re[RPG];
            bool valid[RPG], queued[RPG];
#pragma unroll
            for (uint32_t q = 0; q < RPG; ++q) {
                rs[q] = __shfl_sync(0xffffffffu, rpv, (lane & ~7u) + q);
                re[q] = __shfl_sync(0xffffffffu, rpv, (lane & ~7u) + q + 1);
                valid[q] = r0 + q < hi;
                uint32_t qd = 0;
                if (valid[q] && re[q] - rs[q] > kLight && g == 0) {
                    const uint32_t hidx = atomicAdd(&sc.nheavy, 1u);
                    if (hidx < (uint32_t)kMaxHeavy) { sc.heavy[hidx] = r0 + q; qd = 1u; }
                }
                queued[q] = __shfl_sync(0xffffffffu, qd, lane & ~7u) != 0u;
                if (!valid[q] || queued[q]) re[q] = rs[q];  // nothing to do for this row here
            }
            float acc[RPG] = {0.f, 0.f, 0.f, 0.f};
            // passes of 16 keys per row (2 per lane); most rows (Pareto, mean ~32) need 1-2 passes
            int32_t maxlen = 0;
#pragma unroll
            for (uint32_t q = 0; q < RPG; ++q) maxlen = max(maxlen, re[q] - rs[q]);
            for (int32_t off = (int32_t)g; off < maxlen; off += 16) {
                int32_t c[RPG][2];
                float v[RPG][2];
                // branch-free: out-of-row slots load a valid key of the row (or of row_ptr[lo]) and are
                // multiplied by zero, so every lane issues all 8 (col, val) and 8 x loads back to back
#pragma unroll
                for (uint32_t q = 0; q < RPG; ++q)
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int32_t j = rs[q] + off + 8 * u;
                        const bool in = j < re[q];
                        const int32_t jj = in ? j : s;
                        c[q][u] = ld_col(&a.col[jj]);
                        v[q][u] = in ? ld_val(&a.val[jj]) : 0.f;
                    }
#pragma unroll
                for (uint32_t q = 0; q < RPG; ++q)
#pragma unroll
                    for (int u = 0; u < 2; ++u) acc[q] = fmaf(v[q][u], __ldg(&a.x[c[q][u]]), acc[q]);
            }
#pragma unroll
            for (uint32_t q = 0; q < RPG; ++q) {
                float t = acc[q];
                t += __shfl_xor_sync(0xffffffffu, t, 4);
                t += __shfl_xor_sync(0xffffffffu, t, 2);
                t += __shfl_xor_sync(0xffffffffu, t, 1);
                if (g == q && valid[q] && !queued[q]) a.y[r0 + q] = t;
            }
        }
        __syncthreads();
        // heavy rows: whole block per row
        const uint32_t nh = min(sc.nheavy, (uint32_t)kMaxHeavy);
        for (uint32_t h = 0; h < nh; ++h) {
            const uint32_t row = sc.heavy[h];
            const int32_t rs = __ldg(&a.row_ptr[row]), re = __ldg(&a.row_ptr[row + 1]);
            float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
            int32_t j = rs + (int32_t)tid;
            const int32_t st = (int32_t)bd;
            for (; j + 3 * st < re; j += 4 * st) {
                const int32_t c0 = ld_col(&a.col[j]), c1 = ld_col(&a.col[j + st]);
                const int32_t c2 = ld_col(&a.col[j + 2 * st]), c3 = ld_col(&a.col[j + 3 * st]);
                const float v0 = ld_val(&a.val[j]), v1 = ld_val(&a.val[j + st]);
                const float v2 = ld_val(&a.val[j + 2 * st]), v3 = ld_val(&a.val[j + 3 * st]);
                acc0 = fmaf(v0, __ldg(&a.x[c0]), acc0);
                acc1 = fmaf(v1, __ldg(&a.x[c1]), acc1);
                acc2 = fmaf(v2, __ldg(&a.x[c2]), acc2);
                acc3 = fmaf(v3, __ldg(&a.x[c3]), acc3);
            }
            for (; j < re; j += st) acc0 = fmaf(__ldg(&a.val[j]), __ldg(&a.x[__ldg(&a.col[j])]), acc0);
            float acc = (acc0 + acc1) + (acc2 + acc3);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) sc.red[tid >> 5] = acc;
            __syncthreads();
            if (tid < 32) {
                float v = (tid < (bd >> 5)) ? sc.red[tid] : 0.f;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (tid == 0) a.y[row] = v;
            }
            __syncthreads();
        }
        if (tid == 0) ctx.finish_void();
    }
};

static int validate_spmv(const gtap_task_table* t, uint32_t fn, const uint32_t* d) {
    SpmvTable::Args a;
    std::memcpy(&a, t->args, sizeof(a));
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
