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

    __device__ __forceinline__ static float row_group8(const Args& a, int32_t s, int32_t e, uint32_t g) {
        float acc = 0.f;
        int32_t j = s + (int32_t)g;
        for (; j + 8 < e; j += 16) {
            const int32_t c0 = __ldg(&a.col[j]), c1 = __ldg(&a.col[j + 8]);
            const float v0 = __ldg(&a.val[j]), v1 = __ldg(&a.val[j + 8]);
            acc = fmaf(v0, __ldg(&a.x[c0]), acc);
            acc = fmaf(v1, __ldg(&a.x[c1]), acc);
        }
        if (j < e) acc = fmaf(__ldg(&a.val[j]), __ldg(&a.x[__ldg(&a.col[j])]), acc);
        return acc;
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
        // light rows: 8-lane groups, 4 rows per warp
        const uint32_t lane = tid & 31u, g = lane & 7u;
        const uint32_t grp = tid >> 3, ngrp = bd >> 3;
        for (uint32_t base = lo; base < hi; base += ngrp) {   // uniform trip count
            const uint32_t row = base + grp;
            const bool valid = row < hi;
            int32_t rs = 0, re = 0;
            if (valid) { rs = __ldg(&a.row_ptr[row]); re = __ldg(&a.row_ptr[row + 1]); }
            uint32_t queued = 0;
            if (valid && re - rs > kLight && g == 0) {
                const uint32_t hidx = atomicAdd(&sc.nheavy, 1u);
                if (hidx < (uint32_t)kMaxHeavy) { sc.heavy[hidx] = row; queued = 1u; }
            }
            queued = __shfl_sync(0xffffffffu, queued, lane & ~7u);
            const bool compute = valid && !queued;
            float acc = compute ? row_group8(a, rs, re, g) : 0.f;
            acc += __shfl_xor_sync(0xffffffffu, acc, 4);
            acc += __shfl_xor_sync(0xffffffffu, acc, 2);
            acc += __shfl_xor_sync(0xffffffffu, acc, 1);
            if (compute && g == 0) a.y[row] = acc;
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
                const int32_t c0 = __ldg(&a.col[j]), c1 = __ldg(&a.col[j + st]);
                const int32_t c2 = __ldg(&a.col[j + 2 * st]), c3 = __ldg(&a.col[j + 3 * st]);
                acc0 = fmaf(__ldg(&a.val[j]), __ldg(&a.x[c0]), acc0);
                acc1 = fmaf(__ldg(&a.val[j + st]), __ldg(&a.x[c1]), acc1);
                acc2 = fmaf(__ldg(&a.val[j + 2 * st]), __ldg(&a.x[c2]), acc2);
                acc3 = fmaf(__ldg(&a.val[j + 3 * st]), __ldg(&a.x[c3]), acc3);
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
