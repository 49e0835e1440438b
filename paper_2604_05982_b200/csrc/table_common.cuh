// table_common.cuh -- host-side task-table object and the launch/occupancy
// glue that instantiates one persistent kernel per table (the paper compiles
// one exec_kernel per program).
#pragma once
#include <cstring>
#include <new>

#include "gtap.h"
#include "gtap_internal.cuh"
#include "sched_thread.cuh"
#include "sched_block.cuh"

struct gtap_task_table {
    uint32_t kind;          // gtap_worker_kind
    uint32_t taskwait;      // table ever suspends (otherwise GTAP_ASSUME_NO_TASKWAIT semantics)
    uint32_t max_children;  // compile-time bound of the table (GTAP_MAX_CHILD_TASKS)
    uint32_t nfn;           // number of task functions
    uint32_t max_block;     // __launch_bounds__ max threads of the table's kernel
    uint32_t num_queues;    // EPAQ queues the table routes tasks to (1 = no EPAQ)
    const char* name;
    cudaError_t (*launch)(const gtap_task_table*, const gtap::KParams&, uint32_t grid, uint32_t block,
                          cudaStream_t);
    cudaError_t (*occupancy)(const gtap_task_table*, uint32_t block, int* blocks_per_sm, size_t* smem);
    int (*validate_root)(const gtap_task_table*, uint32_t fn, const uint32_t* d);
    // optional: device memory owned by the table (freed by gtap_table_destroy) and a per-run
    // reset enqueued by gtap_run before the launch
    void* dev_scratch = nullptr;
    cudaError_t (*prepare)(const gtap_task_table*, cudaStream_t) = nullptr;
    alignas(16) unsigned char args[128];
};

namespace gtap {

template <class T>
inline size_t thread_smem(uint32_t block) {
    return block_extra_bytes<T>() + (size_t)(block / 32) * sizeof(WarpSmem<T::kMaxChildren, free_stack_of<T>::value>);
}

template <class T>
cudaError_t launch_thread(const gtap_task_table* t, const KParams& p, uint32_t grid, uint32_t block,
                          cudaStream_t s) {
    typename T::Args a;
    std::memcpy(&a, t->args, sizeof(a));
    const size_t smem = thread_smem<T>(block);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(thread_sched_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    thread_sched_kernel<T><<<grid, block, smem, s>>>(p, a);
    return cudaGetLastError();
}

template <class T>
cudaError_t occupancy_thread(const gtap_task_table*, uint32_t block, int* bps, size_t* smem) {
    *smem = thread_smem<T>(block);
    if (*smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(thread_sched_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem);
        if (e != cudaSuccess) return e;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, thread_sched_kernel<T>, (int)block, *smem);
}

template <class T>
cudaError_t launch_block(const gtap_task_table* t, const KParams& p, uint32_t grid, uint32_t block,
                         cudaStream_t s) {
    typename T::Args a;
    std::memcpy(&a, t->args, sizeof(a));
    block_sched_kernel<T><<<grid, block, 0, s>>>(p, a);
    return cudaGetLastError();
}

template <class T>
cudaError_t occupancy_block(const gtap_task_table*, uint32_t block, int* bps, size_t* smem) {
    *smem = 0;  // static shared memory (BlockSmem<T>)
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, block_sched_kernel<T>, (int)block, 0);
}

template <class T>
gtap_task_table* make_table(const char* name, const typename T::Args& a,
                            int (*validate)(const gtap_task_table*, uint32_t, const uint32_t*)) {
    static_assert(sizeof(typename T::Args) <= 128, "table args too large");
    gtap_task_table* t = new (std::nothrow) gtap_task_table();
    if (!t) return nullptr;
    t->kind = T::kKind;
    t->taskwait = T::kTaskwait ? 1u : 0u;
    t->max_children = (uint32_t)T::kMaxChildren;
    t->nfn = T::kNumFn;
    t->max_block = (uint32_t)T::kMaxThreads;
    if constexpr (T::kKind == GTAP_WORKER_THREAD) t->num_queues = (uint32_t)num_queues_of<T>::value;
    else t->num_queues = 1;
    t->name = name;
    if constexpr (T::kKind == GTAP_WORKER_THREAD) {
        t->launch = &launch_thread<T>;
        t->occupancy = &occupancy_thread<T>;
    } else {
        t->launch = &launch_block<T>;
        t->occupancy = &occupancy_block<T>;
    }
    t->validate_root = validate;
    std::memcpy(t->args, &a, sizeof(a));
    return t;
}

}  // namespace gtap
