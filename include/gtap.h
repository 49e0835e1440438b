/*
 * gtap.h -- C ABI of the B200-native GTaP hot path: a device-resident,
 * persistent-kernel fork-join scheduler (§4) behind plain
 * pointers and sizes. No torch types cross this boundary; the Python binding
 * (paper_2604_05982_b200/gtap.py) only marshals arguments.
 *
 * Paper mapping (P:n = line n of reference/PAPER.md):
 *   gtap_initialize() pre-allocates task storage (§5.1.2)
 *                                             -> gtap_workspace_bytes + gtap_init
 *   #pragma gtap entry: enqueue root + start
 *                                             -> gtap_spawn_root + gtap_run
 *   exec_kernel<<<GRID,BLOCK>>> + cudaDeviceSynchronize
 *                                             -> gtap_run + gtap_sync
 *   cudaMemcpyFromSymbol(&h_result, d_result) -> gtap_root_result
 *   gtap_finalize()                  -> gtap_finalize
 *   compile-time capacity macros (Table "Preprocessor macros")
 *                                             -> gtap_config fields
 *   #pragma gtap function task bodies -> per-benchmark task
 *                                                 tables (gtap_table_*)
 *
 * Conventions (every call):
 *   - returns gtap_status; nothing aborts, throws or prints;
 *   - device pointers are plain CUDA device addresses on the runtime's device
 *     (e.g. torch.Tensor.data_ptr()); they are caller-owned and must stay
 *     alive until gtap_sync returns for the run that uses them;
 *   - a cudaStream_t is passed as void* (NULL = legacy default stream);
 *   - one runtime per device per process thread; a runtime runs one table at
 *     a time; all roots of a run use that run's table.
 */
#ifndef GTAP_H
#define GTAP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GTAP_ABI_VERSION 2u  /* 2: gtap_config gained queue_policy / victim_policy (round 2) */

typedef enum {
    GTAP_OK = 0,
    GTAP_E_INVAL = 1,          /* bad argument / configuration */
    GTAP_E_CUDA = 2,           /* a CUDA runtime call failed */
    GTAP_E_NOMEM = 3,          /* device or host allocation failed */
    GTAP_E_BUSY = 4,           /* a run is in flight (call gtap_sync first) */
    GTAP_E_POOL_EXHAUSTED = 5, /* a worker's task-record pool ran out */
    GTAP_E_QUEUE_OVERFLOW = 6, /* a deque ring overflowed (fixed capacity) */
    GTAP_E_CHILD_LIMIT = 7,    /* > max_child_tasks spawns in one invocation */
    GTAP_E_TIMEOUT = 8,        /* liveness watchdog expired (config.watchdog_ns) */
    GTAP_E_BAD_STATE = 9,      /* unknown (task function, state) dispatched (P:1188 default:) */
    GTAP_E_NO_DEVICE = 10,     /* no CUDA device / not sm_100 */
    GTAP_E_UNSUPPORTED = 11,   /* table/config combination not built */
    GTAP_E_INVARIANT = 12      /* GTAP_CHECK builds: a scheduler invariant failed (gtap_check_read) */
} gtap_status;

typedef enum {
    GTAP_WORKER_THREAD = 0,    /* thread-executed: one CUDA thread runs one task */
    GTAP_WORKER_BLOCK = 1      /* block-cooperative: one block runs one task */
} gtap_worker_kind;

/* Runtime configuration: the paper's compile-time macros as run-time fields.
 * Zero means "default" where stated. */
typedef struct {
    uint32_t struct_size;          /* = sizeof(gtap_config); ABI guard */
    int32_t  device;               /* CUDA ordinal of this process's GPU */
    uint32_t worker_kind;          /* gtap_worker_kind */
    uint32_t grid_size;            /* GTAP_GRID_SIZE; 0 = all co-resident blocks */
    uint32_t block_size;           /* GTAP_BLOCK_SIZE; multiple of 32; 0 = 128 */
    uint32_t max_tasks_per_worker; /* GTAP_MAX_TASKS_PER_WARP / _PER_BLOCK;
                                      records per worker pool, power of two; 0 = 4096 */
    uint32_t queue_capacity;       /* ring slots per deque, power of two; 0 = max_tasks_per_worker */
    uint32_t max_child_tasks;      /* GTAP_MAX_CHILD_TASKS: an invocation spawning more fails
                                      the run with GTAP_E_CHILD_LIMIT; 0 = the table's own bound (a larger
                                      value is clamped to it) */
    uint32_t num_queues;           /* GTAP_NUM_QUEUES (EPAQ): deques per warp, 1..8;
                                      block-level workers: 1; 0 = 1 */
    uint32_t max_task_data_size;   /* GTAP_MAX_TASK_DATA_SIZE bytes; 0 = 16 */
    uint32_t assume_no_taskwait;   /* GTAP_ASSUME_NO_TASKWAIT; informative:
                                      tables that never join set it themselves */
    uint32_t steal_attempts;       /* victims probed per idle cycle; 0 = 4 */
    uint32_t steal_max;            /* max tasks per steal, <= 32; 0 = 32 (warp) / 1 (block). A block-level
                                      steal of c > 1 runs one task and keeps c - 1 in the thief's own deque */
    uint32_t max_roots;            /* forest capacity (roots per run); 0 = 65536 */
    uint64_t seed;                 /* victim-selection PRNG seed */
    uint64_t watchdog_ns;          /* 0 = off; else a run longer than this fails with GTAP_E_TIMEOUT */
    uint32_t idle_backoff_ns;      /* cap of an idle worker's exponential nanosleep backoff; 0 = 8192 */
    uint32_t queue_policy;         /* EPAQ (num_queues > 1) class kept for a warp's next cycle:
                                      0 = the next queue in round-robin order every cycle (DESIGN R24);
                                      1 = stay on the queue in use while the cycle produced runnable tasks
                                      of it, else the next one (round robin) that has some */
    uint32_t victim_policy;        /* steal-victim choice ("random"): 0 = uniform over the other workers;
                                      1 = die-aware: gtap_init measures the SM -> L2-die map and which die homes
                                      each worker's deque line (gtap_ubench_die_probe), and 3 of 4 probing
                                      lanes then draw victims whose deque line is near the thief's die */
    uint32_t reserved2;
} gtap_config;

typedef struct gtap_runtime gtap_runtime;
typedef struct gtap_task_table gtap_task_table;

/* Counters of one run, summed over workers on the device at kernel exit. */
typedef struct {
    uint64_t tasks;            /* task records created (roots included) */
    uint64_t invocations;      /* task-function invocations (one per state executed) */
    uint64_t pops;             /* tasks taken from the worker's own deque */
    uint64_t kept;             /* tasks run from the keep-for-next-cycle set */
    uint64_t steals_ok;        /* successful steal operations */
    uint64_t steals_failed;    /* steal attempts that found nothing or lost the race */
    uint64_t stolen_tasks;     /* tasks moved by steals */
    uint64_t pushes;           /* tasks written to deques */
    uint64_t cycles;           /* scheduler loop iterations that executed >= 1 task */
    uint64_t idle_cycles;      /* scheduler loop iterations without a task */
    uint64_t remote_frees;     /* records freed by a worker other than their home */
    uint64_t max_pool_used;    /* max records ever drawn from one worker's bump region */
    uint32_t error_word;       /* gtap_status set on the device (0 = none) */
    uint32_t workers;          /* warps (thread-level) or blocks (block-level) */
    float    device_ms;        /* CUDA-event time of the persistent kernel */
    uint32_t grid_size;        /* launched grid */
    uint32_t block_size;       /* launched block */
    uint32_t assists;          /* task bodies run by the whole warp (warp assist, tables with kAssist) */
    uint32_t reserved;
} gtap_stats;

/* ---- lifecycle ---------------------------------------------------------- */

/* Version of this ABI (GTAP_ABI_VERSION). */
uint32_t gtap_abi_version(void);

/* Human-readable name of a status code (static storage, never NULL). */
const char *gtap_status_str(gtap_status s);

/* Fill *cfg with defaults for `kind` on `device` (struct_size set). */
gtap_status gtap_config_default(gtap_config *cfg, int32_t device, uint32_t kind);

/* Device bytes gtap_init needs for *cfg (0 on invalid cfg). Layout: task
 * records (32 B each, 16-B aligned), deque rings, per-deque metadata lines,
 * per-worker free rings, control block. */
size_t gtap_workspace_bytes(const gtap_config *cfg);

/* Create a runtime ("pre-allocates the memory regions required for
 * task management on the host side"). d_workspace: caller-owned device buffer
 * of >= gtap_workspace_bytes(cfg) bytes, 256-B aligned, or NULL to let the
 * runtime cudaMalloc (and free) it. On success *out is a new runtime. */
gtap_status gtap_init(const gtap_config *cfg, void *d_workspace, size_t bytes, gtap_runtime **out);

/* Stage a root task ("entry enqueues the initial (root) task"). The
 * args (nbytes <= 16) are copied now (firstprivate). Several calls
 * before one gtap_run make a forest; roots are spread round-robin over the
 * workers. *root_idx (may be NULL) indexes gtap_root_result. All roots of a
 * run must use the same table. */
gtap_status gtap_spawn_root(gtap_runtime *rt, const gtap_task_table *table, uint32_t fn,
                            const void *args, uint32_t nbytes, uint32_t *root_idx);

/* Re-arm the workspace for a new run (zero queues, pools, counters; drop
 * staged roots). Asynchronous on `stream`; the next gtap_run waits for it
 * (an event recorded here, waited for on the run's stream), so reset and run
 * may use different streams. */
gtap_status gtap_reset(gtap_runtime *rt, void *stream);

/* Launch the persistent kernel for the staged roots on `stream` (async).
 * Implies gtap_reset unless the runtime was reset since the last run.
 * Everything a run enqueues is SM work on `stream`: a small kernel stages the
 * roots and control block from the runtime's mapped pinned host buffers, the
 * table's scratch/board and workspace resets are fill kernels, and the control
 * block returns the same way after the scheduler -- no copy-engine transfer,
 * so a run never queues behind the caller's bulk copies on other streams.
 * Returns GTAP_E_BUSY if a run is in flight, GTAP_E_INVAL if no root is
 * staged or the grid cannot be co-resident. Any other failure drops the
 * staged roots and the table binding (stage them again after fixing the
 * cause); the workspace is fully reset before the next run. */
gtap_status gtap_run(gtap_runtime *rt, void *stream);

/* Block until the run finishes; decode the device error word; fill *out
 * (may be NULL). Returns the device error (GTAP_E_POOL_EXHAUSTED, ...) if any. */
gtap_status gtap_sync(gtap_runtime *rt, gtap_stats *out);

/* Copy root result `root_idx` (int64 on the device) into *out
 * (nbytes <= 8, little-endian truncation). Valid after gtap_sync. */
gtap_status gtap_root_result(gtap_runtime *rt, uint32_t root_idx, void *out, uint32_t nbytes);

/* Scheduler-invariant counters of the last run (the
 * correctness sketch of P:137-141): available only in the diagnostic build
 * compiled with -DGTAP_CHECK (libgtap_gtap_check.so), else GTAP_E_UNSUPPORTED.
 * That build keeps per-record tokens (allocated, published-and-unclaimed,
 * children of the current join epoch) and checks them at every scheduler
 * event; a violation fails the run with GTAP_E_INVARIANT. Valid after
 * gtap_sync. out[0..15]: events and violations in this order -- allocs,
 * frees, publications, dispatches, suspends, child joins, continuation
 * dispatches, double allocs, double frees, double publications, dispatches of
 * unpublished tasks, continuations dispatched before their last child joined,
 * join underflows, suspends over a live join; out[16] = records still
 * allocated, out[17] = tasks still published, out[18] = records with a join
 * count != 0, out[19] = outstanding counter, out[20] = roots not finished.
 * n: capacity of out (>= 21). */
gtap_status gtap_check_read(gtap_runtime *rt, uint64_t *out, uint32_t n);

/* Release everything gtap_init allocated. rt may be NULL. */
gtap_status gtap_finalize(gtap_runtime *rt);

/* Effective launch geometry of `table` on this runtime (after defaults and
 * the occupancy clamp): workers, grid, block. */
gtap_status gtap_geometry(gtap_runtime *rt, const gtap_task_table *table,
                          uint32_t *workers, uint32_t *grid, uint32_t *block);

/* ---- task tables (the "#pragma gtap function" bodies, hand-transformed) -- */

/* Free a table returned by a gtap_table_* constructor (NULL ok). */
void gtap_table_destroy(const gtap_task_table *t);

/* fib (P:1023-1033 + transformed P:1160-1190), thread-level, no cutoff.
 * fn 0, root args {int32 n}, 0 <= n <= 46; result int64 fib(n). */
const gtap_task_table *gtap_table_fib(void);

/* fib with a cutoff (the EPAQ experiment), thread-level:
 * n < cutoff runs the serial recursion inside the task. num_queues = 1 (no
 * EPAQ) or 3 (EPAQ: non-cutoff children -> queue 0, cutoff children ->
 * queue 1, continuations -> queue 2; needs config.num_queues >= 3). fn 0, root
 * args {int32 n}, 0 <= n <= 46; result int64 fib(n). NULL on bad arguments. */
const gtap_task_table *gtap_table_fib_cutoff(int32_t cutoff, uint32_t num_queues);

/* N-Queens: bitmask backtracking, one task per free column while
 * fewer than `cutoff` rows are placed, serial counting below; no taskwait.
 * n in [1, 20]; d_count: caller-owned device uint64, zeroed by the caller,
 * receives the number of solutions. fn 0, root args {} (nbytes 0). */
const gtap_task_table *gtap_table_nqueens(int32_t n, int32_t cutoff, unsigned long long *d_count);
/* N-Queens with an explicit leaf_mode: 0 = the paper's serial leaf on the task's lane; 1 = the
 * task's warp counts the leaf (two rows expanded, sub-problems counted round robin by the lanes;
 * DESIGN.md R28). Same tasks and count. gtap_table_nqueens is leaf_mode 1. */
const gtap_task_table *gtap_table_nqueens_ex(int32_t n, int32_t cutoff, unsigned long long *d_count,
                                             uint32_t leaf_mode);

/* Synthetic tree (§6.3), on either worker kind
 * (worker_kind = GTAP_WORKER_THREAD: one task per lane; GTAP_WORKER_BLOCK: the
 * body runs data-parallel over the block). A node spawns its children, joins
 * (taskwait), then runs do_memory_and_compute.
 * B = 0: full binary tree of depth D (2^(D+1) - 1 tasks), root args
 *        {id lo = 1, id hi = 0, depth = 0}; children of id are 2id, 2id+1.
 * B in [1, 8]: pruned B-ary tree, root args {0, 0, 0}; child k of id at
 *        depth d is B*id + 1 + k, kept iff mix(seed ^ child) >> 11 <
 *        floor((D - d) * 2^53 / D) (p(d) = 1 - d/D; R27); D >= 1.
 * do_memory_and_compute(id): mem_ops 64-bit loads of buf[mix(id * G + i) & (len-1)]
 * and compute_iters FP64 FMAs in min(64, compute_iters) chains, summed with the
 * chains' final bits mod 2^64 (R27). buf: device uint64[len], len a power of
 * two, read-only; d_total: caller-owned device uint64[32], zeroed by the
 * caller; the run's value is the sum of the 32 words mod 2^64. D in [0, 40].
 * NULL on bad arguments. */
const gtap_task_table *gtap_table_tree(int32_t worker_kind, int32_t D, int32_t B, uint64_t seed,
                                       const unsigned long long *buf, uint64_t len, uint32_t mem_ops,
                                       uint32_t compute_iters, unsigned long long *d_total);

/* mergesort with cutoff (state machine P:59-74), thread-level.
 * keys: int32[n] device buffer sorted in place; scratch: int32[n] device
 * buffer (ping-pong target); cutoff in [1, 256]. fn 0, root args
 * {uint32 l, uint32 r} (normally {0, n}); result 0. Same as
 * gtap_table_mergesort_ex(..., GTAP_MERGE_WARP). */
const gtap_task_table *gtap_table_mergesort(int32_t *keys, int32_t *scratch, uint64_t n,
                                            int32_t cutoff);

/* How a merge task body runs. GTAP_MERGE_THREAD: on the task's own
 * lane (the paper's thread-level merge; merges >= 8192 keys stream
 * through shared memory by TMA). GTAP_MERGE_WARP: merges >= 8192 keys are run
 * by all 32 lanes of the task's warp after the cycle's bodies (merge-path
 * slices); the task graph, task counts and the
 * sorted output are identical. */
enum { GTAP_MERGE_THREAD = 0, GTAP_MERGE_WARP = 1 };
const gtap_task_table *gtap_table_mergesort_ex(int32_t *keys, int32_t *scratch, uint64_t n,
                                               int32_t cutoff, uint32_t merge_mode);

/* Cilksort: mergesort whose merge is fork-join (split the
 * longer run at its middle, binary-search the other). keys/scratch: int32[n]
 * device buffers, n < 2^25; cut_sort in [1, 256], cut_merge >= 2 (paper: 64 /
 * 256). Output sorted in keys. fn 0, root args {uint32 l, uint32 r}. */
const gtap_task_table *gtap_table_cilksort(int32_t *keys, int32_t *scratch, uint64_t n, int32_t cut_sort,
                                           int32_t cut_merge);
/* Cilksort with an explicit merge_mode (GTAP_MERGE_THREAD: leaf sorts and sequential merges on
 * the task's lane; GTAP_MERGE_WARP: those bodies run by the task's warp -- bitonic networks, same
 * task graph and output). gtap_table_cilksort is merge_mode GTAP_MERGE_WARP. */
const gtap_task_table *gtap_table_cilksort_ex(int32_t *keys, int32_t *scratch, uint64_t n, int32_t cut_sort,
                                              int32_t cut_merge, uint32_t merge_mode);

/* SpMV y = A x over CSR (P:42 names SpMV as block-cooperative), block-level,
 * no taskwait. Task spmv(lo, hi) splits the row range into `fanout` equal
 * parts while it holds more than nnz_cut non-zeros (and > 1 row); leaves are
 * computed cooperatively by the block in fp32. fn 0, root args
 * {uint32 lo, uint32 hi}. fn 1 = part(k, R, r0, r1), root args {uint32 k,
 * uint32 R, uint32 r0, uint32 r1} (r1 = 0: nrows), k < R: the k-th of R
 * contiguous row ranges of [r0, r1) balanced by non-zeros (boundary j = first
 * row whose start offset reaches row_ptr[r0] + floor(j * nnz(r0, r1) / R),
 * found in the kernel), then processed as spmv(lo, hi); the R roots k =
 * 0..R-1 cover every row of [r0, r1) once (a forest: each worker starts with
 * its own range, R20).
 * y rows outside roots' ranges are untouched. */
const gtap_task_table *gtap_table_spmv(const int32_t *row_ptr, const int32_t *col,
                                       const float *val, const float *x, float *y,
                                       uint32_t nrows, uint32_t nnz_cut, uint32_t fanout);

/* BFS frontier expansion, block-level, no taskwait.
 * depth: int32[nv], caller sets INT32_MAX everywhere and 0 at the source
 * before the run (reading R18). fn 0, root args {int32 v}. */
const gtap_task_table *gtap_table_bfs(const int32_t *row_ptr, const int32_t *col,
                                      int32_t *depth, uint32_t nv);

/* BFS with a choice of owner pop order (a B200 scheduling option, semantics-free: the levels are the
 * same): order 0 = gtap_table_bfs (LIFO pops of the own deque, the block keeps its newest child,
 * P:89-93); order 1 = oldest-first batch pops, every child pushed -- the deques behave FIFO, closer to
 * level order, fewer re-expansions, but each deque may hold a whole local frontier (size
 * max_tasks_per_worker / queue_capacity accordingly; an undersized ring fails the run with
 * GTAP_E_QUEUE_OVERFLOW). NULL on bad arguments or order > 1. */
const gtap_task_table *gtap_table_bfs_ex(const int32_t *row_ptr, const int32_t *col,
                                         int32_t *depth, uint32_t nv, uint32_t order);

/* BFS with hub splitting (a B200 decomposition, R29; the levels are the same): as
 * gtap_table_bfs_ex, and a bfs(v) task whose vertex has more than edge_split edges spawns fn 1
 * bfs_edges(v, lo, hi) tasks for the pieces [s + k*edge_split, ...) of its edge list beyond the first,
 * which it scans itself; a piece re-reads depth[v] (it can only have decreased). edge_split 0 = never
 * (= gtap_table_bfs_ex). Roots are fn 0. NULL on bad arguments or order > 1. */
const gtap_task_table *gtap_table_bfs_split(const int32_t *row_ptr, const int32_t *col,
                                            int32_t *depth, uint32_t nv, uint32_t order,
                                            uint32_t edge_split);

/* BFS input preparation (reading R18): depth[v] = INT32_MAX for v != src,
 * depth[src] = 0, asynchronously on `stream`. */
gtap_status gtap_bfs_init_depth(int32_t *depth, uint32_t nv, int32_t src, void *stream);

/* ---- microbenchmarks (roofline denominators) ----------- */

/* SM -> L2-die map (SURVEY.md §8(d) probe (vi)), synchronous on `stream`: one block per SM, in turn,
 * times dependent strong (L2) loads to n_addr addresses spaced bytes / n_addr apart in d_buf (>= 2 KB apart
 * to see distinct L2 homes). h_sm_die[smid] (sm_cap entries) = 0 for SM 0's die, 1 for the other;
 * h_addr_near[k] (may be NULL) = the die whose SMs reach address k faster; h_out3 (may be NULL) = {mean
 * near latency, mean far latency (cycles), consistency = mean fraction of addresses on which an SM's
 * near/far pattern matches its die}. Needs the GPU to itself (timing). */
gtap_status gtap_ubench_die_probe(const void *d_buf, uint64_t bytes, uint32_t n_addr, uint8_t *h_sm_die,
                                  uint32_t sm_cap, uint8_t *h_addr_near, float *h_out3, void *stream);

/* L2-atomic throughput probe on `stream`, synchronous. kind: 0 atom.add with
 * return on distinct words (the join decrement), 1 red.add (no return),
 * 2 atom.cas, 3 atom.min, 4 same-address atom.add, 5 atom.acq_rel.add, 6 relaxed
 * 64-bit atom.add with return (the fused fib join word). d_buf: device buffer of
 * >= words*4 bytes (zeroed by the call). ops_per_thread atomics per thread on
 * grid x block threads. *ms = kernel time. */
gtap_status gtap_ubench_atomics(void *d_buf, uint64_t words, uint32_t kind, uint32_t grid,
                                uint32_t block, uint32_t ops_per_thread, void *stream, float *ms);

#ifdef __cplusplus
}
#endif

#endif /* GTAP_H */
