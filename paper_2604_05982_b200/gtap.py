"""ctypes binding of the C ABI in include/gtap.h (argument marshalling only).

Every step of the hot path runs in libgtap.so's CUDA kernels; this module
converts Python/torch arguments to plain pointers and sizes, allocates the
runtime workspace through PyTorch (caller-owned device memory) and turns
status codes into exceptions. It never computes task results itself and has
no CPU fallback: if libgtap.so is missing or no B200 is present, it raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GTAP_LIB") or os.path.join(_PKG, "libgtap.so")  # GTAP_LIB: diagnostic builds

GTAP_WORKER_THREAD = 0
GTAP_WORKER_BLOCK = 1

STATUS = {
    0: "GTAP_OK", 1: "GTAP_E_INVAL", 2: "GTAP_E_CUDA", 3: "GTAP_E_NOMEM", 4: "GTAP_E_BUSY",
    5: "GTAP_E_POOL_EXHAUSTED", 6: "GTAP_E_QUEUE_OVERFLOW", 7: "GTAP_E_CHILD_LIMIT",
    8: "GTAP_E_TIMEOUT", 9: "GTAP_E_BAD_STATE", 10: "GTAP_E_NO_DEVICE", 11: "GTAP_E_UNSUPPORTED", 12: "GTAP_E_INVARIANT",
}


class GtapError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {STATUS.get(code, code)}")


class Config(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32), ("device", ctypes.c_int32), ("worker_kind", ctypes.c_uint32),
        ("grid_size", ctypes.c_uint32), ("block_size", ctypes.c_uint32),
        ("max_tasks_per_worker", ctypes.c_uint32), ("queue_capacity", ctypes.c_uint32),
        ("max_child_tasks", ctypes.c_uint32), ("num_queues", ctypes.c_uint32),
        ("max_task_data_size", ctypes.c_uint32), ("assume_no_taskwait", ctypes.c_uint32),
        ("steal_attempts", ctypes.c_uint32), ("steal_max", ctypes.c_uint32), ("max_roots", ctypes.c_uint32),
        ("seed", ctypes.c_uint64), ("watchdog_ns", ctypes.c_uint64),
        ("idle_backoff_ns", ctypes.c_uint32), ("queue_policy", ctypes.c_uint32),
        ("victim_policy", ctypes.c_uint32), ("reserved2", ctypes.c_uint32),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("tasks", ctypes.c_uint64), ("invocations", ctypes.c_uint64), ("pops", ctypes.c_uint64),
        ("kept", ctypes.c_uint64), ("steals_ok", ctypes.c_uint64), ("steals_failed", ctypes.c_uint64),
        ("stolen_tasks", ctypes.c_uint64), ("pushes", ctypes.c_uint64), ("cycles", ctypes.c_uint64),
        ("idle_cycles", ctypes.c_uint64), ("remote_frees", ctypes.c_uint64), ("max_pool_used", ctypes.c_uint64),
        ("error_word", ctypes.c_uint32), ("workers", ctypes.c_uint32), ("device_ms", ctypes.c_float),
        ("grid_size", ctypes.c_uint32), ("block_size", ctypes.c_uint32), ("assists", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
    ]

    def as_dict(self) -> dict:
        return {k: (getattr(self, k) if k != "reserved" else None) for k, _ in self._fields_ if k != "reserved"}


ABI_VERSION = 2  # include/gtap.h GTAP_ABI_VERSION

# Every symbol include/gtap.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "gtap_abi_version", "gtap_status_str", "gtap_config_default", "gtap_workspace_bytes", "gtap_init",
    "gtap_spawn_root", "gtap_reset", "gtap_run", "gtap_sync", "gtap_root_result", "gtap_finalize",
    "gtap_geometry", "gtap_table_destroy", "gtap_table_fib", "gtap_table_fib_cutoff", "gtap_table_nqueens", "gtap_table_nqueens_ex", "gtap_table_tree", "gtap_table_mergesort", "gtap_table_mergesort_ex", "gtap_table_cilksort", "gtap_table_cilksort_ex",
    "gtap_table_spmv",
    "gtap_table_bfs", "gtap_table_bfs_ex", "gtap_table_bfs_split", "gtap_bfs_init_depth", "gtap_ubench_atomics", "gtap_ubench_die_probe", "gtap_check_read",
]

_lib = None


def lib():
    """Load libgtap.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run python -c 'import __graft_entry__ as g; g.build()'")
    L = ctypes.CDLL(LIB_PATH)
    vp, u32, i32, u64, sz = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_size_t
    P = ctypes.POINTER
    L.gtap_abi_version.restype = u32
    L.gtap_status_str.restype = ctypes.c_char_p
    L.gtap_status_str.argtypes = [ctypes.c_int]
    L.gtap_config_default.argtypes = [P(Config), i32, u32]
    L.gtap_workspace_bytes.argtypes = [P(Config)]
    L.gtap_workspace_bytes.restype = sz
    L.gtap_init.argtypes = [P(Config), vp, sz, P(vp)]
    L.gtap_spawn_root.argtypes = [vp, vp, u32, vp, u32, P(u32)]
    L.gtap_reset.argtypes = [vp, vp]
    L.gtap_run.argtypes = [vp, vp]
    L.gtap_sync.argtypes = [vp, P(Stats)]
    L.gtap_root_result.argtypes = [vp, u32, vp, u32]
    L.gtap_finalize.argtypes = [vp]
    L.gtap_geometry.argtypes = [vp, vp, P(u32), P(u32), P(u32)]
    L.gtap_table_destroy.argtypes = [vp]
    L.gtap_table_destroy.restype = None
    L.gtap_table_fib.argtypes = []
    L.gtap_table_fib.restype = vp
    L.gtap_table_fib_cutoff.argtypes = [i32, u32]
    L.gtap_table_fib_cutoff.restype = vp
    L.gtap_table_nqueens.argtypes = [i32, i32, vp]
    L.gtap_table_nqueens.restype = vp
    L.gtap_table_nqueens_ex.argtypes = [i32, i32, vp, ctypes.c_uint32]
    L.gtap_table_nqueens_ex.restype = vp
    L.gtap_table_tree.argtypes = [i32, i32, i32, ctypes.c_uint64, vp, ctypes.c_uint64, ctypes.c_uint32,
                                  ctypes.c_uint32, vp]
    L.gtap_table_tree.restype = vp
    L.gtap_table_mergesort.argtypes = [vp, vp, u64, i32]
    L.gtap_table_mergesort.restype = vp
    L.gtap_table_mergesort_ex.argtypes = [vp, vp, u64, i32, ctypes.c_uint32]
    L.gtap_table_mergesort_ex.restype = vp
    L.gtap_table_cilksort.argtypes = [vp, vp, u64, i32, i32]
    L.gtap_table_cilksort.restype = vp
    L.gtap_table_cilksort_ex.argtypes = [vp, vp, u64, i32, i32, ctypes.c_uint32]
    L.gtap_table_cilksort_ex.restype = vp
    L.gtap_table_spmv.argtypes = [vp, vp, vp, vp, vp, u32, u32, u32]
    L.gtap_table_spmv.restype = vp
    L.gtap_table_bfs.argtypes = [vp, vp, vp, u32]
    L.gtap_table_bfs.restype = vp
    L.gtap_table_bfs_ex.argtypes = [vp, vp, vp, u32, u32]
    L.gtap_table_bfs_ex.restype = vp
    L.gtap_table_bfs_split.argtypes = [vp, vp, vp, u32, u32, u32]
    L.gtap_table_bfs_split.restype = vp
    L.gtap_bfs_init_depth.argtypes = [vp, u32, i32, vp]
    L.gtap_ubench_atomics.argtypes = [vp, u64, u32, u32, u32, u32, vp, P(ctypes.c_float)]
    L.gtap_check_read.argtypes = [vp, P(u64), u32]
    L.gtap_ubench_die_probe.argtypes = [vp, u64, u32, vp, u32, vp, vp, vp]
    for name in ("gtap_config_default", "gtap_init", "gtap_spawn_root", "gtap_reset", "gtap_run", "gtap_sync",
                 "gtap_root_result", "gtap_finalize", "gtap_geometry", "gtap_ubench_atomics", "gtap_bfs_init_depth",
                 "gtap_check_read", "gtap_ubench_die_probe"):
        getattr(L, name).restype = ctypes.c_int
    if L.gtap_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH}: ABI version {L.gtap_abi_version()} != binding's {ABI_VERSION}; rebuild")
    _lib = L
    return L


def _check(code: int, where: str):
    if code != 0:
        raise GtapError(code, where)


def _stream_ptr(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream or None
    return getattr(stream, "cuda_stream", stream) or None


class Table:
    """A task table (one persistent-kernel instantiation + its constant args).

    Holds references to the tensors whose pointers the table captured so they
    outlive every run that uses it."""

    def __init__(self, ptr: int, name: str, kind: int, keep=()):
        if not ptr:
            raise GtapError(1, f"gtap_table_{name}")
        self.ptr = ptr
        self.name = name
        self.kind = kind
        self._keep = tuple(keep)

    def close(self):
        if self.ptr:
            lib().gtap_table_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- constructors (include/gtap.h) ----
    @staticmethod
    def fib() -> "Table":
        return Table(lib().gtap_table_fib(), "fib", GTAP_WORKER_THREAD)

    @staticmethod
    def fib_cutoff(cutoff: int, num_queues: int = 1) -> "Table":
        """fib with a cutoff; num_queues=3 routes tasks with the paper's EPAQ classifier."""
        return Table(lib().gtap_table_fib_cutoff(cutoff, num_queues), "fib_cutoff", GTAP_WORKER_THREAD)

    @staticmethod
    def tree(kind: int, D: int, B: int, seed: int, buf, mem_ops: int, compute_iters: int, total) -> "Table":
        """Synthetic tree (B = 0: full binary; else pruned B-ary); buf: CUDA int64/uint64 tensor of
        power-of-two length, total: CUDA int64 tensor of 32 zeros."""
        import torch
        for t, n in ((buf, "buf"), (total, "total")):
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.int64 and t.is_contiguous()):
                raise TypeError(f"{n} must be a contiguous CUDA int64 tensor")
        if total.numel() < 32:
            raise ValueError("total must hold 32 counters")
        h = lib().gtap_table_tree(kind, D, B, seed & ((1 << 64) - 1), buf.data_ptr(), buf.numel(), mem_ops,
                                  compute_iters, total.data_ptr())
        return Table(h, f"tree_{'thread' if kind == GTAP_WORKER_THREAD else 'block'}", kind, (buf, total))

    @staticmethod
    def nqueens(n: int, cutoff: int, count, leaf_mode: int = 1) -> "Table":
        """N-Queens; `count` is a CUDA int64 tensor of one element the run adds solutions to;
        leaf_mode 0 = serial leaf on the task's lane (paper), 1 = the warp counts the leaf."""
        return Table(lib().gtap_table_nqueens_ex(n, cutoff, count.data_ptr(), leaf_mode), "nqueens",
                     GTAP_WORKER_THREAD, (count,))

    @staticmethod
    def mergesort(keys, scratch, cutoff: int = 128, merge_mode: int = 1) -> "Table":
        """merge_mode: GTAP_MERGE_WARP (1, default) or GTAP_MERGE_THREAD (0, the paper's one-lane merge)."""
        _dev_i32(keys, "keys"); _dev_i32(scratch, "scratch")
        if scratch.numel() < keys.numel():
            raise ValueError("scratch must hold n keys")
        return Table(lib().gtap_table_mergesort_ex(keys.data_ptr(), scratch.data_ptr(), keys.numel(), cutoff,
                                                   merge_mode),
                     "mergesort", GTAP_WORKER_THREAD, (keys, scratch))

    @staticmethod
    def cilksort(keys, scratch, cut_sort: int = 64, cut_merge: int = 256, merge_mode: int = 1) -> "Table":
        _dev_i32(keys, "keys"); _dev_i32(scratch, "scratch")
        if scratch.numel() < keys.numel():
            raise ValueError("scratch must hold n keys")
        return Table(lib().gtap_table_cilksort_ex(keys.data_ptr(), scratch.data_ptr(), keys.numel(), cut_sort, cut_merge,
                                                  merge_mode),
                     "cilksort", GTAP_WORKER_THREAD, (keys, scratch))

    @staticmethod
    def spmv(row_ptr, col, val, x, y, nnz_cut: int = 8192, fanout: int = 16) -> "Table":
        for t, n in ((row_ptr, "row_ptr"), (col, "col")):
            _dev_i32(t, n)
        nrows = row_ptr.numel() - 1
        return Table(lib().gtap_table_spmv(row_ptr.data_ptr(), col.data_ptr(), val.data_ptr(), x.data_ptr(),
                                           y.data_ptr(), nrows, nnz_cut, fanout),
                     "spmv", GTAP_WORKER_BLOCK, (row_ptr, col, val, x, y))

    @staticmethod
    def bfs(row_ptr, col, depth, order: int = 0, edge_split: int = 0) -> "Table":
        """order 0: the paper's LIFO owner pops; 1: oldest-first pops (see gtap.h gtap_table_bfs_ex);
        edge_split > 0: hubs' edge lists cut into bfs_edges pieces (gtap.h gtap_table_bfs_split)."""
        _dev_i32(row_ptr, "row_ptr"); _dev_i32(col, "col"); _dev_i32(depth, "depth")
        return Table(lib().gtap_table_bfs_split(row_ptr.data_ptr(), col.data_ptr(), depth.data_ptr(), depth.numel(),
                                                order, edge_split), "bfs", GTAP_WORKER_BLOCK, (row_ptr, col, depth))


def _dev_i32(t, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.int32 and t.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous CUDA int32 tensor")


@dataclass
class RunStats:
    tasks: int
    invocations: int
    pops: int
    kept: int
    steals_ok: int
    steals_failed: int
    stolen_tasks: int
    pushes: int
    cycles: int
    idle_cycles: int
    remote_frees: int
    max_pool_used: int
    error_word: int
    workers: int
    device_ms: float
    grid_size: int
    block_size: int
    assists: int = 0


class Runtime:
    """gtap_init / gtap_finalize around a torch-allocated workspace."""

    def __init__(self, kind: int, device: int = 0, *, grid_size: int = 0, block_size: int = 0,
                 max_tasks_per_worker: int = 0, queue_capacity: int = 0, steal_attempts: int = 0,
                 steal_max: int = 0, seed: int = 0x5EED, watchdog_ns: int = 0, max_roots: int = 0,
                 idle_backoff_ns: int = 0, num_queues: int = 0, max_child_tasks: int = 0, queue_policy: int = 0,
                 victim_policy: int = 0,
                 torch_workspace: bool = True):
        import torch
        L = lib()
        cfg = Config()
        _check(L.gtap_config_default(ctypes.byref(cfg), device, kind), "gtap_config_default")
        for k, v in dict(grid_size=grid_size, block_size=block_size, max_tasks_per_worker=max_tasks_per_worker,
                         queue_capacity=queue_capacity, steal_attempts=steal_attempts, steal_max=steal_max,
                         watchdog_ns=watchdog_ns, max_roots=max_roots, idle_backoff_ns=idle_backoff_ns,
                         num_queues=num_queues, max_child_tasks=max_child_tasks, queue_policy=queue_policy,
                         victim_policy=victim_policy).items():
            if v:
                setattr(cfg, k, v)
        cfg.seed = seed
        self.cfg = cfg
        self.kind = kind
        self.device = device
        nbytes = L.gtap_workspace_bytes(ctypes.byref(cfg))
        if nbytes == 0:
            raise GtapError(1, "gtap_workspace_bytes")
        self.workspace = None
        ptr = None
        if torch_workspace:
            self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=f"cuda:{device}")
            ptr = (self.workspace.data_ptr() + 255) // 256 * 256
        h = ctypes.c_void_p()
        _check(L.gtap_init(ctypes.byref(cfg), ptr, nbytes, ctypes.byref(h)), "gtap_init")
        self.h = h.value
        self.workspace_bytes = nbytes

    def spawn_root(self, table: Table, args=(), fn: int = 0) -> int:
        words = (ctypes.c_uint32 * 4)(*[int(a) & 0xFFFFFFFF for a in args])
        idx = ctypes.c_uint32()
        _check(lib().gtap_spawn_root(self.h, table.ptr, fn, words, 4 * len(args), ctypes.byref(idx)),
               "gtap_spawn_root")
        return idx.value

    def run(self, stream=None):
        _check(lib().gtap_run(self.h, _stream_ptr(stream)), "gtap_run")

    def sync(self, raise_on_error: bool = True) -> RunStats:
        st = Stats()
        code = lib().gtap_sync(self.h, ctypes.byref(st))
        if raise_on_error:
            _check(code, "gtap_sync")
        d = st.as_dict()
        return RunStats(**d)

    def reset(self, stream=None):
        _check(lib().gtap_reset(self.h, _stream_ptr(stream)), "gtap_reset")

    def root_result(self, idx: int = 0) -> int:
        v = ctypes.c_int64()
        _check(lib().gtap_root_result(self.h, idx, ctypes.byref(v), 8), "gtap_root_result")
        return v.value

    CHECK_FIELDS = ("allocs", "frees", "publications", "dispatches", "suspends", "joins", "continuations",
                    "v_double_alloc", "v_double_free", "v_double_publish", "v_dispatch_unpublished",
                    "v_early_resume", "v_join_underflow", "v_suspend_dirty", "_r14", "_r15",
                    "live_records", "published_unclaimed", "join_counts_open", "outstanding", "roots_left")

    def check_read(self) -> dict:
        """Scheduler-invariant counters of the last run (GTAP_CHECK build only; else GtapError UNSUPPORTED)."""
        buf = (ctypes.c_uint64 * 21)()
        _check(lib().gtap_check_read(self.h, buf, 21), "gtap_check_read")
        return {k: int(v) for k, v in zip(self.CHECK_FIELDS, buf) if not k.startswith("_")}

    def geometry(self, table: Table):
        W, g, b = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        _check(lib().gtap_geometry(self.h, table.ptr, ctypes.byref(W), ctypes.byref(g), ctypes.byref(b)),
               "gtap_geometry")
        return W.value, g.value, b.value

    def close(self):
        if getattr(self, "h", None):
            lib().gtap_finalize(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ubench_atomics(buf, kind: int, grid: int, block: int, ops_per_thread: int, stream=None) -> float:
    """Kernel ms of the L2-atomic probe `kind` (see gtap.h) over the int32 CUDA tensor buf."""
    ms = ctypes.c_float()
    _check(lib().gtap_ubench_atomics(buf.data_ptr(), buf.numel(), kind, grid, block, ops_per_thread,
                                     _stream_ptr(stream), ctypes.byref(ms)), "gtap_ubench_atomics")
    return ms.value


def ubench_die_probe(buf, n_addr: int = 256, stream=None) -> dict:
    """SM -> L2-die map measured over n_addr addresses of the CUDA tensor buf (gtap.h gtap_ubench_die_probe)."""
    import numpy as np
    sm_die = np.zeros(256, np.uint8)
    near = np.zeros(n_addr, np.uint8)
    out3 = np.zeros(3, np.float32)
    _check(lib().gtap_ubench_die_probe(buf.data_ptr(), buf.numel() * buf.element_size(), n_addr,
                                       sm_die.ctypes.data, 256, near.ctypes.data, out3.ctypes.data,
                                       _stream_ptr(stream)), "gtap_ubench_die_probe")
    return dict(sm_die=sm_die, addr_near=near, near_cycles=float(out3[0]), far_cycles=float(out3[1]),
                consistency=float(out3[2]))


def bfs_init_depth(depth, src: int, stream=None):
    """depth[:] = INT32_MAX, depth[src] = 0 on the device (libgtap kernel)."""
    _dev_i32(depth, "depth")
    _check(lib().gtap_bfs_init_depth(depth.data_ptr(), depth.numel(), src, _stream_ptr(stream)),
           "gtap_bfs_init_depth")
