"""B200-native GTaP hot path: a persistent-kernel fork-join scheduler (sm_100a).

User-facing calls (each runs the whole path in libgtap.so's CUDA kernels and
fails loudly when the library or the GPU is missing -- there is no CPU path):

    fib(n)                       -> (F(n), stats)      thread-level
    fib_forest([n, ...])         -> ([F(n)], stats)    independent roots (forest)
    mergesort_(keys)             -> stats (in place)   thread-level
    mergesort_forest_(keys, seg) -> stats              independent roots (forest)
    spmv(row_ptr, col, val, x)   -> (y, stats)         block-level
    bfs(row_ptr, col, src)       -> (depth, stats)     block-level
    tree(D, buf, mem, comp)      -> (sum, stats)       thread- or block-level
    nqueens(n) / cilksort_(keys) / fib_cutoff(n, c)    NEXT rows

Lower level: gtap.Runtime / gtap.Table mirror include/gtap.h one to one.
"""
from __future__ import annotations

from . import gtap
from .gtap import (GTAP_WORKER_BLOCK, GTAP_WORKER_THREAD, GtapError, Runtime, RunStats, Table,
                   bfs_init_depth, ubench_atomics)

__all__ = ["gtap", "Runtime", "Table", "RunStats", "GtapError", "fib", "fib_forest", "fib_cutoff", "nqueens", "tree", "mergesort_", "cilksort_", "mergesort_forest_",
           "spmv", "bfs", "ubench_atomics", "GTAP_WORKER_THREAD", "GTAP_WORKER_BLOCK"]


def _runtime(kind, rt, device, cfg):
    if rt is not None:
        return rt, False
    return Runtime(kind, device, **cfg), True


def fib(n: int, rt: Runtime | None = None, device: int = 0, stream=None, **cfg):
    """fib(n) as the paper's no-cutoff task program on thread-level workers."""
    rt, own = _runtime(GTAP_WORKER_THREAD, rt, device, cfg)
    table = Table.fib()
    try:
        rt.spawn_root(table, (n,))
        rt.run(stream)
        st = rt.sync()
        return rt.root_result(0), st
    finally:
        table.close()
        if own:
            rt.close()


def fib_forest(ns, rt: Runtime | None = None, device: int = 0, stream=None, **cfg):
    """A forest of independent fib roots in ONE run (root r starts on worker r mod W):
    returns ([F(n) for n in ns], stats)."""
    cfg.setdefault("max_roots", max(len(ns), 1))
    rt, own = _runtime(GTAP_WORKER_THREAD, rt, device, cfg)
    table = Table.fib()
    try:
        for n in ns:
            rt.spawn_root(table, (n,))
        rt.run(stream)
        st = rt.sync()
        return [rt.root_result(i) for i in range(len(ns))], st
    finally:
        table.close()
        if own:
            rt.close()


def fib_cutoff(n: int, cutoff: int, num_queues: int = 1, rt: Runtime | None = None, device: int = 0, stream=None,
               **cfg):
    """fib(n) with a cutoff; num_queues=3 enables EPAQ with the paper's classifier."""
    cfg.setdefault("num_queues", num_queues)
    rt, own = _runtime(GTAP_WORKER_THREAD, rt, device, cfg)
    table = Table.fib_cutoff(cutoff, num_queues)
    try:
        rt.spawn_root(table, (n,))
        rt.run(stream)
        st = rt.sync()
        return rt.root_result(0), st
    finally:
        table.close()
        if own:
            rt.close()


def nqueens(n: int, cutoff: int = 7, leaf_mode: int = 1, rt: Runtime | None = None, device: int = 0, stream=None,
            **cfg):
    """Number of n-queens solutions by the paper's bitmask task program; returns (count, stats)."""
    import torch
    count = torch.zeros(1, dtype=torch.int64, device=f"cuda:{device}")
    rt, own = _runtime(GTAP_WORKER_THREAD, rt, device, cfg)
    table = Table.nqueens(n, cutoff, count, leaf_mode)
    try:
        rt.spawn_root(table, ())
        rt.run(stream)
        st = rt.sync()
        return int(count.item()), st
    finally:
        table.close()
        if own:
            rt.close()


def tree(D: int, buf, mem_ops: int, compute_iters: int, pruned: bool = False, B: int = 3, seed: int = 1,
         worker: int = GTAP_WORKER_THREAD, rt: Runtime | None = None, stream=None, **cfg):
    """Synthetic tree on thread- or block-level workers.

    Returns (sum of do_memory_and_compute over all nodes mod 2^64, stats); buf: CUDA int64 tensor of
    power-of-two length (the words the pseudo-random loads read)."""
    import torch
    total = torch.zeros(32, dtype=torch.int64, device=buf.device)
    rt, own = _runtime(worker, rt, buf.device.index or 0, cfg)
    table = Table.tree(worker, D, B if pruned else 0, seed, buf, mem_ops, compute_iters, total)
    try:
        rt.spawn_root(table, (0 if pruned else 1, 0, 0))
        rt.run(stream)
        st = rt.sync()
        return int(total.sum().item()) & ((1 << 64) - 1), st
    finally:
        table.close()
        if own:
            rt.close()


def mergesort_(keys, scratch=None, cutoff: int = 128, merge_mode: int = 1, rt: Runtime | None = None, stream=None,
               **cfg):
    """Sort a CUDA int32 tensor in place with the cutoff mergesort task program
    (merge_mode 1: heavy merges run by the task's whole warp; 0: the paper's one-lane merge)."""
    import torch
    if scratch is None:
        scratch = torch.empty_like(keys)
    rt, own = _runtime(GTAP_WORKER_THREAD, rt, keys.device.index or 0, cfg)
    table = Table.mergesort(keys, scratch, cutoff, merge_mode)
    try:
        rt.spawn_root(table, (0, keys.numel()))
        rt.run(stream)
        return rt.sync()
    finally:
        table.close()
        if own:
            rt.close()


def cilksort_(keys, scratch=None, cut_sort: int = 64, cut_merge: int = 256, merge_mode: int = 1,
              rt: Runtime | None = None, stream=None,
              **cfg):
    """Sort a CUDA int32 tensor in place with Cilksort (parallel merge)."""
    import torch
    if scratch is None:
        scratch = torch.empty_like(keys)
    rt, own = _runtime(GTAP_WORKER_THREAD, rt, keys.device.index or 0, cfg)
    table = Table.cilksort(keys, scratch, cut_sort, cut_merge, merge_mode)
    try:
        rt.spawn_root(table, (0, keys.numel()))
        rt.run(stream)
        return rt.sync()
    finally:
        table.close()
        if own:
            rt.close()


def mergesort_forest_(keys, segments, scratch=None, cutoff: int = 128, merge_mode: int = 1, rt: Runtime | None = None,
                      stream=None, **cfg):
    """Sort independent segments [(l, r), ...] of one CUDA int32 tensor: one root per segment."""
    import torch
    if scratch is None:
        scratch = torch.empty_like(keys)
    cfg.setdefault("max_roots", max(len(segments), 1))
    rt, own = _runtime(GTAP_WORKER_THREAD, rt, keys.device.index or 0, cfg)
    table = Table.mergesort(keys, scratch, cutoff, merge_mode)
    try:
        for l, r in segments:
            rt.spawn_root(table, (l, r))
        rt.run(stream)
        return rt.sync()
    finally:
        table.close()
        if own:
            rt.close()


def spmv(row_ptr, col, val, x, y=None, nnz_cut: int = 8192, fanout: int = 16, rows=None, parts: int = 0,
         rt: Runtime | None = None, stream=None, **cfg):
    """y = A x for a CSR matrix with block-cooperative task leaves.

    rows=(lo, hi) restricts the work to a row range; parts=R > 0 spawns a forest of R roots
    part(k, R, lo, hi) (nnz-balanced row ranges found in the kernel) instead of one root."""
    import torch
    if y is None:
        y = torch.empty(row_ptr.numel() - 1, dtype=torch.float32, device=row_ptr.device)
    if parts:
        cfg.setdefault("max_roots", parts)
    rt, own = _runtime(GTAP_WORKER_BLOCK, rt, row_ptr.device.index or 0, cfg)
    table = Table.spmv(row_ptr, col, val, x, y, nnz_cut, fanout)
    lo, hi = rows if rows is not None else (0, row_ptr.numel() - 1)
    try:
        if parts:
            for k in range(parts):
                rt.spawn_root(table, (k, parts, lo, hi), fn=1)
        else:
            rt.spawn_root(table, (lo, hi))
        rt.run(stream)
        return y, rt.sync()
    finally:
        table.close()
        if own:
            rt.close()


def bfs(row_ptr, col, src: int, depth=None, rt: Runtime | None = None, stream=None, order: int = 0,
        edge_split: int = 0, **cfg):
    """BFS levels from src (INT32_MAX = unreached) by the paper's frontier-expansion tasks
    (order 0: LIFO owner pops as in the paper; 1: oldest-first pops, gtap.h gtap_table_bfs_ex;
    edge_split > 0: a vertex with more edges hands pieces of its edge list to bfs_edges tasks)."""
    import torch
    nv = row_ptr.numel() - 1
    if depth is None:
        depth = torch.empty(nv, dtype=torch.int32, device=row_ptr.device)
    rt, own = _runtime(GTAP_WORKER_BLOCK, rt, row_ptr.device.index or 0, cfg)
    table = Table.bfs(row_ptr, col, depth, order, edge_split)
    try:
        bfs_init_depth(depth, src, stream)
        rt.spawn_root(table, (src,))
        rt.run(stream)
        return depth, rt.sync()
    finally:
        table.close()
        if own:
            rt.close()
