"""Multi-GPU partitioning of the GTaP workloads (host logic).

Only workloads that shard naturally are split; nothing on the scheduler path
crosses GPUs (BASELINE north_star: no cross-GPU stealing or atomics):

* independent roots (fib forests, mergesort forests, BFS sources): round-robin
  over ranks, weak or strong scaling, results gathered once at the end;
* SpMV: contiguous row ranges balanced by non-zeros (a binary search of
  row_ptr for k * nnz / world), x replicated, each rank writes its y slice,
  ONE all_gather of the (padded) slices after the timed region.

These helpers take ranks / world sizes as plain ints so they run the same with
the gloo backend on CPU (tests) and NCCL on B200s (bench.py under torchrun).
"""
from __future__ import annotations

import bisect


def split_round_robin(n_items: int, world: int, rank: int) -> list[int]:
    """Indices of the items rank `rank` owns when n_items independent roots are dealt out."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return list(range(rank, n_items, world))


def split_rows_by_nnz(row_ptr, world: int) -> list[tuple[int, int]]:
    """Contiguous row ranges [(lo, hi)] covering all rows, balanced by non-zeros.

    Boundary k is the first row whose start offset reaches k * nnz / world (binary search on
    row_ptr), so each rank's nnz is within one row of nnz / world.
    """
    rp = [int(v) for v in (row_ptr.tolist() if hasattr(row_ptr, "tolist") else row_ptr)]
    nrows = len(rp) - 1
    nnz = rp[-1]
    bounds = [0]
    for k in range(1, world):
        target = (nnz * k) // world
        r = bisect.bisect_left(rp, target, lo=bounds[-1], hi=nrows)
        bounds.append(min(max(r, bounds[-1]), nrows))
    bounds.append(nrows)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


def gather_slices(local, ranges, rank: int, group=None):
    """all_gather of per-rank 1-D slices of different lengths (padded to the longest).

    `local` is this rank's slice (a torch tensor on the process group's device);
    returns the concatenation in rank order (the full vector) on every rank.
    """
    import torch
    import torch.distributed as dist
    world = len(ranges)
    width = max(hi - lo for lo, hi in ranges)
    pad = torch.zeros(width, dtype=local.dtype, device=local.device)
    pad[: local.numel()] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([bufs[i][: ranges[i][1] - ranges[i][0]] for i in range(world)])


def max_over_ranks(x: float, device="cpu", group=None) -> float:
    """Device time of a multi-rank run = max over ranks (the slowest rank ends the job)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_round_robin(rows, n_items: int, world: int, rank: int, device="cpu", group=None):
    """all_gather of per-item result rows of round-robin-dealt items -> list indexed by item.

    `rows[j]` is this rank's row (a list of floats, all rows of one width) for item
    split_round_robin(n_items, world, rank)[j]. Each rank pads its rows to the largest share, ONE
    all_gather moves them, and the rows are put back in item order on every rank.
    """
    import torch
    import torch.distributed as dist
    mine = split_round_robin(n_items, world, rank)
    if len(rows) != len(mine):
        raise ValueError("one row per owned item")
    width = len(rows[0]) if rows else 0
    widths = torch.tensor([width], dtype=torch.int64, device=device)
    if world > 1:
        dist.all_reduce(widths, op=dist.ReduceOp.MAX, group=group)
    width = int(widths.item())
    share = len(split_round_robin(n_items, world, 0))
    flat = torch.zeros(share * width, dtype=torch.float64, device=device)
    if rows:
        flat[: len(rows) * width] = torch.tensor([float(v) for r in rows for v in r], dtype=torch.float64)
    if world > 1:
        bufs = [torch.empty_like(flat) for _ in range(world)]
        dist.all_gather(bufs, flat, group=group)
    else:
        bufs = [flat]
    out = [None] * n_items
    for r in range(world):
        b = bufs[r].view(share, width).tolist() if width else [[] for _ in range(share)]
        for j, k in enumerate(split_round_robin(n_items, world, r)):
            out[k] = b[j]
    return out
