"""The N>1 host path with world_size 2 on the gloo backend (CPU): partitioning, the single
final gather, max-over-ranks timing. Each rank computes its shard with the CPU oracle in place
of the GPU (the GPU-side work per rank is the 1-GPU path already covered by the -m gpu tests).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_05982_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def spmv_shard(rank, world):
    import oracle
    import synth
    rp, col, val, x = synth.powerlaw_csr(20000, seed=3)
    ranges = shard.split_rows_by_nnz(rp, world)
    lo, hi = ranges[rank]
    # this rank's row slice of the CSR (x replicated)
    rps = rp[lo: hi + 1] - rp[lo]
    cs, vs = col[int(rp[lo]): int(rp[hi])], val[int(rp[lo]): int(rp[hi])]
    _, y_local = oracle.spmv(rps, cs, vs, x)
    y = shard.gather_slices(torch.from_numpy(y_local), ranges, rank)
    _, y_full = oracle.spmv(rp, col, val, x)
    t = shard.max_over_ranks(1.0 + rank)
    return bool(np.array_equal(y.numpy(), y_full)), t, ranges


def forest_shard(rank, world):
    import oracle
    import synth
    n_arrays = 7
    mine = shard.split_round_robin(n_arrays, world, rank)
    sums = torch.zeros(n_arrays, dtype=torch.int64)
    ok = True
    for i in mine:
        keys = synth.keys_int32(5000 + 13 * i, seed=100 + i).numpy()
        out, _, _ = oracle.mergesort(keys, 128)
        ok &= bool(np.all(out[1:] >= out[:-1]))
        sums[i] = int(out.astype(np.int64).sum())
    dist.all_reduce(sums)  # the one gather of per-array checksums
    ref = [int(synth.keys_int32(5000 + 13 * i, seed=100 + i).numpy().astype(np.int64).sum()) for i in range(n_arrays)]
    return ok and sums.tolist() == ref


@pytest.mark.timeout(300)
def test_spmv_row_partition_world2():
    out = run_world(spmv_shard)
    for r in (0, 1):
        ok, t, ranges = out[r]
        assert ok, out
        assert t == 2.0  # max over ranks
    assert ranges[0][0] == 0 and ranges[-1][1] == 20000 and ranges[0][1] == ranges[1][0]


@pytest.mark.timeout(300)
def test_forest_round_robin_world2():
    out = run_world(forest_shard)
    assert out[0] is True and out[1] is True, out


def test_split_rows_balanced():
    import synth
    rp, _, _, _ = synth.powerlaw_csr(1 << 14, seed=5)
    for world in (1, 2, 3, 4, 8):
        ranges = shard.split_rows_by_nnz(rp, world)
        assert ranges[0][0] == 0 and ranges[-1][1] == (1 << 14)
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
        nnz = [int(rp[hi] - rp[lo]) for lo, hi in ranges]
        maxdeg = int((rp[1:] - rp[:-1]).max())
        assert max(nnz) - min(nnz) <= 2 * maxdeg


def test_split_round_robin():
    assert shard.split_round_robin(7, 2, 0) == [0, 2, 4, 6]
    assert shard.split_round_robin(7, 2, 1) == [1, 3, 5]
    with pytest.raises(ValueError):
        shard.split_round_robin(3, 2, 2)


def bfs_source_split(rank, world):
    """C5a at N ranks: the graph replicated, 16 sources dealt round robin, one gather of per-source rows."""
    import oracle
    import synth
    rp, col = synth.rmat_csr(10, 16, seed=3)
    srcs = synth.bfs_sources(rp, 16, seed=5)
    mine = shard.split_round_robin(16, world, rank)
    rows = []
    for k in mine:
        lv = oracle.bfs(rp, col, srcs[k])
        reached = lv != 0x7FFFFFFF
        rows.append([float(k), float(reached.sum()), float(lv[reached].astype(np.int64).sum())])
    return shard.gather_round_robin(rows, 16, world, rank)


def fib_forest_split(rank, world):
    """A fib forest at N ranks: roots dealt round robin, one gather of the 4-B root results."""
    import oracle
    ns = [5 + (k % 11) for k in range(13)]
    mine = shard.split_round_robin(len(ns), world, rank)
    return shard.gather_round_robin([[float(oracle.fib(ns[k])[0])] for k in mine], len(ns), world, rank)


@pytest.mark.timeout(300)
def test_bfs_sources_split_world2():
    import oracle
    import synth
    out = run_world(bfs_source_split)
    rp, col = synth.rmat_csr(10, 16, seed=3)
    srcs = synth.bfs_sources(rp, 16, seed=5)
    for r in (0, 1):
        rows = out[r]
        assert isinstance(rows, list) and len(rows) == 16, rows
        for k, row in enumerate(rows):
            lv = oracle.bfs(rp, col, srcs[k])
            reached = lv != 0x7FFFFFFF
            assert row == [float(k), float(reached.sum()), float(lv[reached].astype(np.int64).sum())]


@pytest.mark.timeout(300)
def test_fib_forest_split_world3():
    out = run_world(fib_forest_split, world=3)
    ns = [5 + (k % 11) for k in range(13)]
    fibs = [0, 1]
    while len(fibs) < 20:
        fibs.append(fibs[-1] + fibs[-2])
    for r in range(3):
        assert out[r] == [[float(fibs[n])] for n in ns], out[r]


def test_gather_round_robin_single_rank():
    rows = [[float(k), 2.0 * k] for k in range(5)]
    assert shard.gather_round_robin(rows, 5, 1, 0) == rows
    with pytest.raises(ValueError):
        shard.gather_round_robin(rows[:3], 5, 1, 0)


def test_bench_world_size_mismatch_fails():
    """bench.py refuses a world size other than --gpus (the driver's N must be the ranks that ran)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert p.returncode != 0 and "world size 1 != --gpus 2" in p.stderr


@pytest.mark.timeout(600)
def test_bench_reference_self_launch_two_ranks():
    """bench.py --gpus 2 outside torchrun re-launches itself as 2 ranks; rank 0 alone prints the line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--steps", "1", "--warmup", "0"], env=env, capture_output=True, text=True, timeout=540)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
