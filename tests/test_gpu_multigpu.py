"""Multi-GPU on real GPUs: NCCL ranks, each running its shard through the C ABI.

The NCCL tests skip below 2 visible GPUs (gpurun and the round-end driver give one GPU; the 2-rank host
logic is covered on CPU with gloo in test_multiproc.py, and the same 2-rank program runs on ONE GPU with gloo
collectives in test_forests_and_spmv_two_ranks_one_gpu_gloo). With >= 2 GPUs:

* each rank runs its round-robin share of a fib forest and of a mergesort forest in ONE launch, the
  per-root results travel in one all_gather, and rank 0 compares every root with the oracle;
* SpMV rows split by nnz, one all_gather of y, per-row 1e-5 gate against the fp64 oracle;
* `bench.py --gpus 2` (self-launching two ranks) prints n_gpus 2 and a correct line.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


needs2 = pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs (gpurun gives one)")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, backend="nccl"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import synth
    import paper_2604_05982_b200 as g
    from paper_2604_05982_b200 import shard
    # nccl: one GPU per rank; gloo (one-GPU test mode): every rank's CUDA work on cuda:0, collectives on the CPU
    gpu = rank if backend == "nccl" else 0
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    cdev = dev if backend == "nccl" else torch.device("cpu")
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        # fib forest: 10 roots of varying n
        ns = [10 + k for k in range(10)]
        mine = shard.split_round_robin(len(ns), world, rank)
        vals, _ = g.fib_forest([ns[k] for k in mine], device=gpu, grid_size=148, block_size=128,
                               max_tasks_per_worker=4096)
        fibs = shard.gather_round_robin([[float(v)] for v in vals], len(ns), world, rank, cdev)
        # mergesort forest: 6 arrays of ragged sizes, one root per array
        sizes = [1000 + 777 * k for k in range(6)]
        mine = shard.split_round_robin(len(sizes), world, rank)
        parts = [synth.keys_int32(sizes[k], seed=50 + k, device=dev) for k in mine]
        keys = torch.cat(parts)
        offs = np.cumsum([0] + [sizes[k] for k in mine]).tolist()
        g.mergesort_forest_(keys, [(offs[j], offs[j + 1]) for j in range(len(mine))], grid_size=148,
                            block_size=128, max_tasks_per_worker=1024)
        rows = [[float(keys[offs[j]:offs[j + 1]].to(torch.int64).sum().item()),
                 float(bool(torch.all(keys[offs[j] + 1:offs[j + 1]] >= keys[offs[j]:offs[j + 1] - 1]).item())),
                 float(keys[offs[j]].item()), float(keys[offs[j + 1] - 1].item())] for j in range(len(mine))]
        arrays = shard.gather_round_robin(rows, len(sizes), world, rank, cdev)
        # SpMV row partition, one all_gather of y
        rp, col, val, x = synth.powerlaw_csr(1 << 14, seed=7, device=dev)
        ranges = shard.split_rows_by_nnz(rp.cpu(), world)
        lo, hi = ranges[rank]
        y, _ = g.spmv(rp, col, val, x, torch.zeros(1 << 14, device=dev), 2048, 16, rows=(lo, hi),
                      grid_size=148, block_size=128, max_tasks_per_worker=1024)
        yfull = shard.gather_slices(y[lo:hi].contiguous().to(cdev), ranges, rank)
        q.put((rank, fibs, arrays, yfull.cpu().numpy()))
    except Exception as e:
        q.put((rank, repr(e), None, None))
    finally:
        dist.destroy_process_group()


def _two_ranks(backend):
    import torch.multiprocessing as mp

    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, backend)) for r in range(2)]
    for p in procs:
        p.start()
    out = {r: (f, a, y) for r, f, a, y in (q.get(timeout=300) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
    ns = [10 + k for k in range(10)]
    sizes = [1000 + 777 * k for k in range(6)]
    rp, col, val, x = synth.powerlaw_csr(1 << 14, seed=7)
    y64, _ = oracle.spmv(rp, col, val, x)
    for r in (0, 1):
        fibs, arrays, y = out[r]
        assert not isinstance(fibs, str), fibs
        assert [int(v[0]) for v in fibs] == [oracle.fib(n)[0] for n in ns]
        for k, row in enumerate(arrays):
            ref, _, _ = oracle.mergesort(synth.keys_int32(sizes[k], seed=50 + k).numpy(), 128)
            assert row == [float(ref.astype(np.int64).sum()), 1.0, float(ref[0]), float(ref[-1])]
        err = np.abs(y.astype(np.float64) - y64) / np.maximum(np.abs(y64), 1e-30)
        assert np.all((y64 == 0) & (y == 0) | (err <= 1e-5))


@needs2
@pytest.mark.timeout(600)
def test_forests_and_spmv_two_ranks_nccl():
    _two_ranks("nccl")


@pytest.mark.timeout(600)
def test_forests_and_spmv_two_ranks_one_gpu_gloo():
    """The same two-rank program on ONE GPU (gpurun and the round-end driver give one): both ranks run their
    shards through the C ABI on cuda:0 (independent persistent kernels: no rank waits on another's kernel),
    gloo carries the gathers on the CPU; every root and row is checked against the oracle."""
    _two_ranks("gloo")


@needs2
@pytest.mark.timeout(900)
def test_bench_two_gpus():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup",
                        "3", "--no-cpu-baseline"], env=env, capture_output=True, text=True, timeout=840)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["correct"] and d["config"]["arrays_total"] == 2
    assert d["summary"]["fib_forest"]["correct"]
