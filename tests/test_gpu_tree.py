"""GPU parity: synthetic trees on both worker kinds vs the oracle.

The per-node value (mem_ops 64-bit loads + compute_iters FP64 FMAs) is integer-combined mod 2^64,
so the comparison is exact: the total over all nodes and the task count must equal the oracle's.
The FMA chains are the same IEEE operations on both sides (fma() in C, __fma_rn on the GPU).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
WD = 60_000_000_000


@pytest.fixture(scope="module")
def g(cuda_device):
    import paper_2604_05982_b200 as g
    return g


@pytest.fixture(scope="module")
def buf_cpu():
    return synth.tree_buffer(1 << 14)


@pytest.fixture(scope="module")
def buf(buf_cpu):
    return buf_cpu.to("cuda")


def _np(b):
    return b.numpy().view(np.uint64)


@pytest.fixture(scope="module")
def rts(g):
    rt = g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148 * 4, block_size=128, max_tasks_per_worker=4096,
                   watchdog_ns=WD)
    rb = g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148 * 8, block_size=64, max_tasks_per_worker=1024,
                   watchdog_ns=WD)
    yield {"thread": rt, "block": rb}
    rt.close()
    rb.close()


KINDS = ["thread", "block"]


def _kind(g, k):
    return g.GTAP_WORKER_THREAD if k == "thread" else g.GTAP_WORKER_BLOCK


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("D", [0, 1, 2, 7, 12])
@pytest.mark.parametrize("mem,comp", [(0, 0), (3, 0), (0, 5), (7, 65), (33, 200)])
def test_full_tree(g, rts, buf, buf_cpu, kind, D, mem, comp):
    total, st = g.tree(D, buf, mem, comp, worker=_kind(g, kind), rt=rts[kind])
    ot, otasks = oracle.tree(D, _np(buf_cpu), mem, comp)
    assert total == ot
    assert st.tasks == otasks == 2 ** (D + 1) - 1
    assert st.invocations == otasks + (2 ** D - 1)   # internal nodes resume once after the join


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("D,seed", [(1, 1), (4, 2), (9, 3), (14, 4)])
@pytest.mark.parametrize("mem,comp", [(0, 0), (5, 70)])
def test_pruned_tree(g, rts, buf, buf_cpu, kind, D, seed, mem, comp):
    total, st = g.tree(D, buf, mem, comp, pruned=True, seed=seed, worker=_kind(g, kind), rt=rts[kind])
    assert (total, st.tasks) == oracle.tree(D, _np(buf_cpu), mem, comp, pruned=True, seed=seed)


@pytest.mark.parametrize("B", [1, 2, 5, 8])
@pytest.mark.parametrize("kind", KINDS)
def test_pruned_branching(g, rts, buf, buf_cpu, kind, B):
    total, st = g.tree(8, buf, 4, 40, pruned=True, B=B, seed=11, worker=_kind(g, kind), rt=rts[kind])
    assert (total, st.tasks) == oracle.tree(8, _np(buf_cpu), 4, 40, pruned=True, B=B, seed=11)


@pytest.mark.parametrize("kind,grid,block", [("thread", 1, 32), ("thread", 37, 64), ("thread", 148 * 2, 256),
                                             ("block", 1, 32), ("block", 37, 128), ("block", 148 * 4, 256),
                                             ("block", 148, 1024)])
def test_geometry(g, buf, buf_cpu, kind, grid, block):
    with g.Runtime(_kind(g, kind), 0, grid_size=grid, block_size=block, max_tasks_per_worker=4096,
                   watchdog_ns=WD) as r:
        total, st = g.tree(10, buf, 9, 130, worker=_kind(g, kind), rt=r)
        assert (total, st.tasks) == oracle.tree(10, _np(buf_cpu), 9, 130)
        total, st = g.tree(11, buf, 9, 130, pruned=True, seed=5, worker=_kind(g, kind), rt=r)
        assert (total, st.tasks) == oracle.tree(11, _np(buf_cpu), 9, 130, pruned=True, seed=5)


@pytest.mark.parametrize("kind", KINDS)
def test_bench_size(g, kind):
    """The bench's shapes (full D = 22: 8.4M tasks; pruned D = 28), lighter per-node work so the
    oracle finishes in seconds; bench launch configuration."""
    b_cpu = synth.tree_buffer(1 << 20)
    b = b_cpu.to("cuda")
    cfg = dict(grid_size=0, block_size=128, max_tasks_per_worker=4096) if kind == "thread" else \
        dict(grid_size=148 * 8, block_size=64, max_tasks_per_worker=1024)
    with g.Runtime(_kind(g, kind), 0, watchdog_ns=WD, **cfg) as r:
        total, st = g.tree(22, b, 2, 8, worker=_kind(g, kind), rt=r)
        assert (total, st.tasks) == oracle.tree(22, _np(b_cpu), 2, 8)
        total, st = g.tree(28, b, 2, 8, pruned=True, seed=1, worker=_kind(g, kind), rt=r)
        assert (total, st.tasks) == oracle.tree(28, _np(b_cpu), 2, 8, pruned=True, seed=1)


def test_bad_args(g, buf):
    import torch
    tot = torch.zeros(32, dtype=torch.int64, device="cuda")
    L = g.gtap.lib()
    assert not L.gtap_table_tree(g.GTAP_WORKER_THREAD, 5, 0, 1, buf.data_ptr(), 3000, 1, 1, tot.data_ptr())
    assert not L.gtap_table_tree(g.GTAP_WORKER_THREAD, 41, 0, 1, buf.data_ptr(), 1024, 1, 1, tot.data_ptr())
    assert not L.gtap_table_tree(g.GTAP_WORKER_BLOCK, 5, 9, 1, buf.data_ptr(), 1024, 1, 1, tot.data_ptr())
    assert not L.gtap_table_tree(g.GTAP_WORKER_BLOCK, 0, 3, 1, buf.data_ptr(), 1024, 1, 1, tot.data_ptr())
    assert not L.gtap_table_tree(7, 5, 0, 1, buf.data_ptr(), 1024, 1, 1, tot.data_ptr())


@pytest.mark.parametrize("steal_max", [4, 32])
def test_block_batch_steal(g, buf, buf_cpu, steal_max):
    """Block-level batch steals with taskwait (joins of stolen children land in other blocks)."""
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148 * 8, block_size=64, max_tasks_per_worker=2048,
                   steal_max=steal_max, watchdog_ns=WD) as r:
        total, st = g.tree(14, buf, 5, 70, worker=g.GTAP_WORKER_BLOCK, rt=r)
        assert (total, st.tasks) == oracle.tree(14, _np(buf_cpu), 5, 70)
        total, st = g.tree(16, buf, 5, 70, pruned=True, seed=9, worker=g.GTAP_WORKER_BLOCK, rt=r)
        assert (total, st.tasks) == oracle.tree(16, _np(buf_cpu), 5, 70, pruned=True, seed=9)


@pytest.mark.parametrize("kind", KINDS)
def test_bench_per_node_work(g, kind):
    """The bench's per-node work (mem_ops 64 with compute_iters 256 on the full tree, 32768 on the pruned
    tree: bench.bench_tree) at reduced depth so the oracle finishes in seconds; bench launch configuration."""
    import bench
    b_cpu = synth.tree_buffer(1 << 20)
    b = b_cpu.to("cuda")
    with g.Runtime(_kind(g, kind), 0, watchdog_ns=WD, **bench.TREE_CFG[kind]) as r:
        total, st = g.tree(12, b, 64, 256, worker=_kind(g, kind), rt=r)
        assert (total, st.tasks) == oracle.tree(12, _np(b_cpu), 64, 256)
        total, st = g.tree(9, b, 64, 32768, pruned=True, seed=1, worker=_kind(g, kind), rt=r)
        assert (total, st.tasks) == oracle.tree(9, _np(b_cpu), 64, 32768, pruned=True, seed=1)
