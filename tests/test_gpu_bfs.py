"""GPU parity: BFS task table vs FIFO BFS (bit-exact levels).

PAPER.md P:1053-1068. Small special graphs, random small graphs, RMAT graphs
from several sources, and BASELINE configs[4] (RMAT scale 22, edge factor 16)
at the bench's launch configuration. The task count is nondeterministic
(reading in DESIGN.md: parity unpinned), so only its lower bound is checked.
"""
import itertools

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
WD = 30_000_000_000


@pytest.fixture(scope="module")
def g(cuda_device):
    import paper_2604_05982_b200 as g
    return g


@pytest.fixture(scope="module")
def rt(g):
    r = g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148 * 2, block_size=128, max_tasks_per_worker=4096,
                  watchdog_ns=WD)
    yield r
    r.close()


def csr_from_edges(nv, edges):
    adj = [[] for _ in range(nv)]
    for u, v in edges:
        adj[u].append(v)
        adj[v].append(u)
    rp = [0]
    col = []
    for a in adj:
        col += sorted(a)
        rp.append(len(col))
    return torch.tensor(rp, dtype=torch.int32), torch.tensor(col if col else [0], dtype=torch.int32)


def check(g, rt, rp, col, src, order=0, edge_split=0):
    depth, st = g.bfs(rp.cuda(), col.cuda(), src, rt=rt, order=order, edge_split=edge_split)
    ref = oracle.bfs(rp, col[: int(rp[-1])] if int(rp[-1]) else col, src)
    assert np.array_equal(depth.cpu().numpy(), ref)
    reached = int((ref != oracle.INT32_MAX).sum())
    assert st.tasks >= reached  # every reached vertex was expanded at least once
    return st


def test_special_graphs(g, rt):
    n = 300
    check(g, rt, *csr_from_edges(n, [(i, i + 1) for i in range(n - 1)]), 0)        # path
    check(g, rt, *csr_from_edges(n, [(0, i) for i in range(1, n)]), 5)            # star from a leaf
    check(g, rt, *csr_from_edges(60, list(itertools.combinations(range(60), 2))), 7)  # complete
    check(g, rt, *csr_from_edges(50, [(1, 2), (3, 4)]), 0)                         # isolated source


@pytest.mark.parametrize("seed", range(10))
def test_random_small(g, rt, seed):
    rng = np.random.default_rng(seed)
    nv = int(rng.integers(2, 200))
    m = int(rng.integers(0, 4 * nv))
    edges = [tuple(rng.integers(0, nv, 2).tolist()) for _ in range(m)]
    rp, col = csr_from_edges(nv, edges)
    check(g, rt, rp, col, int(rng.integers(0, nv)))


@pytest.mark.parametrize("scale", [10, 14, 16])
def test_rmat(g, rt, scale):
    rp, col = synth.rmat_csr(scale, 16, seed=scale)
    for s in synth.bfs_sources(rp, 3, seed=scale):
        check(g, rt, rp, col, s)


def test_hub_overflows_staging(g):
    # one vertex adjacent to 20k others: spawns exceed the shared-memory staging and are flushed mid-task
    n = 20001
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148, block_size=256, max_tasks_per_worker=1 << 15,
                   watchdog_ns=WD) as r:
        check(g, r, *csr_from_edges(n, [(0, i) for i in range(1, n)]), 0)


def test_hub_capacity_error(g):
    # the same hub with a 4096-slot deque must fail loudly (fixed capacity), not hang
    n = 20001
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=16, block_size=256, max_tasks_per_worker=4096,
                   watchdog_ns=WD) as r:
        with pytest.raises(g.GtapError) as e:
            check(g, r, *csr_from_edges(n, [(0, i) for i in range(1, n)]), 0)
        assert e.value.code in (5, 6)


@pytest.mark.parametrize("order", [0, 1])
def test_full_size_config4(g, order):
    import bench
    rp, col = synth.rmat_csr(22, 16, seed=3, device="cuda")
    src = synth.bfs_sources(rp, 1, seed=5)[0]
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, watchdog_ns=60_000_000_000, **bench.BFS_CFG) as r:
        depth, st = g.bfs(rp, col, src, rt=r, order=order)
    ref = oracle.bfs(rp.cpu(), col.cpu(), src)
    assert np.array_equal(depth.cpu().numpy(), ref)


@pytest.mark.parametrize("steal_max", [2, 7, 32])
def test_batch_steal(g, steal_max):
    """Block-level batch steals (steal_max > 1: run one, keep the rest): levels stay exact."""
    rp, col = synth.rmat_csr(14, 16, seed=21)
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148 * 4, block_size=64, max_tasks_per_worker=1 << 15,
                   steal_max=steal_max, watchdog_ns=WD) as r:
        for s in synth.bfs_sources(rp, 3, seed=steal_max):
            check(g, r, rp, col, s)


@pytest.mark.parametrize("scale", [10, 14, 16])
def test_rmat_fifo_order(g, scale):
    """gtap_table_bfs_ex order 1 (oldest-first pops, every child pushed): same levels; deques sized for a
    local frontier."""
    rp, col = synth.rmat_csr(scale, 16, seed=scale)
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148 * 2, block_size=128, max_tasks_per_worker=1 << 16,
                   watchdog_ns=WD) as r:
        for s in synth.bfs_sources(rp, 3, seed=scale):
            check(g, r, rp, col, s, order=1)
        check(g, r, *csr_from_edges(300, [(i, i + 1) for i in range(299)]), 0, order=1)   # path
        check(g, r, *csr_from_edges(50, [(1, 2), (3, 4)]), 0, order=1)                    # isolated source


def test_fifo_order_overflow_fails_loudly(g):
    """order 1 holds frontiers in the deques: an undersized ring must fail with an error, not hang."""
    rp, col = synth.rmat_csr(16, 16, seed=16)
    src = synth.bfs_sources(rp, 1, seed=16)[0]
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=2, block_size=64, max_tasks_per_worker=64,
                   watchdog_ns=WD) as r:
        with pytest.raises(g.GtapError) as e:
            check(g, r, rp, col, src, order=1)
        assert e.value.code in (5, 6)


def test_die_aware_victims_block_level(g):
    """victim_policy 1 on block-level workers (BFS): same levels."""
    rp, col = synth.rmat_csr(14, 16, seed=14)
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148 * 4, block_size=64, max_tasks_per_worker=1 << 15,
                   steal_max=32, victim_policy=1, watchdog_ns=WD) as r:
        for s in synth.bfs_sources(rp, 2, seed=14):
            check(g, r, rp, col, s)
            check(g, r, rp, col, s, order=1)


@pytest.mark.parametrize("block", [32, 64])
@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("edge_split", [1, 7, 64, 1000])
def test_hub_split(g, order, edge_split, block):
    """gtap_table_bfs_split: vertices above edge_split edges hand pieces of their edge list to bfs_edges
    tasks (fn 1); the levels stay exact (stars, complete graph, RMAT hubs, one-edge pieces, ragged last piece).
    Block 32 runs the one-warp kernel with multi-task cycles (lane groups), block 64 one task per cycle."""
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148 * 2, block_size=block, max_tasks_per_worker=1 << 16,
                   steal_max=32, watchdog_ns=WD) as r:
        check(g, r, *csr_from_edges(5001, [(0, i) for i in range(1, 5001)]), 0, order, edge_split)   # hub source
        check(g, r, *csr_from_edges(5001, [(0, i) for i in range(1, 5001)]), 9, order, edge_split)   # via the hub
        check(g, r, *csr_from_edges(60, list(itertools.combinations(range(60), 2))), 7, order, edge_split)
        check(g, r, *csr_from_edges(50, [(1, 2), (3, 4)]), 0, order, edge_split)                    # isolated
        rp, col = synth.rmat_csr(14, 16, seed=edge_split)
        for s in synth.bfs_sources(rp, 2, seed=edge_split):
            check(g, r, rp, col, s, order, edge_split)


def test_hub_split_full_size(g):
    """the bench's split + geometry at RMAT-22 (configs[4]), bit-exact levels"""
    import bench
    rp, col = synth.rmat_csr(22, 16, seed=3, device="cuda")
    src = synth.bfs_sources(rp, 2, seed=5)[1]
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, watchdog_ns=60_000_000_000, **bench.BFS_CFG) as r:
        depth, st = g.bfs(rp, col, src, rt=r, order=bench.BFS_ORDER, edge_split=bench.BFS_SPLIT or 2048)
    assert np.array_equal(depth.cpu().numpy(), oracle.bfs(rp.cpu(), col.cpu(), src))


@pytest.mark.parametrize("order", [0, 1])
def test_one_warp_blocks(g, order):
    """one-warp blocks (multi-task cycles) without hub splitting: special graphs, random graphs, RMAT"""
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148 * 4, block_size=32, max_tasks_per_worker=1 << 15,
                   steal_max=32, watchdog_ns=WD) as r:
        n = 300
        check(g, r, *csr_from_edges(n, [(i, i + 1) for i in range(n - 1)]), 0, order)
        check(g, r, *csr_from_edges(n, [(0, i) for i in range(1, n)]), 5, order)
        check(g, r, *csr_from_edges(60, list(itertools.combinations(range(60), 2))), 7, order)
        for seed in range(4):
            rng = np.random.default_rng(100 + seed)
            nv = int(rng.integers(2, 400))
            edges = [tuple(rng.integers(0, nv, 2).tolist()) for _ in range(int(rng.integers(0, 6 * nv)))]
            check(g, r, *csr_from_edges(nv, edges), int(rng.integers(0, nv)), order)
        rp, col = synth.rmat_csr(16, 16, seed=31)
        for s in synth.bfs_sources(rp, 2, seed=31):
            check(g, r, rp, col, s, order)
