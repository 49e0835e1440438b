"""Pins for the BFS oracle.

Why FIFO BFS is the right oracle for the paper's asynchronous label-correcting
traversal (bfs(v): dv = depth[v]; for each neighbour u: old =
atomicMin(&depth[u], dv + 1); if old > dv + 1 spawn bfs(u)), from depth[src]=0:
  1. depth only decreases, and every value written is dv + 1 for a value dv
     that depth[v] held, so depth[u] >= dist(u) at all times (induction).
  2. When depth[v] drops to its final value d, the task that lowered it
     spawned bfs(v); that task runs later, reads d (no later decrease), and
     relaxes every neighbour to <= d + 1.
  3. At quiescence every edge (v, u) has depth[u] <= depth[v] + 1, which with
     (1) gives depth = dist on the source's component; others stay INT32_MAX.
So the unique fixed point equals textbook BFS levels; the oracle is pinned to
all-pairs shortest paths (scipy) on every 5-vertex graph and to Graph500-style
validation on RMAT graphs.
"""
import itertools

import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import connected_components, shortest_path

import oracle
import synth

IMAX = oracle.INT32_MAX


def csr_from_edges(nv, edges):
    adj = [[] for _ in range(nv)]
    for u, v in edges:
        adj[u].append(v)
        adj[v].append(u)
    rp = np.zeros(nv + 1, np.int32)
    col = []
    for i in range(nv):
        col.extend(sorted(adj[i]))
        rp[i + 1] = len(col)
    return rp, np.array(col, np.int32)


def scipy_levels(rp, col, src):
    nv = rp.size - 1
    m = csr_matrix((np.ones(col.size), col, rp), shape=(nv, nv))
    d = shortest_path(m, unweighted=True, indices=src, directed=True)
    return np.where(np.isinf(d), IMAX, d).astype(np.int64)


def test_all_5_vertex_graphs():
    pairs = list(itertools.combinations(range(5), 2))
    for mask in range(1 << len(pairs)):
        edges = [p for k, p in enumerate(pairs) if mask >> k & 1]
        rp, col = csr_from_edges(5, edges)
        for s in range(5):
            assert np.array_equal(oracle.bfs(rp, col, s), scipy_levels(rp, col, s)), (edges, s)


def test_special_graphs():
    n = 50
    rp, col = csr_from_edges(n, [(i, i + 1) for i in range(n - 1)])
    assert oracle.bfs(rp, col, 0).tolist() == list(range(n))
    rp, col = csr_from_edges(n, [(0, i) for i in range(1, n)])
    assert oracle.bfs(rp, col, 0).tolist() == [0] + [1] * (n - 1)
    assert oracle.bfs(rp, col, 3).tolist() == [1, 2, 2, 0] + [2] * (n - 4)
    rp, col = csr_from_edges(n, list(itertools.combinations(range(n), 2)))
    assert oracle.bfs(rp, col, 7).tolist() == [1] * 7 + [0] + [1] * (n - 8)
    rp, col = csr_from_edges(n, [(1, 2)])
    d = oracle.bfs(rp, col, 0)
    assert d[0] == 0 and np.all(d[1:] == IMAX)


def graph500_validate(rp, col, src, level):
    nv = rp.size - 1
    assert level[src] == 0
    deg = rp[1:] - rp[:-1]
    srcs = np.repeat(np.arange(nv), deg)
    lu, lv = level[srcs].astype(np.int64), level[col].astype(np.int64)
    reach_u, reach_v = lu != IMAX, lv != IMAX
    assert np.all(reach_u == reach_v)  # an edge never crosses the component boundary
    both = reach_u & reach_v
    assert np.all(np.abs(lu[both] - lv[both]) <= 1)
    # every reached v != src has a neighbour one level up
    has_parent = np.zeros(nv, bool)
    ok = both & (lv == lu - 1)
    has_parent[srcs[ok]] = True
    reached = level != IMAX
    reached[src] = False
    assert np.all(has_parent[reached])
    m = csr_matrix((np.ones(col.size), col, rp), shape=(nv, nv))
    _, lab = connected_components(m, directed=False)
    assert np.array_equal(level != IMAX, lab == lab[src])


@pytest.mark.parametrize("scale", [8, 11, 13])
def test_rmat_graph500_validity(scale):
    rp, col = synth.rmat_csr(scale, 16, seed=scale)
    rp, col = rp.numpy(), col.numpy()
    for s in synth.bfs_sources(torch_tensor(rp), 3, seed=scale):
        level = oracle.bfs(rp, col, s)
        graph500_validate(rp, col, s, level)
        assert np.array_equal(level, scipy_levels(rp, col, s))


def torch_tensor(a):
    import torch
    return torch.from_numpy(a)


def test_rmat_shape():
    rp, col = synth.rmat_csr(12, 16, seed=1)
    assert int(rp[-1]) == 2 * 16 * (1 << 12)
    deg = (rp[1:] - rp[:-1]).numpy()
    assert (deg == 0).mean() > 0.1  # RMAT leaves many isolated vertices
    assert deg.max() > 20 * deg.mean()  # skewed hubs
