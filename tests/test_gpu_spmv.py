"""GPU parity: SpMV task table vs the fp64 oracle, |y - y_ref| <= 1e-5 |y_ref| per row.

The tolerance is BASELINE.json north_star's. Empty rows must be exactly 0.
Cases: tiny matrices with empty rows / duplicates, a single 65,536-nnz row
(block-cooperative heavy path), ragged row counts, both leaf and split paths,
and BASELINE configs[3] (2^22 rows, power-law, ~32 nnz/row) at the bench's
launch configuration (every row checked).
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
WD = 30_000_000_000
RTOL = 1e-5


@pytest.fixture(scope="module")
def g(cuda_device):
    import paper_2604_05982_b200 as g
    return g


@pytest.fixture(scope="module")
def rt(g):
    r = g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148 * 2, block_size=256, max_tasks_per_worker=1024,
                  watchdog_ns=WD)
    yield r
    r.close()


def check(g, rt, rp, col, val, x, **kw):
    dev = [t.cuda() for t in (rp, col, val, x)]
    y, st = g.spmv(*dev, rt=rt, **kw)
    y64, _ = oracle.spmv(rp, col, val, x)
    y = y.cpu().numpy().astype(np.float64)
    empty = (rp[1:] == rp[:-1]).numpy()
    assert np.all(y[empty] == 0.0)
    ne = ~empty
    rel = np.abs(y[ne] - y64[ne]) / np.abs(y64[ne])
    assert rel.max(initial=0.0) <= RTOL, rel.max()
    return st


def csr(rows):
    rp = [0]
    cols, vals = [], []
    for r in rows:
        cols += [c for c, _ in r]
        vals += [v for _, v in r]
        rp.append(len(cols))
    return (torch.tensor(rp, dtype=torch.int32), torch.tensor(cols, dtype=torch.int32),
            torch.tensor(vals, dtype=torch.float32))


@pytest.mark.parametrize("nrows", [1, 7, 33, 1000, 4099])
@pytest.mark.parametrize("nnz_cut", [64, 8192])
def test_powerlaw_small(g, rt, nrows, nnz_cut):
    rp, col, val, x = synth.powerlaw_csr(nrows, seed=nrows)
    check(g, rt, rp, col, val, x, nnz_cut=nnz_cut)


def test_empty_rows_and_duplicates(g, rt):
    rng = np.random.default_rng(0)
    rows = []
    for i in range(3000):
        k = 0 if i % 5 == 0 else int(rng.integers(1, 40))
        c = rng.integers(0, 500, k)
        if k > 2:
            c[1] = c[0]
        rows.append(list(zip(c.tolist(), (0.5 + rng.random(k)).tolist())))
    rp, col, val = csr(rows)
    x = (0.5 + torch.rand(500, generator=torch.Generator().manual_seed(0))).float()
    check(g, rt, rp, col, val, x, nnz_cut=256, fanout=3)


def test_heavy_row(g, rt):
    n = 1 << 16
    rows = [[(j, 0.5 + (j % 7) / 7) for j in range(n)], [(1, 1.0)], [], [(j, 1.0) for j in range(300)]]
    rp, col, val = csr(rows)
    x = synth.powerlaw_csr(4, n)[3]
    check(g, rt, rp, col, val, x, nnz_cut=1 << 20)


def test_identity(g, rt):
    n = 10000
    rp = torch.arange(n + 1, dtype=torch.int32)
    col = torch.arange(n, dtype=torch.int32)
    val = torch.ones(n, dtype=torch.float32)
    x = synth.powerlaw_csr(4, n)[3]
    y, _ = g.spmv(rp.cuda(), col.cuda(), val.cuda(), x.cuda(), rt=rt, nnz_cut=512)
    assert torch.equal(y.cpu(), x)


def test_full_size_config3(g):
    import bench
    rp, col, val, x = synth.powerlaw_csr(1 << 22, seed=7, device="cuda")
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, watchdog_ns=60_000_000_000, **bench.SPMV_CFG) as r:
        y, st = g.spmv(rp, col, val, x, rt=r, nnz_cut=bench.SPMV_NNZ_CUT, fanout=bench.SPMV_FANOUT,
                       parts=bench.SPMV_PARTS)
    y64, _ = oracle.spmv(rp.cpu(), col.cpu(), val.cpu(), x.cpu())
    rel = np.abs(y.cpu().numpy().astype(np.float64) - y64) / np.abs(y64)
    assert rel.max() <= RTOL, rel.max()


@pytest.mark.parametrize("parts", [1, 2, 7, 148, 1184, 5000])
@pytest.mark.parametrize("nnz_cut", [128, 1 << 20])
def test_forest_parts(g, parts, nnz_cut):
    """Forest of part(k, R) roots (nnz-balanced ranges found in the kernel): every row exactly once,
    including R larger than the number of rows (empty parts) and heavy rows at range borders."""
    rp, col, val, x = synth.powerlaw_csr(4099, seed=11)
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148, block_size=128, max_tasks_per_worker=4096,
                   max_roots=parts, watchdog_ns=WD) as r:
        st = check(g, r, rp, col, val, x, nnz_cut=nnz_cut, parts=parts)
    assert st.tasks >= parts


def test_forest_subrange(g):
    """parts over a row sub-range [lo, hi): rows outside keep their previous values."""
    rp, col, val, x = synth.powerlaw_csr(5000, seed=12)
    y64, _ = oracle.spmv(rp, col, val, x)
    lo, hi = 1234, 4321
    dev = [t.cuda() for t in (rp, col, val, x)]
    y = torch.full((5000,), -7.0, dtype=torch.float32, device="cuda")
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=64, block_size=128, max_tasks_per_worker=4096, max_roots=37,
                   watchdog_ns=WD) as r:
        y, _ = g.spmv(*dev, y, nnz_cut=256, rows=(lo, hi), parts=37, rt=r)
    y = y.cpu().numpy().astype(np.float64)
    assert np.all(y[:lo] == -7.0) and np.all(y[hi:] == -7.0)
    ne = rp[lo + 1:hi + 1].numpy() != rp[lo:hi].numpy()
    rel = np.abs(y[lo:hi][ne] - y64[lo:hi][ne]) / np.abs(y64[lo:hi][ne])
    assert rel.max() <= RTOL
    assert np.all(y[lo:hi][~ne] == 0.0)


@pytest.mark.parametrize("steal_max", [3, 32])
def test_batch_steal(g, steal_max):
    rp, col, val, x = synth.powerlaw_csr(20011, seed=13)
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148 * 2, block_size=128, max_tasks_per_worker=4096,
                   steal_max=steal_max, watchdog_ns=WD) as r:
        check(g, r, rp, col, val, x, nnz_cut=256, fanout=8)
