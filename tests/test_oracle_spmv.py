"""Pins for the SpMV oracle (standard CSR product; PAPER.md P:42 names SpMV).

Pinned against a dense fp64 matrix-vector product (numpy) on tiny matrices
with random sparsity, empty rows and duplicate column indices, and against
special cases with known results (identity, a row of ones).
"""
import numpy as np
import pytest

import oracle
import synth


def random_csr(rng, nrows, ncols, density):
    rows, cols, vals = [], [], []
    rp = [0]
    for i in range(nrows):
        k = rng.binomial(ncols, density)
        if rng.random() < 0.15:
            k = 0  # empty rows
        c = rng.integers(0, ncols, k)
        if k >= 2 and rng.random() < 0.3:
            c[-1] = c[0]  # duplicate column index
        cols.extend(c.tolist())
        vals.extend((0.5 + rng.random(k)).astype(np.float32).tolist())
        rp.append(len(cols))
    return (np.array(rp, np.int32), np.array(cols, np.int32), np.array(vals, np.float32))


@pytest.mark.parametrize("seed", range(20))
def test_dense_brute_force(seed):
    rng = np.random.default_rng(seed)
    nrows, ncols = rng.integers(1, 65, 2)
    rp, col, val = random_csr(rng, nrows, ncols, rng.random() * 0.5)
    x = (0.5 + rng.random(ncols)).astype(np.float32)
    dense = np.zeros((nrows, ncols), np.float64)
    for i in range(nrows):
        for j in range(rp[i], rp[i + 1]):
            dense[i, col[j]] += float(val[j])  # duplicates are summed
    ref = dense @ x.astype(np.float64)
    y64, y32 = oracle.spmv(rp, col, val, x)
    np.testing.assert_allclose(y64, ref, rtol=1e-13, atol=0)
    assert np.all(np.abs(y32.astype(np.float64) - ref) <= np.spacing(np.abs(ref).astype(np.float32)))
    empty = rp[1:] == rp[:-1]
    assert np.all(y32[empty] == 0)


def test_identity():
    n = 1000
    x = synth.powerlaw_csr(4, n)[3].numpy()
    rp = np.arange(n + 1, dtype=np.int32)
    col = np.arange(n, dtype=np.int32)
    val = np.ones(n, np.float32)
    _, y32 = oracle.spmv(rp, col, val, x)
    assert np.array_equal(y32, x)


def test_row_of_ones():
    n = 4096
    x = synth.powerlaw_csr(4, n)[3].numpy()
    rp = np.array([0, n], np.int32)
    col = np.arange(n, dtype=np.int32)
    val = np.ones(n, np.float32)
    y64, _ = oracle.spmv(rp, col, val, x)
    assert y64[0] == pytest.approx(float(np.sum(x.astype(np.float64))), rel=1e-15)


def test_powerlaw_generator_shape():
    rp, col, val, x = synth.powerlaw_csr(1 << 14)
    deg = (rp[1:] - rp[:-1]).numpy()
    assert deg.min() >= 16 and deg.max() <= 1 << 16
    assert 25 < deg.mean() < 40  # Pareto(2, 16): mean 32 before the floor / cap
    y64, y32 = oracle.spmv(rp, col, val, x)
    assert np.all(y64 > 0)
