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


# ---- exact task / invocation counts on inputs whose splits do not depend on the key values ----
#
# Reading R26: merge(A, B) with |A| + |B| > CUTOFF_MERGE splits the longer run at its middle
# (floor), lower_bound of that key in B when A is the longer run, upper_bound in A when B is. When every
# key of A is <= every key of B (sorted or all-equal input: each sort task's left half holds the smaller
# keys) both searches land at the start of B / the end of A; when every key of A is > every key of B
# (reverse input) they land at the end of B / the start of A. The split sizes then depend on (|A|, |B|)
# only, and the counts follow from this recurrence -- written here from the rule, never calling oracle.c.
from functools import lru_cache


def _counts(n, cut_sort, cut_merge, a_le_b):
    @lru_cache(maxsize=None)
    def merge(na, nb):
        if na + nb <= cut_merge:
            return 1, 1                                    # leaf merge: one invocation
        if na >= nb:
            h = na // 2
            left, right = ((h, 0), (na - h, nb)) if a_le_b else ((h, nb), (na - h, 0))
        else:
            h = nb // 2
            left, right = ((na, h), (0, nb - h)) if a_le_b else ((0, h), (na, nb - h))
        t0, i0 = merge(*left)
        t1, i1 = merge(*right)
        return 1 + t0 + t1, 2 + i0 + i1                    # spawn + resume after the join

    @lru_cache(maxsize=None)
    def sort(m):
        if m <= cut_sort:
            return 1, 1
        h = m // 2                                         # mid = l + (r - l) / 2
        t0, i0 = sort(h)
        t1, i1 = sort(m - h)
        tm, im = merge(h, m - h)
        return 1 + t0 + t1 + tm, 3 + i0 + i1 + im           # spawn sorts, spawn merge, finish

    return sort(n)


@pytest.mark.parametrize("kind", ["sorted", "equal", "reverse"])
@pytest.mark.parametrize("n", [0, 1, 64, 65, 255, 256, 257, 1000, 4099, 1 << 12, (1 << 14) + 5, 1 << 16])
@pytest.mark.parametrize("cuts", [(64, 256), (1, 2), (4, 8), (16, 300), (256, 2048)])
def test_exact_counts_value_independent_splits(kind, n, cuts):
    if cuts[1] <= 8 and n > 5000:
        pytest.skip("tiny merge cutoffs: the oracle's per-key tasks make this slow; smaller n covers them")
    a = {"sorted": np.arange(n), "equal": np.full(n, 7), "reverse": np.arange(n, 0, -1)}[kind].astype(np.int32)
    out, tasks, inv = oracle.cilksort(a, *cuts)
    assert np.array_equal(out, np.sort(a))
    assert (tasks, inv) == _counts(n, *cuts, a_le_b=(kind != "reverse"))


def test_recurrence_closed_forms():
    """Sanity of the recurrence itself: with CUTOFF_MERGE >= n no merge splits, so the counts are
    mergesort's 2n/C - 1 sort tasks plus one merge leaf per internal sort (n = 2^k)."""
    for k in range(6, 14):
        n = 1 << k
        internal = n // 64 - 1
        assert _counts(n, 64, 1 << 30, True) == (2 * (n // 64) - 1 + internal, n // 64 + 3 * internal + internal)
