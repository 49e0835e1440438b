"""Pins for the mergesort oracle.

Sorting integer keys has a unique result, so the oracle output is pinned to a
library sort (numpy), to exhaustive enumeration of all permutations of small
inputs (cutoffs small enough that merges run), and to adversarial inputs.
The task count is pinned to the closed form 2n/C - 1 (n = 2^k >= C): a full
binary split down to leaves of exactly C keys.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth


@pytest.mark.parametrize("n,cutoff", [(0, 128), (1, 128), (127, 128), (128, 128), (129, 128),
                                      (1000, 128), (4097, 64), (100000, 128), (65536, 1)])
def test_random_vs_numpy(n, cutoff):
    keys = synth.keys_int32(n, seed=n + cutoff).numpy()
    out, tasks, inv = oracle.mergesort(keys, cutoff)
    assert np.array_equal(out, np.sort(keys, kind="stable"))
    if n <= cutoff:
        assert (tasks, inv) == (1, 1)


@pytest.mark.parametrize("cutoff", [1, 2, 4])
@pytest.mark.parametrize("n", range(0, 8))
def test_exhaustive_permutations(n, cutoff):
    base = list(range(n))
    for perm in itertools.permutations(base):
        out, _, _ = oracle.mergesort(np.array(perm, np.int32), cutoff)
        assert out.tolist() == base


def test_exhaustive_with_duplicates():
    for vals in itertools.product([0, 1, 2], repeat=7):
        out, _, _ = oracle.mergesort(np.array(vals, np.int32), 2)
        assert out.tolist() == sorted(vals)


@pytest.mark.parametrize("kind", ["sorted", "reverse", "equal", "two", "extremes"])
def test_adversarial(kind):
    n = 5000
    rng = np.random.default_rng(1)
    if kind == "sorted":
        a = np.arange(n, dtype=np.int32)
    elif kind == "reverse":
        a = np.arange(n, 0, -1).astype(np.int32)
    elif kind == "equal":
        a = np.full(n, 7, np.int32)
    elif kind == "two":
        a = rng.integers(0, 2, n).astype(np.int32)
    else:
        a = rng.choice(np.array([-2**31, 2**31 - 1, 0, -1], np.int64), n).astype(np.int32)
    out, _, _ = oracle.mergesort(a, 128)
    assert np.array_equal(out, np.sort(a))


@pytest.mark.parametrize("k,cutoff", [(7, 128), (10, 128), (14, 128), (12, 64), (6, 1)])
def test_task_count_closed_form(k, cutoff):
    n = 1 << k
    _, tasks, inv = oracle.mergesort(synth.keys_int32(n, seed=k).numpy(), cutoff)
    leaves = max(n // cutoff, 1)
    assert tasks == 2 * leaves - 1
    assert inv == leaves + 2 * (leaves - 1)


def test_task_count_2_24_value():
    # 2^24 keys, cutoff 128 -> 262,143 tasks, 393,214 invocations
    n, c = 1 << 24, 128
    assert 2 * (n // c) - 1 == 262143
    assert (n // c) + 2 * (n // c - 1) == 393214
