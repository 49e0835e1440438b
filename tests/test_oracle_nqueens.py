"""Pins for the N-Queens oracle.

Solution counts pinned to OEIS A000170 (tests/golden/nqueens.txt) and to a brute-force
permutation check for n <= 8; the task count (one task per partial placement of fewer
than `cutoff` rows, plus the root) pinned to an explicit enumeration of partial placements.
"""
import itertools
import os

import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "nqueens.txt")


def golden():
    out = []
    for line in open(GOLDEN):
        if line.strip() and not line.startswith("#"):
            a, b = line.split()[:2]
            out.append((int(a), int(b)))
    return out


def brute(n):
    return sum(1 for p in itertools.permutations(range(n))
               if len({p[i] + i for i in range(n)}) == n and len({p[i] - i for i in range(n)}) == n)


def partial_placements(n, rows):
    """number of non-attacking placements of queens on the first `rows` rows (explicit search)."""
    cnt = 0
    def ok(prefix, c):
        r = len(prefix)
        return all(c != pc and abs(c - pc) != r - pr for pr, pc in enumerate(prefix))
    frontier = [()]
    for r in range(rows):
        frontier = [p + (c,) for p in frontier for c in range(n) if ok(p, c)]
    return len(frontier)


@pytest.mark.parametrize("n,sol", [g for g in golden() if g[0] <= 14])
def test_golden_counts(n, sol):
    for cutoff in (0, 3, 7):
        assert oracle.nqueens(n, cutoff)[0] == sol


@pytest.mark.slow
def test_golden_16():
    assert oracle.nqueens(16, 7)[0] == 14772512


@pytest.mark.parametrize("n", range(1, 9))
def test_brute_force(n):
    assert oracle.nqueens(n, 7)[0] == brute(n)


@pytest.mark.parametrize("n,cutoff", [(6, 2), (8, 3), (8, 7), (10, 4), (11, 7)])
def test_task_count(n, cutoff):
    # tasks = sum over r <= min(cutoff, n) of partial placements of r rows (the root is r = 0)
    expect = sum(partial_placements(n, r) for r in range(0, min(cutoff, n) + 1))
    assert oracle.nqueens(n, cutoff)[1] == expect
