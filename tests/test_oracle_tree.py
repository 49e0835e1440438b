"""Pins for the synthetic-tree oracle.

* full binary tree: tasks = 2^(D+1) - 1 (closed form);
* pruned B-ary tree: p(0) = 1 so the root always has B children; for D = 1 exactly 1 + B tasks;
  the shape is a pure function of (D, B, seed) (counter-based) and thins with depth;
* do_memory_and_compute, pinned without restating it: the load indices are SplitMix64's published
  test vector (seed 0); a constant buffer gives c * mem_ops * tasks; the FMA chains match the closed
  form of the linear recurrence f <- A f + B (geometric series) within the FMA rounding bound;
* also one node restated in Python (exact-rational FMA), via a 1-node tree (D = 0), and small trees.
"""
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

M64 = (1 << 64) - 1


def mix(z):
    z ^= z >> 30; z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27; z = (z * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def fma(a, b, c):
    """Fused multiply-add: the exact rational a*b + c rounded once (float(Fraction) rounds to nearest-even)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def work_py(node, buf, mem_ops, compute_iters):
    s = 0
    for i in range(mem_ops):
        s += int(buf[mix((node * 0x9E3779B97F4A7C15 + i) & M64) % len(buf)])
    for c in range(min(64, compute_iters)):
        f = 1.0 + ((node + c) & 1023) / 1024.0
        for _ in range(compute_iters // 64 + (1 if c < compute_iters % 64 else 0)):
            f = fma(f, 0.999999, 1e-7)
        s += struct.unpack("<Q", struct.pack("<d", f))[0]
    return s & M64


@pytest.fixture(scope="module")
def buf():
    return synth.tree_buffer(1 << 12).numpy().astype(np.uint64)


@pytest.mark.parametrize("D", [0, 1, 5, 10])
def test_full_tree_count(buf, D):
    assert oracle.tree(D, buf, 3, 40)[1] == 2 ** (D + 1) - 1


@pytest.mark.parametrize("mem,comp", [(0, 0), (5, 0), (0, 70), (17, 33), (0, 130)])
def test_single_node_work(buf, mem, comp):
    total, tasks = oracle.tree(0, buf, mem, comp)   # full tree, D = 0: just the root (id 1)
    assert tasks == 1 and total == work_py(1, buf, mem, comp)


def test_full_tree_sum_small(buf):
    total, tasks = oracle.tree(3, buf, 4, 35)
    assert total == sum(work_py(i, buf, 4, 35) for i in range(1, 16)) & M64


def test_pruned_shape(buf):
    assert oracle.tree(1, buf, 0, 0, pruned=True)[1] == 1 + 3
    t1 = oracle.tree(12, buf, 0, 0, pruned=True, seed=1)[1]
    assert t1 == oracle.tree(12, buf, 0, 0, pruned=True, seed=1)[1]   # deterministic
    assert t1 != oracle.tree(12, buf, 0, 0, pruned=True, seed=2)[1]   # depends on the seed
    assert t1 < (3 ** 13 - 1) // 2                                   # thinner than the full 3-ary tree


@pytest.mark.parametrize("D,seed", [(4, 1), (6, 7), (7, 3)])
def test_pruned_bruteforce(buf, D, seed):
    """Enumerate the pruned 3-ary tree in Python: child k of node i (depth d) is 3i+1+k, kept iff
    its 53-bit draw is below p(d) = 1 - d/D scaled to 2^53 (floor)."""
    nodes, stack = [], [(0, 0)]
    while stack:
        i, d = stack.pop()
        nodes.append(i)
        if d < D:
            for k in range(3):
                c = 3 * i + 1 + k
                if (mix(seed ^ c) >> 11) < ((D - d) << 53) // D:
                    stack.append((c, d + 1))
    total, tasks = oracle.tree(D, buf, 2, 33, pruned=True, seed=seed)
    assert tasks == len(nodes)
    assert total == sum(work_py(i, buf, 2, 33) for i in nodes) & M64


# ---- pins that do not restate do_memory_and_compute (reading R27) ----

# SplitMix64 (Steele, Lea, Flood 2014) seeded with 0: its first outputs are the finaliser applied to
# k * 0x9E3779B97F4A7C15, the published test vector of the generator. R27 draws load i of node id at
# index mix(id * 0x9E3779B97F4A7C15 + i) mod len, so with i = 0 node id's first load index is the id-th
# output of SplitMix64(0).
SPLITMIX64_SEED0 = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_load_index_is_splitmix64_published_vector():
    ident = np.arange(1 << 20, dtype=np.uint64)          # buf[j] = j: the total is the sum of the indices
    total, tasks = oracle.tree(0, ident, 1, 0)          # root only (heap id 1), one load
    assert (total, tasks) == (SPLITMIX64_SEED0[0] % (1 << 20), 1)
    total, tasks = oracle.tree(1, ident, 1, 0)          # heap ids 1, 2, 3
    assert (total, tasks) == (sum(v % (1 << 20) for v in SPLITMIX64_SEED0), 3)


@pytest.mark.parametrize("D,pruned,seed", [(0, False, 1), (6, False, 1), (9, True, 4)])
@pytest.mark.parametrize("mem", [1, 7, 64])
def test_constant_buffer_closed_form(buf, D, pruned, seed, mem):
    """buf = c everywhere and no FMAs: the total is c * mem_ops * tasks mod 2^64, whatever the indices."""
    tasks = oracle.tree(D, buf, 0, 0, pruned=pruned, seed=seed)[1]
    for c in (1, 3, (1 << 63) + 5):
        total, t = oracle.tree(D, np.full(1 << 10, c, np.uint64), mem, 0, pruned=pruned, seed=seed)
        assert t == tasks and total == (c * mem * tasks) & M64


A = Fraction(0.999999)   # the exact doubles R27's chains use: f <- fma(f, A, B)
B = Fraction(1e-7)


def _chains_closed_form(ids, compute_iters):
    """Sum over the nodes and chains of f_k = B/(1-A) + (f_0 - B/(1-A)) A^k (the solution of the linear
    recurrence f <- A f + B in exact arithmetic), f_0 = 1 + ((id + c) & 1023) / 1024 for chain c < 64,
    k = compute_iters // 64 (+1 for c < compute_iters % 64). Returns (sum of (f - 1) * 2^52, chains, steps)."""
    fix = B / (1 - A)
    pw = {}
    s, nch, steps = Fraction(0), 0, 0
    for node in ids:
        for c in range(min(64, compute_iters)):
            k = compute_iters // 64 + (1 if c < compute_iters % 64 else 0)
            if k not in pw:
                pw[k] = A ** k
            f0 = 1 + Fraction((node + c) & 1023, 1024)
            s += (fix + (f0 - fix) * pw[k] - 1) * (1 << 52)
            nch += 1
            steps += k
    return s, nch, steps


@pytest.mark.parametrize("D", [0, 1])
@pytest.mark.parametrize("comp", [1, 5, 64, 100, 6400, 32768])
def test_fma_chains_match_geometric_closed_form(D, comp):
    """With mem_ops = 0 the total is the sum of the chains' final bit patterns. Every f stays in [1, 2)
    (f_0 >= 1 + 1/1024 and at most 512 steps of a 1e-6 contraction), where bits(f) = 0x3FF0000000000000
    + (f - 1) 2^52 exactly; each FMA rounds once (<= 1/2 ulp = 1/2 in these units) and the contraction
    A < 1 never amplifies an earlier error, so the total is within steps / 2 + chains of the closed form.
    One missing or extra FMA in one chain moves it by ~0.9e-6 * 2^52 ~ 4e9 units."""
    ids = [1] if D == 0 else [1, 2, 3]
    total, tasks = oracle.tree(D, np.zeros(16, np.uint64), 0, comp)
    exact, nch, steps = _chains_closed_form(ids, comp)
    base = nch * 0x3FF0000000000000
    assert abs(Fraction(total) - (base + exact) % (1 << 64)) <= Fraction(steps, 2) + nch
