"""Pins for the synthetic-tree oracle.

* full binary tree: tasks = 2^(D+1) - 1 (closed form);
* pruned B-ary tree: p(0) = 1 so the root always has B children; for D = 1 exactly 1 + B tasks;
  the shape is a pure function of (D, B, seed) (counter-based) and thins with depth;
* do_memory_and_compute: one node restated in Python (sum of 64-bit words at mixed indices, FMA
  chains with an exact-rational FMA), via a 1-node tree (D = 0), and summed over small trees.
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
