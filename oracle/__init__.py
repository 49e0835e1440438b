"""CPU oracle for the GTaP hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The
product path (``paper_2604_05982_b200``) never imports it; it shares no code
with the CUDA side. The arithmetic lives in ``oracle.c`` (plain sequential C,
each function citing the PAPER.md passage it restates); this module is the
ctypes marshalling around it plus a build step (gcc, no CUDA).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc -O3, single thread)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O3", "-std=gnu11", "-ffp-contract=off", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i64p = ctypes.POINTER(ctypes.c_int64)
        vp = ctypes.c_void_p
        L.oracle_fib.argtypes = [ctypes.c_int32, i64p, i64p, i64p]
        L.oracle_fib_cutoff.argtypes = [ctypes.c_int32, ctypes.c_int32, i64p, i64p, i64p, i64p]
        L.oracle_fib_cutoff.restype = ctypes.c_int
        L.oracle_tree.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, vp,
                                  ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                  ctypes.POINTER(ctypes.c_uint64), i64p]
        L.oracle_tree.restype = ctypes.c_int
        L.oracle_nqueens.argtypes = [ctypes.c_int32, ctypes.c_int32, i64p, i64p]
        L.oracle_nqueens.restype = ctypes.c_int
        L.oracle_mergesort.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int64, i64p, i64p]
        L.oracle_cilksort.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, i64p, i64p]
        L.oracle_cilksort.restype = ctypes.c_int
        L.oracle_spmv.argtypes = [vp, vp, vp, vp, ctypes.c_int64, vp, vp]
        L.oracle_bfs.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_int32, vp]
        for f in (L.oracle_fib, L.oracle_mergesort, L.oracle_spmv, L.oracle_bfs):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


def _np(a, dtype):
    """Contiguous numpy view/copy of a numpy array or CPU torch tensor."""
    if hasattr(a, "detach"):
        a = a.detach().to("cpu").numpy()
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def fib(n: int):
    """(value, tasks, invocations) of fib(n) as the paper's task program."""
    v, c, i = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    rc = lib().oracle_fib(n, ctypes.byref(v), ctypes.byref(c), ctypes.byref(i))
    if rc != 0:
        raise ValueError(f"fib: n={n} out of range")
    return v.value, c.value, i.value


def fib_cutoff(n: int, cutoff: int):
    """(value, tasks, invocations, serial_calls) of fib with a cutoff."""
    v, t, i, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    rc = lib().oracle_fib_cutoff(n, cutoff, ctypes.byref(v), ctypes.byref(t), ctypes.byref(i), ctypes.byref(c))
    if rc != 0:
        raise ValueError(f"fib_cutoff: bad arguments n={n} cutoff={cutoff}")
    return v.value, t.value, i.value, c.value


def tree(D: int, buf, mem_ops: int, compute_iters: int, pruned: bool = False, B: int = 3, seed: int = 1):
    """(sum of do_memory_and_compute over all nodes mod 2^64, tasks) of the synthetic tree."""
    b = _np(buf, np.uint64)
    tot, t = ctypes.c_uint64(), ctypes.c_int64()
    rc = lib().oracle_tree(D, B, 1 if pruned else 0, seed, _ptr(b), b.size, mem_ops, compute_iters,
                           ctypes.byref(tot), ctypes.byref(t))
    if rc != 0:
        raise ValueError("tree: bad arguments")
    return tot.value, t.value


def nqueens(n: int, cutoff: int = 7):
    """(solutions, tasks) of the bitmask N-Queens task program with a cutoff depth."""
    v, t = ctypes.c_int64(), ctypes.c_int64()
    if lib().oracle_nqueens(n, cutoff, ctypes.byref(v), ctypes.byref(t)) != 0:
        raise ValueError("nqueens: bad arguments")
    return v.value, t.value


def mergesort(keys, cutoff: int = 128):
    """(sorted copy, tasks, invocations) of the cutoff mergesort."""
    a = _np(keys, np.int32).copy()
    tmp = np.empty_like(a)
    t, i = ctypes.c_int64(), ctypes.c_int64()
    rc = lib().oracle_mergesort(_ptr(a), _ptr(tmp), a.size, cutoff, ctypes.byref(t), ctypes.byref(i))
    if rc != 0:
        raise ValueError("mergesort: bad arguments")
    return a, t.value, i.value


def cilksort(keys, cut_sort: int = 64, cut_merge: int = 256):
    """(sorted copy, tasks, invocations) of Cilksort (parallel merge)."""
    a = _np(keys, np.int32).copy()
    tmp = np.empty_like(a)
    t, i = ctypes.c_int64(), ctypes.c_int64()
    rc = lib().oracle_cilksort(_ptr(a), _ptr(tmp), a.size, cut_sort, cut_merge, ctypes.byref(t), ctypes.byref(i))
    if rc != 0:
        raise ValueError("cilksort: bad arguments")
    return a, t.value, i.value


def spmv(row_ptr, col, val, x):
    """(y fp64, y rounded to fp32) of the CSR product, fp64 accumulation."""
    rp = _np(row_ptr, np.int32)
    c = _np(col, np.int32)
    v = _np(val, np.float32)
    xx = _np(x, np.float32)
    n = rp.size - 1
    y64 = np.empty(n, np.float64)
    y32 = np.empty(n, np.float32)
    lib().oracle_spmv(_ptr(rp), _ptr(c), _ptr(v), _ptr(xx), n, _ptr(y64), _ptr(y32))
    return y64, y32


def bfs(row_ptr, col, src: int):
    """BFS levels from src (INT32_MAX = unreached), FIFO order."""
    rp = _np(row_ptr, np.int32)
    c = _np(col, np.int32)
    nv = rp.size - 1
    depth = np.empty(nv, np.int32)
    rc = lib().oracle_bfs(_ptr(rp), _ptr(c), nv, src, _ptr(depth))
    if rc != 0:
        raise ValueError("bfs: bad source")
    return depth


INT32_MAX = 2**31 - 1
