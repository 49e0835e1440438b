"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no scheduling, sorting, SpMV or
BFS logic). It only draws the input data of the paper's workloads from a
counter-based generator, so both sides (``oracle/`` and the CUDA path) read the
very same arrays:

* a SplitMix64 finaliser over ``key + (i + 1) * GAMMA`` gives the i-th 64-bit
  draw of a stream (counter-based: no state, identical on any device);
* everything is written with torch integer ops, which wrap mod 2^64 identically
  on CPU and CUDA, so a tensor generated on ``cuda`` equals the one generated on
  ``cpu`` bit for bit (floats are built from integers by exact scalings).

Workload shapes follow SURVEY.md §8(c)/(d) and DESIGN.md "Input recipe":

* mergesort keys: "random 4-byte integer arrays" (§6.2) —
  uniform over the full signed int32 range;
* SpMV: power-law CSR, 2^22 rows, ~32 nnz/row (BASELINE.json configs[3]) —
  Pareto(alpha=2, x_m=16) row degrees capped at 2^16, uniform columns,
  values and x uniform in [0.5, 1.5);
* BFS: Graph500-style RMAT(a=.57, b=.19, c=.19, d=.05), edge factor 16,
  symmetrised, seeded vertex permutation (BASELINE.json configs[4]).
"""
from __future__ import annotations

import torch

__all__ = [
    "mix64", "counter_u64", "uniform01_f64",
    "keys_int32", "powerlaw_csr", "rmat_csr", "bfs_sources", "stream_key", "tree_buffer",
]

_GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


def _s64(c: int) -> int:
    """Two's-complement view of a 64-bit constant (torch int64 wraps mod 2^64)."""
    c &= (1 << 64) - 1
    return c - (1 << 64) if c >= (1 << 63) else c


def _srl(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of an int64 tensor viewed as uint64."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def mix64(z: torch.Tensor) -> torch.Tensor:
    """SplitMix64 output function (Steele, Lea, Flood 2014), on int64 bit patterns."""
    z = (z ^ _srl(z, 30)) * _s64(_M1)
    z = (z ^ _srl(z, 27)) * _s64(_M2)
    return z ^ _srl(z, 31)


def stream_key(seed: int, stream: int) -> int:
    """A 64-bit key for sub-stream ``stream`` of ``seed`` (plain Python ints)."""
    m = (1 << 64) - 1
    z = (seed * 0x2545F4914F6CDD1D + stream * _GAMMA + 0x632BE59BD9B4E019) & m
    z = ((z ^ (z >> 30)) * _M1) & m
    z = ((z ^ (z >> 27)) * _M2) & m
    return z ^ (z >> 31)


def counter_u64(key: int, idx: torch.Tensor) -> torch.Tensor:
    """i-th draw of the stream ``key``: mix64(key + (i + 1) * GAMMA), int64 bits."""
    z = idx.to(torch.int64) + 1
    z = z * _s64(_GAMMA) + _s64(key)
    return mix64(z)


def uniform01_f64(bits: torch.Tensor) -> torch.Tensor:
    """Top 53 bits -> float64 in [0, 1) (exact)."""
    return _srl(bits, 11).to(torch.float64) * (2.0 ** -53)


def _arange(n: int, device) -> torch.Tensor:
    return torch.arange(n, dtype=torch.int64, device=device)


# ----------------------------------------------------------------- mergesort

def keys_int32(n: int, seed: int = 42, device="cpu") -> torch.Tensor:
    """n keys uniform over the full int32 range ("random 4-byte integer arrays")."""
    h = counter_u64(stream_key(seed, 1), _arange(n, device))
    lo = h & 0xFFFFFFFF
    lo = torch.where(lo >= (1 << 31), lo - (1 << 32), lo)
    return lo.to(torch.int32)


# ---------------------------------------------------------------------- SpMV

def powerlaw_csr(nrows: int, ncols: int | None = None, seed: int = 7, xm: int = 16,
                 deg_cap: int = 1 << 16, device="cpu"):
    """Power-law CSR matrix + dense x (SURVEY.md §8(c) reading 22).

    deg_i = min(floor(xm / sqrt(u_i)), deg_cap), u_i uniform in (0, 1]
    (Pareto alpha=2, mean ~2*xm); columns uniform in [0, ncols) (not sorted,
    duplicates kept); val and x uniform in [0.5, 1.5) (positive, so a relative
    per-row tolerance is meaningful). Returns (row_ptr i32[nrows+1], col i32,
    val f32, x f32[ncols]).
    """
    ncols = nrows if ncols is None else ncols
    r = _arange(nrows, device)
    u = 1.0 - uniform01_f64(counter_u64(stream_key(seed, 11), r))  # (0, 1]
    deg = torch.clamp(torch.floor(xm / torch.sqrt(u)), max=deg_cap).to(torch.int64)
    row_ptr = torch.zeros(nrows + 1, dtype=torch.int64, device=device)
    row_ptr[1:] = torch.cumsum(deg, 0)
    nnz = int(row_ptr[-1].item())
    assert nnz < (1 << 31), "nnz must fit int32 indices"
    e = _arange(nnz, device)
    col = (_srl(counter_u64(stream_key(seed, 12), e), 1) % ncols).to(torch.int32)
    val = (0.5 + _srl(counter_u64(stream_key(seed, 13), e), 41).to(torch.float64)
           * (2.0 ** -23)).to(torch.float32)
    x = (0.5 + _srl(counter_u64(stream_key(seed, 14), _arange(ncols, device)), 41)
         .to(torch.float64) * (2.0 ** -23)).to(torch.float32)
    return row_ptr.to(torch.int32), col, val, x


# ----------------------------------------------------------- synthetic tree

def tree_buffer(n_words: int, seed: int = 9, device="cpu") -> torch.Tensor:
    """n_words pseudo-random 64-bit words (the table do_memory_and_compute reads)."""
    return counter_u64(stream_key(seed, 300), _arange(n_words, device))


# ----------------------------------------------------------------------- BFS

def rmat_csr(scale: int, edgefactor: int = 16, seed: int = 3, a: float = 0.57,
             b: float = 0.19, c: float = 0.19, device="cpu"):
    """Graph500-style RMAT graph as a symmetrised CSR (SURVEY.md §8(c) reading 19).

    2^scale vertices, edgefactor * 2^scale undirected edges; each edge picks one
    quadrant per level with probabilities (a, b, c, 1-a-b-c); a seeded vertex
    permutation relabels the vertices; both directions are stored; self loops
    and duplicate edges are kept (they do not change BFS levels). Adjacency is
    ordered by (src, dst). Returns (row_ptr i32[V+1], col i32[2E]).
    """
    nv = 1 << scale
    ne = edgefactor * nv
    e = _arange(ne, device)
    src = torch.zeros(ne, dtype=torch.int64, device=device)
    dst = torch.zeros(ne, dtype=torch.int64, device=device)
    for lvl in range(scale):
        u = uniform01_f64(counter_u64(stream_key(seed, 100 + lvl), e))
        bi = (u >= a + b).to(torch.int64)                       # lower half: c or d
        bj = ((u >= a) & (u < a + b)) | (u >= a + b + c)        # right half: b or d
        src = src * 2 + bi
        dst = dst * 2 + bj.to(torch.int64)
        del u, bi, bj
    perm = torch.argsort(counter_u64(stream_key(seed, 99), _arange(nv, device)))
    src, dst = perm[src], perm[dst]
    s = torch.cat([src, dst])
    d = torch.cat([dst, src])
    del src, dst
    key = torch.sort(s * nv + d).values
    del s, d
    s = key // nv
    col = (key % nv).to(torch.int32)
    del key
    deg = torch.bincount(s, minlength=nv)
    row_ptr = torch.zeros(nv + 1, dtype=torch.int64, device=device)
    row_ptr[1:] = torch.cumsum(deg, 0)
    assert int(row_ptr[-1]) < (1 << 31)
    return row_ptr.to(torch.int32), col


def bfs_sources(row_ptr: torch.Tensor, k: int, seed: int = 5) -> list[int]:
    """k distinct seeded source vertices with degree > 0 (SURVEY.md reading 18)."""
    rp = row_ptr.to("cpu").to(torch.int64)
    nv = rp.numel() - 1
    deg = rp[1:] - rp[:-1]
    out: list[int] = []
    i = 0
    key = stream_key(seed, 200)
    while len(out) < k and i < 64 * k + 4 * nv:
        v = int(_srl(counter_u64(key, torch.tensor([i])), 1).item() % nv)
        i += 1
        if deg[v] > 0 and v not in out:
            out.append(v)
    return out
