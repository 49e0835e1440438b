"""Small runs of the hot tables for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

usage: compute-sanitizer --tool <tool> python bench_tools/sanitize_probe.py <fib|ms|ms0|spmv|bfs|bfs1|bfs32|tree|cs|nq|fibdie>

Each run is checked against the oracle so a sanitizer-clean run is also a correct one; sizes are small
(the sanitizers slow every memory access down by 10-100x) but span several workers, steals and, for
mergesort, the warp / block / GPU-wide assist paths.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402

WD = 120_000_000_000
what = sys.argv[1]
if what in ("fib", "fibdie"):
    v, st = g.fib(16, grid_size=148, block_size=128, max_tasks_per_worker=1024, watchdog_ns=WD,
                  victim_policy=1 if what == "fibdie" else 0)
    assert (v, st.tasks, st.invocations) == oracle.fib(16)
elif what in ("ms", "ms0"):
    n = 1 << 17 if what == "ms" else 1 << 13
    keys = synth.keys_int32(n, seed=3).numpy()
    d = torch.from_numpy(keys).cuda()
    st = g.mergesort_(d, merge_mode=1 if what == "ms" else 0, grid_size=148, block_size=128,
                      max_tasks_per_worker=1024, watchdog_ns=WD)
    ref, tasks, _ = oracle.mergesort(keys, 128)
    assert np.array_equal(d.cpu().numpy(), ref) and st.tasks == tasks
elif what == "cs":
    keys = synth.keys_int32(1 << 15, seed=3).numpy()
    d = torch.from_numpy(keys).cuda()
    st = g.cilksort_(d, None, 64, 256, grid_size=148, block_size=128, watchdog_ns=WD)
    ref = oracle.cilksort(keys, 64, 256)
    assert np.array_equal(d.cpu().numpy(), ref[0]) and st.tasks == ref[1]
elif what == "nq":
    c, st = g.nqueens(9, 4, grid_size=148, block_size=128, watchdog_ns=WD)
    assert (c, st.tasks) == oracle.nqueens(9, 4)
elif what == "spmv":
    rp, col, val, x = synth.powerlaw_csr(1 << 12, seed=2)
    y, st = g.spmv(rp.cuda(), col.cuda(), val.cuda(), x.cuda(), None, 512, 4, grid_size=148, block_size=128,
                   watchdog_ns=WD)
    y64, _ = oracle.spmv(rp, col, val, x)
    e = np.abs(y.cpu().numpy().astype(np.float64) - y64) / np.maximum(np.abs(y64), 1e-30)
    assert np.all((y64 == 0) | (e <= 1e-5))
elif what == "bfs32":   # the bench's shape: one-warp blocks (128-entry staging kernel), hub pieces, oldest-first pops
    rp, col = synth.rmat_csr(12, 16, seed=4)
    src = synth.bfs_sources(rp, 1, seed=4)[0]
    depth, st = g.bfs(rp.cuda(), col.cuda(), src, grid_size=148 * 4, block_size=32, max_tasks_per_worker=1 << 13,
                      steal_max=32, watchdog_ns=WD, order=1, edge_split=64)
    assert np.array_equal(depth.cpu().numpy(), oracle.bfs(rp, col, src))
elif what in ("bfs", "bfs1"):
    rp, col = synth.rmat_csr(10, 16, seed=4)
    src = synth.bfs_sources(rp, 1, seed=4)[0]
    depth, st = g.bfs(rp.cuda(), col.cuda(), src, grid_size=148, block_size=64, max_tasks_per_worker=1 << 14,
                      steal_max=32, watchdog_ns=WD, order=1 if what == "bfs1" else 0)
    assert np.array_equal(depth.cpu().numpy(), oracle.bfs(rp, col, src))
elif what == "tree":
    buf_cpu = synth.tree_buffer(1 << 12)
    buf = buf_cpu.cuda()
    for kind in (g.GTAP_WORKER_THREAD, g.GTAP_WORKER_BLOCK):
        v, st = g.tree(8, buf, 4, 8, worker=kind, grid_size=148, block_size=64, watchdog_ns=WD)
        assert (v, st.tasks) == oracle.tree(8, buf_cpu.numpy().view(np.uint64), 4, 8)
else:
    raise SystemExit(f"unknown table {what}")
torch.cuda.synchronize()
print(f"{what}: ok ({st.tasks} tasks)")
