"""Synthetic-tree sweeps (§6.3, Fig. binary/pruned tree): thread- vs block-level workers.

Prints one line per point: shape, D, mem_ops, compute_iters, kind, ms, tasks/s.
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

buf = synth.tree_buffer(1 << 25, device="cuda")   # 256 MiB: pseudo-random loads go to HBM
SAME = len(sys.argv) > 2 and sys.argv[2] == "same"   # the paper's protocol: one geometry for both kinds
CFG = {g.GTAP_WORKER_THREAD: dict(grid_size=148 * 8 if SAME else 0, block_size=64 if SAME else 128,
                                  max_tasks_per_worker=4096),
       g.GTAP_WORKER_BLOCK: dict(grid_size=148 * 8 if SAME else 148 * 32, block_size=64 if SAME else 32,
                                 max_tasks_per_worker=2048)}
rts = {k: g.Runtime(k, 0, watchdog_ns=60_000_000_000, **c) for k, c in CFG.items()}
only = sys.argv[1] if len(sys.argv) > 1 else "all"


def point(shape, D, mem, comp):
    out = []
    for k, rt in rts.items():
        ms = []
        for _ in range(3):
            _, st = g.tree(D, buf, mem, comp, pruned=(shape == "pruned"), worker=k, rt=rt)
            ms.append(st.device_ms)
        m = min(ms)
        out.append((k, m, st.tasks))
        print(f"{shape:6s} D={D:2d} mem={mem:5d} comp={comp:5d} "
              f"{'thread' if k == g.GTAP_WORKER_THREAD else 'block ':6s} {m:9.3f} ms  tasks={st.tasks:9d} "
              f"{st.tasks / m / 1e6:8.3f} Gtasks/s  cyc={st.cycles} idle={st.idle_cycles}", flush=True)
    return out


for shape, Ds, D0 in (("full", (12, 16, 20, 22), 18), ("pruned", (16, 20, 24, 28, 32), 24)):
    if only not in ("all", shape):
        continue
    for D in Ds:
        point(shape, D, 64, 256)
    for mem in (0, 256, 2048, 8192):
        point(shape, D0, mem, 256)
    for comp in (0, 2048, 8192, 32768):
        point(shape, D0, 64, comp)
