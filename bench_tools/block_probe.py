"""Block-level workloads at their bench shapes (library from GTAP_LIB): BFS RMAT-22 (2 sources),
SpMV 2^22 rows, full/pruned synthetic trees on block workers; device ms."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

lib = os.path.basename(os.environ.get("GTAP_LIB", "libgtap.so"))
rp, col = synth.rmat_csr(22, 16, seed=3, device="cuda")
srcs = synth.bfs_sources(rp, 2, seed=5)
with g.Runtime(g.GTAP_WORKER_BLOCK, 0, **bench.BFS_CFG) as rt:
    out = []
    for s in srcs:
        ms = []
        for _ in range(3):
            d, st = g.bfs(rp, col, s, rt=rt)
            ms.append(st.device_ms)
        out.append(f"{min(ms):.2f}ms/{st.tasks}")
print(f"{lib:32s} bfs {' '.join(out)}", flush=True)
del rp, col
rp, col, val, x = synth.powerlaw_csr(1 << 22, seed=7, device="cuda")
y = torch.zeros(1 << 22, dtype=torch.float32, device="cuda")
with g.Runtime(g.GTAP_WORKER_BLOCK, 0, **bench.SPMV_CFG) as rt:
    ms = []
    for _ in range(5):
        y, st = g.spmv(rp, col, val, x, y, bench.SPMV_NNZ_CUT, bench.SPMV_FANOUT, parts=bench.SPMV_PARTS, rt=rt)
        ms.append(st.device_ms)
print(f"{lib:32s} spmv {statistics.median(ms[1:]):.3f} ms tasks {st.tasks}", flush=True)
buf = synth.tree_buffer(1 << 25, device="cuda")
cfgb = bench.TREE_CFG["block"]
for name, D, mem, comp, pruned in (("full_D22", 22, 64, 256, False), ("pruned_D24", 24, 64, 32768, True)):
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, **cfgb) as rt:
        ms = []
        for _ in range(3):
            v, st = g.tree(D, buf, mem, comp, pruned=pruned, worker=g.GTAP_WORKER_BLOCK, rt=rt)
            ms.append(st.device_ms)
    print(f"{lib:32s} tree_block_{name} {min(ms):.3f} ms tasks {st.tasks}", flush=True)
