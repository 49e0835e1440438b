"""Block-level steal batch (steal_max 1 = P:92, > 1 = batch) on BFS RMAT-22, SpMV and block-level trees."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

rp, col = synth.rmat_csr(22, 16, seed=3, device="cuda")
srcs = synth.bfs_sources(rp, 2, seed=5)
srp, scol, sval, sx = synth.powerlaw_csr(1 << 22, seed=7, device="cuda")
tbuf = synth.tree_buffer(1 << 25, device="cuda")
for sm in (1, 4, 16, 32):
    out = []
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, watchdog_ns=60_000_000_000, **dict(bench.BFS_CFG, steal_max=sm)) as rt:
        for s in srcs:
            out.append(min(g.bfs(rp, col, s, rt=rt)[1].device_ms for _ in range(3)))
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, steal_max=sm, **bench.SPMV_CFG) as rt:
        sp = statistics.median(g.spmv(srp, scol, sval, sx, None, bench.SPMV_NNZ_CUT, bench.SPMV_FANOUT,
                                      parts=bench.SPMV_PARTS, rt=rt)[1].device_ms for _ in range(4))
        sp1 = statistics.median(g.spmv(srp, scol, sval, sx, None, bench.SPMV_NNZ_CUT, bench.SPMV_FANOUT,
                                       rt=rt)[1].device_ms for _ in range(4))
    tr = []
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, steal_max=sm, **bench.TREE_CFG["block"]) as rt:
        for D, mem, comp, pr in ((22, 64, 256, False), (24, 64, 32768, True), (18, 0, 256, False)):
            tr.append(min(g.tree(D, tbuf, mem, comp, pruned=pr, worker=g.GTAP_WORKER_BLOCK, rt=rt)[1].device_ms
                          for _ in range(3)))
    print(f"steal_max={sm:2d} bfs_ms={out[0]:.2f},{out[1]:.2f} spmv_forest_ms={sp:.3f} spmv_1root_ms={sp1:.3f} "
          f"tree_block_ms(full22,pruned24c32k,full18m0)={tr[0]:.2f},{tr[1]:.3f},{tr[2]:.3f}", flush=True)
