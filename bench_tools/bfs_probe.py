"""BFS RMAT-22 at the bench configuration (library from GTAP_LIB): 4 sources x 4 runs, median ms."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

lib = os.path.basename(os.environ.get("GTAP_LIB", "libgtap.so"))
rp, col = synth.rmat_csr(22, 16, seed=3, device="cuda")
srcs = synth.bfs_sources(rp, 4, seed=5)
with g.Runtime(g.GTAP_WORKER_BLOCK, 0, **bench.BFS_CFG) as rt:
    ms, tasks = [], []
    for s in srcs:
        for _ in range(4):
            d, st = g.bfs(rp, col, s, rt=rt)
            ms.append(st.device_ms)
            tasks.append(st.tasks)
print(f"{lib:32s} bfs median {statistics.median(ms):.2f} ms  mean {statistics.mean(ms):.2f}  tasks {statistics.mean(tasks):.0f}",
      flush=True)
