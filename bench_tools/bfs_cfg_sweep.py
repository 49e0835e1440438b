"""BFS RMAT-22 runtime-parameter sweep (steal_max, idle backoff, grid): 4 sources x 3 runs, median ms."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

rp, col = synth.rmat_csr(22, 16, seed=3, device="cuda")
srcs = synth.bfs_sources(rp, 4, seed=5)
for over in (dict(), dict(steal_max=16), dict(idle_backoff_ns=256), dict(idle_backoff_ns=4096),
             dict(steal_attempts=1), dict(steal_attempts=8)):
    cfg = dict(bench.BFS_CFG, **over)
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, **cfg) as rt:
        ms, tasks = [], []
        for s in srcs:
            for _ in range(3):
                d, st = g.bfs(rp, col, s, rt=rt)
                ms.append(st.device_ms)
                tasks.append(st.tasks)
    print(f"{str(over):28s} median {statistics.median(ms):.2f} ms  mean {statistics.mean(ms):.2f}  tasks {statistics.mean(tasks):.0f}",
          flush=True)
