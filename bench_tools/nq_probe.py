"""N-Queens n = 14..17, cutoff 7, both leaf modes (device ms)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402

for n in (14, 16, 17):
    for mode in (0, 1):
        with g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.NQ_CFG) as rt:
            res = [g.nqueens(n, bench.NQ_CUTOFF, leaf_mode=mode, rt=rt) for _ in range(3)]
        t = statistics.median(r[1].device_ms for r in res)
        print(f"n={n} mode={mode} solutions={res[-1][0]} ms={t:.2f} tasks={res[-1][1].tasks} "
              f"assists={res[-1][1].assists} workers={res[-1][1].workers}", flush=True)
