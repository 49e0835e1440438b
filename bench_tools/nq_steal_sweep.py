"""N-Queens 16 (cutoff 7) steal_max / backoff sweep at the bench configuration: median of 5."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2604_05982_b200 as g

for over in (dict(), dict(steal_max=16), dict(steal_max=8), dict(steal_max=4), dict(idle_backoff_ns=1024),
             dict(idle_backoff_ns=256), dict()):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, **dict(bench.NQ_CFG, **over)) as rt:
        ms = []
        for i in range(6):
            c, st = g.nqueens(bench.NQ_N, bench.NQ_CUTOFF, rt=rt)
            assert c == 14772512
            if i:
                ms.append(st.device_ms)
    print(f"{str(over):32s} median {statistics.median(ms):.3f} ms min {min(ms):.3f}", flush=True)
