"""fib(40) runtime-parameter sweep at the bench configuration: median of 5 device times per configuration."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2604_05982_b200 as g

for over in (dict(), dict(block_size=64), dict(block_size=256), dict(max_tasks_per_worker=2048),
             dict(max_tasks_per_worker=8192), dict(steal_attempts=2), dict(steal_attempts=8), dict(steal_max=16),
             dict(idle_backoff_ns=2048), dict(idle_backoff_ns=32768), dict()):
    cfg = dict(bench.FIB_CFG, **over)
    try:
        with g.Runtime(g.GTAP_WORKER_THREAD, 0, **cfg) as rt:
            ms = []
            for i in range(6):
                v, st = g.fib(40, rt=rt)
                assert v == 102334155
                if i:
                    ms.append(st.device_ms)
        print(f"{str(over):40s} median {statistics.median(ms):.3f} ms  min {min(ms):.3f}  workers {st.workers}", flush=True)
    except Exception as e:
        print(f"{str(over):40s} {e}", flush=True)
