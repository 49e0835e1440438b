"""fib(20) launch-configuration sweep (span-bound C1): median of 21 runs per configuration."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2604_05982_b200 as g

base = bench.FIB20_CFG
for over in (dict(), dict(idle_backoff_ns=64), dict(idle_backoff_ns=128), dict(grid_size=148, block_size=32),
             dict(grid_size=148, block_size=32, idle_backoff_ns=128), dict(grid_size=74, block_size=64),
             dict(grid_size=296, block_size=64), dict(steal_attempts=1), dict(steal_attempts=2),
             dict(grid_size=148, block_size=128), dict(max_tasks_per_worker=1024)):
    cfg = dict(base, **over)
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, **cfg) as rt:
        ms = []
        for i in range(22):
            v, st = g.fib(20, rt=rt)
            assert v == 6765
            if i:
                ms.append(st.device_ms)
    print(f"{str(over):55s} median {statistics.median(ms) * 1e3:7.1f} us  min {min(ms) * 1e3:7.1f}", flush=True)
