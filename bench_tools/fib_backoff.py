"""fib(20) / fib(32) / fib(40) device ms against the idle backoff cap (bench FIB_CFG otherwise)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402

for bo in (8192, 2048, 1024, 256):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, **dict(bench.FIB_CFG, idle_backoff_ns=bo)) as rt:
        row = []
        for n, reps in ((20, 21), (32, 6), (40, 4)):
            ms = []
            for _ in range(reps):
                v, st = g.fib(n, rt=rt)
                ms.append(st.device_ms)
            row.append(f"fib({n}) {statistics.median(ms[1:]):.3f} ms")
    print(f"backoff {bo:5d}: " + "  ".join(row), flush=True)
