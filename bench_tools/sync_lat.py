"""Host-side latency of one small run (gtap_spawn_root + gtap_run + gtap_sync) with the library in GTAP_LIB."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_05982_b200 as g  # noqa: E402

lib = os.path.basename(os.environ.get("GTAP_LIB", "libgtap.so"))
with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148 * 4, block_size=128, max_tasks_per_worker=1024) as rt:
    for rep in range(3):
        t0 = time.perf_counter()
        for _ in range(200):
            v, st = g.fib(10, rt=rt)
        dt = (time.perf_counter() - t0) / 200 * 1e6
        print(f"{lib:24s} fib(10) run+sync {dt:.1f} us/call (device {st.device_ms * 1e3:.1f} us)", flush=True)
