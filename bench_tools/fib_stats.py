"""Scheduler statistics of fib(40) at the bench configuration: cycles, tasks per cycle, pops, steals, idle cycles."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2604_05982_b200 as g

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
with g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.FIB_CFG) as rt:
    for _ in range(3):
        v, st = g.fib(n, rt=rt)
import dataclasses
d = dataclasses.asdict(st)
print({k: d[k] for k in ("tasks", "invocations", "pops", "kept", "steals_ok", "steals_failed", "stolen_tasks", "pushes",
                         "cycles", "idle_cycles", "remote_frees", "max_pool_used", "workers", "device_ms")})
print(f"invocations per busy cycle {d['invocations'] / d['cycles']:.2f}, busy cycles per warp {d['cycles'] / d['workers']:.0f}, "
      f"us per busy cycle per warp {d['device_ms'] * 1e3 / (d['cycles'] / d['workers']):.3f}")
