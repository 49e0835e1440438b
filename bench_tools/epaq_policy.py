"""EPAQ kept-class policy sweep (DESIGN R24): fib(40) with cutoffs 6..16, one queue vs 3 queues under
queue_policy 0 (rotate every cycle) and 1 (stay while the class has work, P:177-178 literal).
Median of 5 runs each; prints ms and the speedup of each 3-queue policy over one queue."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402


POOL = int(os.environ.get("POOL", bench.FIB_CFG["max_tasks_per_worker"]))


def run(cutoff, nq, pol):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, num_queues=3, queue_policy=pol,
                   **dict(bench.FIB_CFG, max_tasks_per_worker=POOL)) as rt:
        ms = []
        for i in range(6):
            try:
                v, st = g.fib_cutoff(40, cutoff, nq, rt=rt)
            except g.GtapError as e:
                return f"error {e}"
            assert v == 102334155
            if i:
                ms.append(st.device_ms)
    return statistics.median(ms)


print(f"records per worker: {POOL}")
for cutoff in (6, 8, 10, 12, 14, 16):
    one = run(cutoff, 1, 0)
    r0 = run(cutoff, 3, 0)
    r1 = run(cutoff, 3, 1)
    sp = lambda r: f"{one / r:.2f}x" if isinstance(r, float) else r
    print(f"cutoff {cutoff:2d}: 1 queue {one:.3f} ms | EPAQ rotate {r0 if isinstance(r0, str) else f'{r0:.3f}'} ms "
          f"({sp(r0)}) | EPAQ stay {r1 if isinstance(r1, str) else f'{r1:.3f}'} ms ({sp(r1)})", flush=True)
