import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_05982_b200 as g
import bench
for cutoff in (2, 6, 10, 14):
    res = {}
    for nq in (1, 3):
        cfg = dict(bench.FIB_CFG, max_tasks_per_worker=4096)
        with g.Runtime(g.GTAP_WORKER_THREAD, 0, num_queues=3, **cfg) as rt:
            ms = [g.fib_cutoff(40, cutoff, nq, rt=rt)[1] for _ in range(3)]
        res[nq] = statistics.median(s.device_ms for s in ms)
    print(f"fib(40) cutoff={cutoff}: 1 queue {res[1]:.2f} ms, EPAQ 3 queues {res[3]:.2f} ms, speedup {res[1]/res[3]:.2f}x", flush=True)
