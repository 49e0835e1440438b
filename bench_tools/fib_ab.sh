#!/bin/bash
# in-situ A/B of fib build variants: bench_tools/fib_ab.sh lib1 lib2 ... (paths under paper_2604_05982_b200/)
cd "$(dirname "$0")/.."
for lib in "$@"; do
  GTAP_LIB=$PWD/paper_2604_05982_b200/$lib timeout 300 python - <<PY
import statistics, sys
sys.path.insert(0, ".")
import bench, paper_2604_05982_b200 as g
for n, cfg, reps in ((40, bench.FIB_CFG, 7), (20, dict(bench.FIB_CFG, idle_backoff_ns=1024), 21)):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, **cfg) as rt:
        ms = []
        for i in range(reps):
            v, st = g.fib(n, rt=rt)
            assert v == bench._fib_value(n), v
            ms.append(st.device_ms)
    print("$lib", f"fib({n})", f"median {statistics.median(ms[1:]):.3f} ms", f"min {min(ms[1:]):.3f}", "tasks", st.tasks, "workers", st.workers)
PY
done
