"""Problem-size sweeps at the bench launch configurations (the paper plots fib and mergesort against n):
fib(n) tasks/s for n = 20..40 and mergesort Mkeys/s for n = 2^16..2^26 in both merge modes
(one-lane mode up to 2^22), device-timed medians."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

with g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.FIB_CFG) as rt:
    for n in (20, 24, 28, 32, 36, 40):
        ms = []
        for _ in range(5):
            v, st = g.fib(n, rt=rt)
            ms.append(st.device_ms)
        t = statistics.median(ms[1:])
        print(f"fib({n:2d}) = {v:10d}  tasks {st.tasks:11d}  {t:9.3f} ms  {st.tasks / t / 1e6:8.3f} G tasks/s", flush=True)
for lg in range(16, 27, 2):
    n = 1 << lg
    pristine = synth.keys_int32(n, seed=42, device="cuda")
    keys = torch.empty_like(pristine)
    scratch = torch.empty_like(pristine)
    for mode, cfg in ((1, bench.MS_CFG), (0, bench.MS0_CFG)):
        if mode == 0 and lg > 22:
            continue
        with g.Runtime(g.GTAP_WORKER_THREAD, 0, **cfg) as rt:
            table = g.Table.mergesort(keys, scratch, 128, mode)
            ms = []
            for _ in range(4 if mode else 2):
                keys.copy_(pristine)
                rt.reset()
                rt.spawn_root(table, (0, n))
                rt.run()
                st = rt.sync()
                ms.append(st.device_ms)
            table.close()
        ok = bool(torch.all(keys[1:] >= keys[:-1]).item())
        t = statistics.median(ms[1:]) if len(ms) > 1 else ms[0]
        print(f"mergesort 2^{lg} mode={mode}  {t:10.3f} ms  {n / t / 1e3:9.1f} Mkeys/s  sorted={ok}", flush=True)
