"""SM -> L2-die map of this B200 (SURVEY §8(d) probe (vi)) and the A/B of die-aware steal-victim choice
(gtap_config.victim_policy 1) on fib(40), SpMV and BFS. Writes a table to stdout."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
from paper_2604_05982_b200 import gtap  # noqa: E402

buf = torch.zeros(256 * 2048 // 4, dtype=torch.int32, device="cuda")
r = gtap.ubench_die_probe(buf, 256)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
die = r["sm_die"][:nsm]
print(f"SMs {nsm}: die 0 {int((die == 0).sum())}, die 1 {int((die == 1).sum())}; near {r['near_cycles']:.1f} cycles, "
      f"far {r['far_cycles']:.1f} cycles (+{r['far_cycles'] - r['near_cycles']:.1f}); consistency {r['consistency']:.3f}; "
      f"addresses near die 0: {int((r['addr_near'] == 0).sum())} / 256")
print("sm_die:", "".join(str(int(x)) for x in die))
r2 = gtap.ubench_die_probe(buf, 256)
same = (r2["sm_die"][:nsm] == die).mean()
print(f"repeat: sm_die identical for {100 * max(same, 1 - same):.1f}% of SMs (labels may swap)")

dev = torch.device("cuda", 0)
for pol in (0, 1, 0, 1):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, victim_policy=pol, **bench.FIB_CFG) as rt:
        ms = []
        for i in range(6):
            v, st = g.fib(40, rt=rt)
            assert v == 102334155
            if i:
                ms.append(st.device_ms)
    print(f"victim_policy {pol}: fib(40) median {statistics.median(ms):.3f} ms, steals {st.steals_ok}")
for pol in (0, 1):
    cfg_s, cfg_b = bench.SPMV_CFG, bench.BFS_CFG
    bench.SPMV_CFG = dict(cfg_s, victim_policy=pol)
    bench.BFS_CFG = dict(cfg_b, victim_policy=pol)
    s = bench.bench_spmv(dev)
    b = bench.bench_bfs(dev)
    bench.SPMV_CFG, bench.BFS_CFG = cfg_s, cfg_b
    print(f"victim_policy {pol}: SpMV {s['ms']:.3f} ms, BFS median {b['ms']:.3f} ms ({b['value']:.2f} GTEPS)")
