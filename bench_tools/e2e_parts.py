"""Where the mergesort e2e step goes: H2D 64 MB, gtap_reset, sort (run + sync), D2H 64 MB (CUDA events)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

n = bench.MS_N
keys0 = synth.keys_int32(n, seed=42, device="cuda")
host_in = keys0.cpu().pin_memory()
host_out = torch.empty_like(host_in).pin_memory()
keys = torch.empty_like(keys0)
scratch = torch.empty_like(keys0)
rt = g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.MS_CFG)
s = torch.cuda.current_stream()
rows = []
for it in range(6):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record(s)
    keys.copy_(host_in, non_blocking=True)
    ev[1].record(s)
    rt.reset(s)
    ev[2].record(s)
    st = g.mergesort_(keys, scratch, bench.MS_CUTOFF, merge_mode=bench.MS_MERGE_MODE, rt=rt, stream=s)
    ev[3].record(s)
    host_out.copy_(keys, non_blocking=True)
    ev[4].record(s)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    rows.append([ev[i].elapsed_time(ev[i + 1]) for i in range(4)] + [ev[0].elapsed_time(ev[4]), st.device_ms, wall])
for r in rows[1:]:
    print("h2d %.3f  reset %.3f  sort(run+sync) %.3f  d2h %.3f  | e2e %.3f  kernel %.3f  wall %.3f" % tuple(r))
