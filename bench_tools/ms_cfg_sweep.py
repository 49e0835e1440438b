"""Mergesort 2^24 runtime-parameter sweep (steal_attempts, idle backoff): median of 7 runs each."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

n = 1 << 24
pristine = synth.keys_int32(n, seed=42, device="cuda")
keys = torch.empty_like(pristine)
scratch = torch.empty_like(pristine)
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
for over in (dict(), dict(steal_attempts=1), dict(steal_attempts=2), dict(idle_backoff_ns=512),
             dict(steal_attempts=1, idle_backoff_ns=512), dict(steal_attempts=8), dict(steal_max=8)):
    cfg = dict(bench.MS_CFG, **over)
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, **cfg) as rt:
        ms = []
        for i in range(8):
            keys.copy_(pristine)
            flush.fill_(1)
            st = g.mergesort_(keys, scratch, 128, merge_mode=1, rt=rt)
            if i:
                ms.append(st.device_ms)
    print(f"{str(over):45s} median {statistics.median(ms):.4f} ms  min {min(ms):.4f}", flush=True)
