"""Mergesort 2^24 (merge_mode 1): device ms for the library in GTAP_LIB at several idle backoffs."""
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

n = 1 << 24
keys = synth.keys_int32(n, seed=42, device="cuda")
ref = torch.sort(keys).values
d = torch.empty_like(keys)
scr = torch.empty_like(keys)
lib = os.path.basename(os.environ.get("GTAP_LIB", "libgtap.so"))
for backoff in tuple(int(b) for b in os.environ.get("BACKOFFS", "1024").split(",")):
    cfg = dict(bench.MS_CFG, idle_backoff_ns=backoff)
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, watchdog_ns=60_000_000_000, **cfg) as rt:
        ms = []
        for it in range(5):
            d.copy_(keys)
            st = g.mergesort_(d, scr, cutoff=128, merge_mode=1, rt=rt)
            assert torch.equal(d, ref)
            ms.append(st.device_ms)
        ms = sorted(ms[1:])
        print(f"{lib:70s} backoff={backoff:6d}  median {ms[len(ms) // 2]:7.3f} ms  min {ms[0]:7.3f}", flush=True)
