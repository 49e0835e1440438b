"""Timeline of one 2^24 mergesort (merge_mode 1 by default) from the GTAP_MS_TRACE build.

usage: python bench_tools/ms_trace.py [merge_mode] [idle_backoff_ns]
Per (kind, size): count, first start / last end (ms from the first record), mean duration.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("GTAP_LIB", os.path.join(ROOT, "paper_2604_05982_b200", "libgtap_gtap_ms_trace.so"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402
from paper_2604_05982_b200 import gtap  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
backoff = int(sys.argv[2]) if len(sys.argv) > 2 else bench.MS_CFG["idle_backoff_ns"]
KIND = {0: "lane merge", 1: "TMA merge", 2: "leaf sort", 3: "warp assist", 4: "block assist", 5: "GPU assist",
        6: "GPU chunk", 7: "block chunk"}
n = 1 << 24
keys = synth.keys_int32(n, seed=42, device="cuda")
scratch = torch.empty_like(keys)
L = gtap.lib()
cap = 1 << 20
buf = np.zeros((cap, 4), np.uint64)
cnt = ctypes.c_uint32()
with g.Runtime(g.GTAP_WORKER_THREAD, 0, **dict(bench.MS_CFG, idle_backoff_ns=backoff)) as rt:
    for _ in range(2):
        k2 = keys.clone()
        L.gtap_ms_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.byref(cnt))
        st = g.mergesort_(k2, scratch, 128, merge_mode=mode, rt=rt)
        L.gtap_ms_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.byref(cnt))
m = min(int(cnt.value), cap)
t0, t1 = buf[:m, 0].astype(np.int64), buf[:m, 1].astype(np.int64)
sz = (buf[:m, 2] >> np.uint64(32)).astype(np.int64)
kind = (buf[:m, 3] & np.uint64(255)).astype(np.int64)
base = t0.min()
print(f"mode={mode} backoff={backoff} kernel_ms={st.device_ms:.3f} records={m} span_ms={(t1.max() - base) / 1e6:.3f}")
for k in sorted(set(kind.tolist())):
    for size in sorted(set(sz[kind == k].tolist()), reverse=True):
        sel = (kind == k) & (sz == size)
        if sel.sum() < 1:
            continue
        d = (t1[sel] - t0[sel]) / 1e3
        print(f"{KIND[k]:12s} size={size:9d} n={sel.sum():6d} start={(t0[sel].min() - base) / 1e6:7.3f} "
              f"end={(t1[sel].max() - base) / 1e6:7.3f} ms  dur_us mean={d.mean():8.1f} max={d.max():8.1f}")
