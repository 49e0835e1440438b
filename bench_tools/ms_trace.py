"""Per-merge trace of one 2^24 mergesort (needs libgtap_gtap_ms_trace.so)."""
import sys, os, ctypes, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["GTAP_LIB"] = os.path.join(ROOT, "paper_2604_05982_b200", "libgtap_gtap_ms_trace.so")
sys.path.insert(0, ROOT)
import numpy as np, torch, synth, bench
import paper_2604_05982_b200 as g
from paper_2604_05982_b200 import gtap
n = 1 << 24
keys = synth.keys_int32(n, seed=42, device="cuda"); scratch = torch.empty_like(keys)
L = gtap.lib()
buf = np.zeros((65536, 4), np.uint64); cnt = ctypes.c_uint32()
with g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.MS_CFG) as rt:
    st = g.mergesort_(keys.clone(), scratch, 128, rt=rt)
    L.gtap_ms_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.byref(cnt))
    k2 = keys.clone()
    st = g.mergesort_(k2, scratch, 128, rt=rt)
    L.gtap_ms_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.byref(cnt))
m = int(cnt.value)
t0, t1, sz, sm = buf[:m, 0].astype(np.int64), buf[:m, 1].astype(np.int64), (buf[:m, 2] >> np.uint64(32)).astype(np.int64), buf[:m, 3]
base = t0.min()
print("kernel ms", st.device_ms, "merges traced", m)
for size in sorted(set(sz.tolist()), reverse=True)[:14]:
    sel = sz == size
    used = (sm[sel] & np.uint64(1)).astype(int)
    d = (t1[sel] - t0[sel]) / 1e6
    print(f"size={size:9d} count={sel.sum():5d} tma={used.sum():5d} dur_ms min={d.min():8.3f} max={d.max():8.3f} "
          f"ns/key={d.max()*1e6/size:6.2f} start_ms={(t0[sel].min()-base)/1e6:8.3f} end_ms={(t1[sel].max()-base)/1e6:8.3f} "
          f"distinct_sm={len(set((sm[sel] >> np.uint64(8)).tolist()))}")
