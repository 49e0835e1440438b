import sys, os, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["GTAP_LIB"] = os.path.join(ROOT, "paper_2604_05982_b200", "libgtap_gtap_ms_probe_stats.so")
sys.path.insert(0, ROOT)
import numpy as np, torch, synth, bench
import paper_2604_05982_b200 as g
from paper_2604_05982_b200 import gtap
n = 1 << 24
keys = synth.keys_int32(n, seed=42, device="cuda"); scratch = torch.empty_like(keys)
L = gtap.lib(); pr = (ctypes.c_longlong * 8)()
with g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.MS_CFG) as rt:
    for i in range(2):
        st = g.mergesort_(keys.clone(), scratch, 128, rt=rt)
        L.gtap_ms_probe_read(pr)
        print("kernel ms", st.device_ms, "largest merge n", pr[7], "cycles total", pr[0], "hot", pr[1], "stretches", pr[2],
              "fast_steps", pr[3], "checked", pr[4], "hot cyc/step", pr[1] / max(pr[3], 1), flush=True)
