"""Histogram of tasks per busy warp-cycle for fib(40) (GTAP_CYC_HIST build): python bench_tools/fib_cyc_hist.py."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("GTAP_LIB", os.path.join(ROOT, "paper_2604_05982_b200", "libgtap_gtap_cyc_hist.so"))
sys.path.insert(0, ROOT)
import bench
import paper_2604_05982_b200 as g
from paper_2604_05982_b200 import gtap

L = gtap.lib()
h = (ctypes.c_ulonglong * 40)()
with g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.FIB_CFG) as rt:
    g.fib(40, rt=rt)
    L.gtap_cyc_hist_read(h)
    v, st = g.fib(int(sys.argv[1]) if len(sys.argv) > 1 else 40, rt=rt)
    L.gtap_cyc_hist_read(h)
cyc = sum(h[1:33])
inv = sum(k * h[k] for k in range(1, 33))
print(f"cycles {cyc} invocations {inv} mean {inv / cyc:.2f}; full cycles {h[32] / cyc:.3f}")
print("n: share of cycles", " ".join(f"{k}:{h[k] / cyc:.3f}" for k in range(1, 33) if h[k] / cyc > 0.004))
print(f"partial cycles with an empty private part and a non-empty own public part: {h[33] / cyc:.3f} of cycles, "
      f"mean public tasks {h[34] / max(h[33], 1):.1f}")
