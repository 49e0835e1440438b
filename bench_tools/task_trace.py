"""Task timeline of one block-level run (needs libgtap_gtap_trace.so): spmv or bfs."""
import sys, os, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["GTAP_LIB"] = os.path.join(ROOT, "paper_2604_05982_b200", "libgtap_gtap_trace.so")
sys.path.insert(0, ROOT)
import numpy as np, torch, synth, bench
import paper_2604_05982_b200 as g
from paper_2604_05982_b200 import gtap
wl = sys.argv[1]
L = gtap.lib()
cap = 1 << 22
buf = np.zeros((cap, 4), np.uint64)  # 32 B records
n = ctypes.c_uint32()
reader = getattr(L, f"gtap_trace_read_{wl}")
if wl == "spmv":
    rp, col, val, x = synth.powerlaw_csr(1 << 22, seed=7, device="cuda")
    cut, fan = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (bench.SPMV_NNZ_CUT, bench.SPMV_FANOUT)
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, **bench.SPMV_CFG) as rt:
        for i in range(2):
            y, st = g.spmv(rp, col, val, x, nnz_cut=cut, fanout=fan, rt=rt)
            reader(buf.ctypes.data_as(ctypes.c_void_p), cap, ctypes.byref(n))
else:
    rp, col = synth.rmat_csr(int(sys.argv[2]) if len(sys.argv) > 2 else 20, 16, seed=3, device="cuda")
    src = synth.bfs_sources(rp, 1, seed=5)[0]
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, **bench.BFS_CFG) as rt:
        for i in range(2):
            d, st = g.bfs(rp, col, src, rt=rt)
            reader(buf.ctypes.data_as(ctypes.c_void_p), cap, ctypes.byref(n))
m = min(int(n.value), cap)
t0 = buf[:m, 0].astype(np.int64); t1 = buf[:m, 1].astype(np.int64)
who = (buf[:m, 2] & np.uint64(0xFFFFFFFF)).astype(np.int64)
blk = who & 0xFFFFFF
base = t0.min(); end = t1.max()
dur = (t1 - t0) / 1e3
print(f"{wl}: kernel_ms={st.device_ms:.3f} tasks={m} span_us={(end-base)/1e3:.1f} task_us mean={dur.mean():.2f} "
      f"p50={np.median(dur):.2f} p99={np.percentile(dur,99):.2f} max={dur.max():.1f} sum_busy_ms={dur.sum()/1e3:.1f} "
      f"blocks_used={len(set(blk.tolist()))}")
# busy fraction over time in 20 bins
bins = np.linspace(base, end, 21)
busy = np.zeros(20)
for a, b in zip(t0, t1):
    i0 = np.searchsorted(bins, a) - 1; i1 = np.searchsorted(bins, b) - 1
    for i in range(max(i0, 0), min(i1, 19) + 1):
        busy[i] += min(b, bins[i + 1]) - max(a, bins[i])
nblk = int(st.grid_size)
print("busy fraction per 5% of time:", " ".join(f"{v/((bins[1]-bins[0])*nblk):.2f}" for v in busy))
first = np.sort(t0)[:: max(1, m // 20)]
print("task start times (us, every 5%):", " ".join(f"{(v-base)/1e3:.0f}" for v in first))
