cd /root/repo
for lib in "$@"; do GTAP_LIB=$PWD/paper_2604_05982_b200/$lib timeout 300 python - <<PY
import statistics, sys, torch
sys.path.insert(0, ".")
import bench, synth, paper_2604_05982_b200 as g
rp, col, val, x = synth.powerlaw_csr(1 << 22, seed=7, device="cuda")
y = torch.empty(1 << 22, dtype=torch.float32, device="cuda")
with g.Runtime(g.GTAP_WORKER_BLOCK, 0, **bench.SPMV_CFG) as rt:
    ms = []
    for i in range(9):
        y.zero_()
        _, st = g.spmv(rp, col, val, x, y, nnz_cut=bench.SPMV_NNZ_CUT, fanout=bench.SPMV_FANOUT, parts=bench.SPMV_PARTS, rt=rt)
        if i: ms.append(st.device_ms)
print("$lib", "median %.4f ms" % statistics.median(ms), "min %.4f" % min(ms), flush=True)
PY
done
