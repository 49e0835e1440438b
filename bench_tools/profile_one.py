"""Run one workload a few times (for ncu): python bench_tools/profile_one.py {ms,fib,spmv,bfs} [size] [reps]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2604_05982_b200 as g
import bench

wl = sys.argv[1]
size = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if wl == "ms":
    n = size or (1 << 20)
    pristine = synth.keys_int32(n, seed=42, device="cuda")
    keys = torch.empty_like(pristine); scratch = torch.empty_like(pristine)
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.MS_CFG) as rt:
        for i in range(reps):
            keys.copy_(pristine)
            st = g.mergesort_(keys, scratch, 128, merge_mode=bench.MS_MERGE_MODE, rt=rt)
            print("ms", n, st.device_ms, flush=True)
elif wl == "fib":
    n = size or 30
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.FIB_CFG) as rt:
        for i in range(reps):
            v, st = g.fib(n, rt=rt)
            print("fib", n, v, st.device_ms, st.tasks, flush=True)
elif wl == "spmv":
    rows = size or (1 << 22)
    rp, col, val, x = synth.powerlaw_csr(rows, seed=7, device="cuda")
    parts = int(os.environ.get("SPMV_PARTS", getattr(bench, "SPMV_PARTS", 0)))
    cut = int(os.environ.get("SPMV_CUT", bench.SPMV_NNZ_CUT))
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, **dict(bench.SPMV_CFG, max_roots=max(parts, 1))) as rt:
        for i in range(reps):
            y, st = g.spmv(rp, col, val, x, nnz_cut=cut, fanout=bench.SPMV_FANOUT, parts=parts, rt=rt)
            print("spmv", rows, st.device_ms, st.tasks, flush=True)
elif wl == "nq":
    n = size or 14
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.NQ_CFG) as rt:
        for i in range(reps):
            c, st = g.nqueens(n, bench.NQ_CUTOFF, rt=rt)
            print("nq", n, c, st.device_ms, st.tasks, flush=True)
elif wl == "bfs":
    scale = size or 22
    rp, col = synth.rmat_csr(scale, 16, seed=3, device="cuda")
    src = synth.bfs_sources(rp, 1, seed=5)[0]
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, **bench.BFS_CFG) as rt:
        for i in range(reps):
            d, st = g.bfs(rp, col, src, rt=rt, order=bench.BFS_ORDER, edge_split=bench.BFS_SPLIT)
            print("bfs", scale, st.device_ms, st.tasks, flush=True)
torch.cuda.synchronize()
