"""SpMV at the bench shape: forest size (parts) x fanout x nnz_cut x idle backoff, median of 7 device times each."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2604_05982_b200 as g
import synth

rp, col, val, x = synth.powerlaw_csr(1 << 22, seed=7, device="cuda")
y = torch.empty(1 << 22, dtype=torch.float32, device="cuda")
for backoff in (1024, 256, 4096):
    cfg = dict(bench.SPMV_CFG, idle_backoff_ns=backoff, max_roots=2368)
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, **cfg) as rt:
        for parts in (592, 1184, 2368):
            for fanout, cut in ((4, 65536), (2, 65536), (8, 65536), (4, 32768), (4, 131072), (4, 1 << 30)):
                if backoff != 1024 and (parts, fanout, cut) != (592, 4, 65536):
                    continue
                ms = []
                for i in range(8):
                    y.zero_()
                    _, st = g.spmv(rp, col, val, x, y, nnz_cut=cut, fanout=fanout, parts=parts, rt=rt)
                    if i:
                        ms.append(st.device_ms)
                print(f"backoff {backoff:5d} parts {parts:5d} fanout {fanout} cut {cut:>10d}: median {statistics.median(ms):.4f} ms "
                      f"min {min(ms):.4f} tasks {st.tasks}", flush=True)
