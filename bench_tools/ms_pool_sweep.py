import os, statistics, sys
sys.path.insert(0, "/root/repo")
import torch, bench, synth
import paper_2604_05982_b200 as g
n = 1 << 24
pristine = synth.keys_int32(n, seed=42, device="cuda")
keys = torch.empty_like(pristine); scratch = torch.empty_like(pristine)
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
for rnd in range(2):
    for over in (dict(), dict(max_tasks_per_worker=512), dict(max_tasks_per_worker=256), dict(max_tasks_per_worker=4096)):
        with g.Runtime(g.GTAP_WORKER_THREAD, 0, **dict(bench.MS_CFG, **over)) as rt:
            ms = []
            for i in range(9):
                keys.copy_(pristine); flush.fill_(1)
                st = g.mergesort_(keys, scratch, 128, merge_mode=1, rt=rt)
                if i: ms.append(st.device_ms)
        print(rnd, over, "median %.4f" % statistics.median(ms), "min %.4f" % min(ms), "maxpool", st.max_pool_used, flush=True)
