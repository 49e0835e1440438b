"""Mergesort 2^24: idle-backoff cap sweep, alternating configurations, median of 8 per round, 3 rounds."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2604_05982_b200 as g
import synth

n = 1 << 24
pristine = synth.keys_int32(n, seed=42, device="cuda")
keys = torch.empty_like(pristine)
scratch = torch.empty_like(pristine)
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
for rnd in range(3):
    for sm_ in (32, 16, 24):
        with g.Runtime(g.GTAP_WORKER_THREAD, 0, **dict(bench.MS_CFG, steal_max=sm_)) as rt:
            ms = []
            for i in range(9):
                keys.copy_(pristine)
                flush.fill_(1)
                st = g.mergesort_(keys, scratch, 128, merge_mode=1, rt=rt)
                if i:
                    ms.append(st.device_ms)
        print(f"round {rnd} steal_max {sm_:3d}: median {statistics.median(ms):.4f} ms  min {min(ms):.4f}", flush=True)
