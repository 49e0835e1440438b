"""Cilksort 2^24 runtime-parameter sweep at the bench configuration: median of 5 per configuration."""
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
OVERS = [dict(), dict(idle_backoff_ns=256), dict(idle_backoff_ns=512), dict(idle_backoff_ns=4096),
         dict(steal_attempts=2), dict(steal_attempts=8), dict(steal_max=8), dict(block_size=64), dict()]
if len(sys.argv) > 1 and sys.argv[1] == "steal":
    OVERS = [dict(steal_max=s) for s in (32, 16, 8, 4, 2, 1, 8, 32)]
for over in OVERS:
    try:
        with g.Runtime(g.GTAP_WORKER_THREAD, 0, **dict(bench.CS_CFG, **over)) as rt:
            ms = []
            for i in range(6):
                keys.copy_(pristine)
                st = g.cilksort_(keys, scratch, 64, 256, rt=rt)
                if i:
                    ms.append(st.device_ms)
        print(f"{str(over):32s} median {statistics.median(ms):.3f} ms min {min(ms):.3f}", flush=True)
    except Exception as e:
        print(over, e, flush=True)
