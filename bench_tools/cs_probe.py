"""Cilksort 2^20..2^24 in both merge modes (device ms, Mkeys/s), at the bench launch configuration."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

for n in [1 << 20, 1 << 22, 1 << 24]:
    pristine = synth.keys_int32(n, seed=42, device="cuda")
    keys = torch.empty_like(pristine)
    scratch = torch.empty_like(pristine)
    for mode in (0, 1):
        for backoff in (8192, 1024):
            with g.Runtime(g.GTAP_WORKER_THREAD, 0, **dict(bench.CS_CFG, idle_backoff_ns=backoff)) as rt:
                ms = []
                for i in range(4):
                    keys.copy_(pristine)
                    st = g.cilksort_(keys, scratch, 64, 256, merge_mode=mode, rt=rt)
                    ms.append(st.device_ms)
            ok = bool(torch.all(keys[1:] >= keys[:-1]).item())
            t = statistics.median(ms[1:])
            print(f"n=2^{n.bit_length() - 1} mode={mode} backoff={backoff} ms={t:.2f} Mkeys/s={n / t / 1e3:.0f} "
                  f"sorted={ok} tasks={st.tasks} assists={st.assists}", flush=True)
