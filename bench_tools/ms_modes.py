"""Mergesort 2^24 (cutoff 128): merge_mode 0 (one-lane merge) vs 1 (warp assist), device ms."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
keys = synth.keys_int32(n, seed=42, device="cuda")
ref = torch.sort(keys).values
d = torch.empty_like(keys)
scr = torch.empty_like(keys)
for mode in (1, 0):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, watchdog_ns=60_000_000_000, **bench.MS_CFG) as rt:
        for it in range(3 if mode else 2):
            d.copy_(keys)
            st = g.mergesort_(d, scr, cutoff=128, merge_mode=mode, rt=rt)
            assert torch.equal(d, ref)
            print(f"mode={mode} n={n} {st.device_ms:.3f} ms  {n / st.device_ms / 1e3:.1f} Mkeys/s  "
                  f"assists={st.assists} cycles={st.cycles} idle={st.idle_cycles}", flush=True)
