"""Quick mergesort timing probe (not the bench): device ms per run at several sizes."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2604_05982_b200 as g
import bench

sizes = [int(a) for a in sys.argv[1:]] or [1 << 20, 1 << 22, 1 << 24]
for n in sizes:
    pristine = synth.keys_int32(n, seed=42, device="cuda")
    keys = torch.empty_like(pristine); scratch = torch.empty_like(pristine)
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.MS_CFG) as rt:
        ms = []
        for i in range(4):
            keys.copy_(pristine)
            st = g.mergesort_(keys, scratch, 128, rt=rt)
            ms.append(st.device_ms)
        ok = bool(torch.all(keys[1:] >= keys[:-1]).item())
        print(f"n=2^{n.bit_length()-1} ms={statistics.median(ms[1:]):.2f} Mkeys/s={n/statistics.median(ms[1:])/1e3:.1f} "
              f"ns/step={statistics.median(ms[1:])*1e6/(2*n):.2f} sorted={ok} tasks={st.tasks} workers={st.workers}", flush=True)
