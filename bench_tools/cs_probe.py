import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, bench
import paper_2604_05982_b200 as g
for n in [1 << 20, 1 << 22, 1 << 24]:
    pristine = synth.keys_int32(n, seed=42, device="cuda")
    keys = torch.empty_like(pristine); scratch = torch.empty_like(pristine)
    for cfg in [bench.CS_CFG, dict(bench.CS_CFG, block_size=64)]:
        with g.Runtime(g.GTAP_WORKER_THREAD, 0, **cfg) as rt:
            ms = []
            for i in range(4):
                keys.copy_(pristine); st = g.cilksort_(keys, scratch, 64, 256, rt=rt); ms.append(st.device_ms)
        ok = bool(torch.all(keys[1:] >= keys[:-1]).item())
        print(f"n=2^{n.bit_length()-1} block={cfg['block_size']} ms={statistics.median(ms[1:]):.2f} Mkeys/s={n/statistics.median(ms[1:])/1e3:.0f} sorted={ok} tasks={st.tasks} workers={st.workers}", flush=True)
