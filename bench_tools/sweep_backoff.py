import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, bench
import paper_2604_05982_b200 as g
n = 1 << 24
pristine = synth.keys_int32(n, seed=42, device="cuda")
keys = torch.empty_like(pristine); scratch = torch.empty_like(pristine)
for bo in [int(a) for a in sys.argv[1:]] or [2048, 8192, 32768, 131072]:
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, idle_backoff_ns=bo, **bench.MS_CFG) as rt:
        ms = []
        for i in range(3):
            keys.copy_(pristine); ms.append(g.mergesort_(keys, scratch, 128, rt=rt).device_ms)
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, idle_backoff_ns=bo, **bench.FIB_CFG) as rt:
        fm = [g.fib(40, rt=rt)[1].device_ms for _ in range(3)]
    print(f"backoff={bo} mergesort2^24 ms={statistics.median(ms):.1f} fib40 ms={statistics.median(fm):.2f}", flush=True)
