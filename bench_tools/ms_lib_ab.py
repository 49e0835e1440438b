"""A/B of mergesort library builds at 2^24 (bench MS_CFG, L2 flushed, median of 9 per build, builds interleaved):
python bench_tools/ms_lib_ab.py libA.so libB.so ... (under paper_2604_05982_b200/)."""
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import os, statistics, sys
sys.path.insert(0, %r)
import torch, bench, synth, paper_2604_05982_b200 as g
n = 1 << 24
pristine = synth.keys_int32(n, seed=42, device="cuda"); keys = torch.empty_like(pristine); scratch = torch.empty_like(pristine)
flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
with g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.MS_CFG) as rt:
    ms = []
    for i in range(10):
        keys.copy_(pristine); flush.fill_(1)
        st = g.mergesort_(keys, scratch, 128, merge_mode=1, rt=rt)
        if i: ms.append(st.device_ms)
assert bool(torch.all(keys[1:] >= keys[:-1]).item())
print(statistics.median(ms))
"""
res = {lib: [] for lib in sys.argv[1:]}
for rnd in range(3):
    for lib in sys.argv[1:]:
        env = dict(os.environ, GTAP_LIB=os.path.join(ROOT, "paper_2604_05982_b200", lib))
        out = subprocess.run([sys.executable, "-c", CHILD % ROOT], env=env, capture_output=True, text=True)
        res[lib].append(float(out.stdout.strip().splitlines()[-1]))
for lib, v in res.items():
    print(f"{lib:50s} median {statistics.median(v):.4f} ms  runs {[round(x, 4) for x in v]}")
