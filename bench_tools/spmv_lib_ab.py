"""A/B of SpMV library builds / block sizes at the bench shape (2^22 rows): python bench_tools/spmv_lib_ab.py
lib[:grid:block] ... (libs under paper_2604_05982_b200/); median of the bench leg, builds interleaved 2 rounds."""
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import os, sys
sys.path.insert(0, %r)
import torch, bench
g, b = os.environ.get("SP_GRID"), os.environ.get("SP_BLOCK")
if g:
    bench.SPMV_CFG = dict(bench.SPMV_CFG, grid_size=int(g), block_size=int(b))
r = bench.bench_spmv(torch.device("cuda", 0), reps=7)
print(r["ms"])
"""
specs = sys.argv[1:]
res = {s: [] for s in specs}
for rnd in range(2):
    for spec in specs:
        lib, *gb = spec.split(":")
        env = dict(os.environ, GTAP_LIB=os.path.join(ROOT, "paper_2604_05982_b200", lib))
        if gb:
            env.update(SP_GRID=gb[0], SP_BLOCK=gb[1])
        out = subprocess.run([sys.executable, "-c", CHILD % ROOT], env=env, capture_output=True, text=True)
        try:
            res[spec].append(float(out.stdout.strip().splitlines()[-1]))
        except Exception:
            res[spec].append(float("nan"))
            print(spec, out.stderr[-500:])
for spec, v in res.items():
    print(f"{spec:55s} {statistics.median(v):.4f} ms  {[round(x, 4) for x in v]}")
