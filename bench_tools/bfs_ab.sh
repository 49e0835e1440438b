#!/bin/bash
# in-situ A/B of BFS build variants / geometries on the bench configuration (RMAT-22, 16 sources):
# bench_tools/bfs_ab.sh lib[:grid:block] ... (libs under paper_2604_05982_b200/)
cd "$(dirname "$0")/.."
for spec in "$@"; do
  IFS=: read lib grid block <<< "$spec"
  GTAP_LIB=$PWD/paper_2604_05982_b200/$lib BFS_GRID=$grid BFS_BLOCK=$block timeout 600 python - <<PY
import os, sys
sys.path.insert(0, ".")
import torch, bench
if os.environ.get("BFS_GRID"):
    bench.BFS_CFG = dict(bench.BFS_CFG, grid_size=int(os.environ["BFS_GRID"]), block_size=int(os.environ["BFS_BLOCK"]))
dev = torch.device("cuda", 0)
r = bench.bench_bfs(dev, atom_min_peak=1.578e11)
print("$spec", "GTEPS %.3f" % r["value"], "ms %.3f" % r["ms"], "tasks/reached %.3f" % r["tasks_over_reached"], "frac %.3f" % r["roofline"]["frac"])
PY
done
