#!/bin/bash
# in-situ A/B of BFS build variants / geometries / hub splits on the bench configuration (RMAT-22, 16 sources):
# bench_tools/bfs_ab.sh lib[:grid:block[:split[:backoff[:steal_max]]]] ... (libs under paper_2604_05982_b200/)
cd "$(dirname "$0")/.."
for spec in "$@"; do
  IFS=: read lib grid block split bo sm <<< "$spec"
  GTAP_LIB=$PWD/paper_2604_05982_b200/$lib BFS_GRID=$grid BFS_BLOCK=$block BFS_SPLIT_ENV=$split BFS_BO=$bo BFS_SM=$sm timeout 600 python - <<PY
import os, sys
sys.path.insert(0, ".")
import torch, bench
if os.environ.get("BFS_GRID"):
    bench.BFS_CFG = dict(bench.BFS_CFG, grid_size=int(os.environ["BFS_GRID"]), block_size=int(os.environ["BFS_BLOCK"]))
if os.environ.get("BFS_BO"):
    bench.BFS_CFG = dict(bench.BFS_CFG, idle_backoff_ns=int(os.environ["BFS_BO"]))
if os.environ.get("BFS_SM"):
    bench.BFS_CFG = dict(bench.BFS_CFG, steal_max=int(os.environ["BFS_SM"]))
if os.environ.get("BFS_SPLIT_ENV"):
    bench.BFS_SPLIT = int(os.environ["BFS_SPLIT_ENV"])
dev = torch.device("cuda", 0)
r = bench.bench_bfs(dev, atom_min_peak=1.578e11)
print("$spec", "GTEPS %.3f" % r["value"], "ms %.3f" % r["ms"], "tasks/reached %.3f" % r["tasks_over_reached"], flush=True)
PY
done
