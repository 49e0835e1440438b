cd /root/repo
for mt in 131072 65536 32768; do BFS_MT=$mt timeout 600 python - <<PY
import os, sys
sys.path.insert(0, ".")
import torch, bench
bench.BFS_CFG = dict(bench.BFS_CFG, max_tasks_per_worker=int(os.environ["BFS_MT"]))
r = bench.bench_bfs(torch.device("cuda", 0), atom_min_peak=1.55e11)
print("max_tasks", os.environ["BFS_MT"], "GTEPS %.3f" % r["value"], "ms %.3f" % r["ms"], flush=True)
PY
done
