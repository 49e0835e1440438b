"""BFS launch-configuration sweep (library from GTAP_LIB): RMAT scale (argv[1], default 22), 2 sources."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
rp, col = synth.rmat_csr(scale, 16, seed=3, device="cuda")
srcs = synth.bfs_sources(rp, 2, seed=5)
ref = {}
lib = os.path.basename(os.environ.get("GTAP_LIB", "libgtap.so"))
SM = int(os.environ.get("STEAL_MAX", "32"))
for grid, block, backoff in ((148 * 4, 256, 1024), (148 * 8, 128, 1024), (148 * 16, 64, 1024), (148 * 16, 64, 256),
                             (148 * 32, 32, 1024), (148 * 32, 32, 256), (148 * 24, 32, 512)):
    try:
        rt = g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=grid, block_size=block, max_tasks_per_worker=1 << 18,
                       idle_backoff_ns=backoff, steal_max=SM, watchdog_ns=60_000_000_000)
        out = []
        for s in srcs:
            ms = []
            for it in range(3):
                d, st = g.bfs(rp, col, s, rt=rt)
                ms.append(st.device_ms)
            if s not in ref:
                ref[s] = d.clone()
            assert torch.equal(d, ref[s])
            out.append((min(ms), st.tasks))
        rt.close()
        edges = col.numel()
        print(f"{lib:20s} steal_max={SM} grid={grid:5d} block={block:4d} backoff={backoff:5d} " +
              " ".join(f"{m:8.2f} ms ({edges / m / 1e6:5.2f} GTEPS, tasks {t})" for m, t in out), flush=True)
    except Exception as e:
        print(f"{lib} grid={grid} block={block}: {e}", flush=True)
