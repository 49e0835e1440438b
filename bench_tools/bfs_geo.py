import sys, os, torch
sys.path.insert(0, "/root/repo")
import paper_2604_05982_b200 as g, synth
rp, col = synth.rmat_csr(22, 16, seed=3, device="cuda")
srcs = synth.bfs_sources(rp, 2, seed=5)
for grid, block, mt in ((148*16, 64, 1<<18), (148*32, 32, 1<<16), (148*24, 32, 1<<16), (148*32, 32, 1<<17), (148*16, 32, 1<<17)):
    try:
        rt = g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=grid, block_size=block, max_tasks_per_worker=mt, idle_backoff_ns=1024, steal_max=32, watchdog_ns=60_000_000_000)
        res = []
        for s in srcs:
            ms = []
            for it in range(3):
                d, st = g.bfs(rp, col, s, rt=rt); ms.append(st.device_ms)
            res.append((min(ms), st.tasks))
        rt.close()
        print(grid, block, mt, res, flush=True)
    except Exception as e:
        print(grid, block, mt, "ERR", e, flush=True)
