import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_05982_b200 as g
for grid, block in [(148*2,128),(148*4,128),(148*6,128),(148*8,128),(148*16,64),(148*4,256),(148*32,32)]:
    try:
        with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=grid, block_size=block, max_tasks_per_worker=4096) as rt:
            res = [g.fib(40, rt=rt)[1] for _ in range(3)]
        st = res[-1]
        print(f"grid={grid} block={block} warps={st.workers} ms={statistics.median(r.device_ms for r in res):.2f} "
              f"maxpool={st.max_pool_used} steals={st.steals_ok} cycles={st.cycles} idle={st.idle_cycles} "
              f"kept={st.kept} pops={st.pops} pushes={st.pushes}", flush=True)
    except Exception as e:
        print(grid, block, "ERR", e, flush=True)
