"""fib(40) launch sweep for the library in GTAP_LIB (grid 0 = occupancy-derived)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_05982_b200 as g  # noqa: E402

lib = os.path.basename(os.environ.get("GTAP_LIB", "libgtap.so"))
for grid, block in [(0, 128), (0, 256), (0, 64)]:
    try:
        with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=grid, block_size=block, max_tasks_per_worker=4096) as rt:
            res = [g.fib(40, rt=rt)[1] for _ in range(4)]
        st = res[-1]
        ms = statistics.median(r.device_ms for r in res[1:])
        print(f"{lib:32s} grid={st.grid_size} block={block} warps={st.workers} ms={ms:.2f} "
              f"Gtasks/s={st.tasks / ms / 1e6:.2f} steals={st.steals_ok} cycles={st.cycles} idle={st.idle_cycles}",
              flush=True)
    except Exception as e:
        print(lib, grid, block, "ERR", e, flush=True)
