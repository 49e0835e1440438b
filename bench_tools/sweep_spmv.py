import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2604_05982_b200 as g
rp, col, val, x = synth.powerlaw_csr(1 << 22, seed=7, device="cuda")
y = torch.empty(1 << 22, dtype=torch.float32, device="cuda")
nnz = int(rp[-1]); algo = 8.0 * nnz + 12.0 * (1 << 22)
for grid, block in [(148*4, 256), (148*8, 128), (148*2, 512)]:
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=grid, block_size=block, max_tasks_per_worker=2048) as rt:
        for cut in (8192, 32768, 131072):
            for fan in (16, 32):
                ms = [g.spmv(rp, col, val, x, y, cut, fan, rt=rt)[1] for _ in range(4)]
                t = statistics.median(s.device_ms for s in ms[1:])
                print(f"grid={grid} block={block} cut={cut} fan={fan} ms={t:.3f} GB/s={algo/t/1e6:.0f} tasks={ms[-1].tasks}", flush=True)
