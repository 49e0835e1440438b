"""SpMV sweep: launch geometry x split cutoff x forest size (parts = 0: one root)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

rp, col, val, x = synth.powerlaw_csr(1 << 22, seed=7, device="cuda")
y = torch.empty(1 << 22, dtype=torch.float32, device="cuda")
nnz = int(rp[-1])
algo = 8.0 * nnz + 12.0 * (1 << 22)
ref = None
CFGS = {'libgtap.so': [(148 * 8, 128)], 'libgtap_gtap_spmv_per16.so': [(148 * 8, 128)], 'libgtap_gtap_spmv_per12.so': [(148 * 8, 128)],
        'libgtap_gtap_spmv_per16_gtap_spmv_minb3.so': [(148 * 6, 128), (148 * 3, 256)]}
FULL = os.environ.get('SWEEP_FULL') == '1'
GEOMS = [(int(os.environ['GRID']), 128)] if os.environ.get('GRID') else [(148 * 8, 128), (148 * 4, 256), (148 * 16, 64)] if FULL else CFGS.get(os.path.basename(os.environ.get('GTAP_LIB', 'libgtap.so')), [(148 * 8, 128)])
for grid, block in GEOMS:
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=grid, block_size=block, max_tasks_per_worker=2048,
                   max_roots=4 * grid) as rt:
        for parts in ((grid, 2 * grid) if FULL else (grid,)):
            for cut in ((8192, 65536, 262144) if FULL else (8192, 65536)):
                sts = []
                for _ in range(4):
                    y.zero_()
                    sts.append(g.spmv(rp, col, val, x, y, cut, 32, parts=parts, rt=rt)[1])
                if ref is None:
                    ref = y.clone()
                err = float(((y - ref).abs() / ref.abs().clamp_min(1e-30)).max())
                t = statistics.median(s.device_ms for s in sts[1:])
                print(f"{os.path.basename(os.environ.get('GTAP_LIB', 'libgtap.so'))[7:]:30s} grid={grid} block={block} parts={parts:5d} cut={cut:6d} ms={t:.3f} GB/s={algo / t / 1e6:.0f} "
                      f"tasks={sts[-1].tasks} maxrel={err:.1e}", flush=True)
