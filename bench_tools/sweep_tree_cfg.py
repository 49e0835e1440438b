"""Launch-configuration sweep for the synthetic tree (grid x block per worker kind)."""
import sys

sys.path.insert(0, ".")
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

buf = synth.tree_buffer(1 << 25, device="cuda")
POINTS = [("full", 22, 64, 256), ("pruned", 24, 64, 32768), ("pruned", 24, 2048, 256), ("full", 18, 0, 256)]
for kind, cfgs in ((g.GTAP_WORKER_BLOCK, [(148 * 8, 64), (148 * 16, 64), (148 * 32, 32), (148 * 16, 32),
                                          (148 * 8, 128), (148 * 4, 256)]),
                   (g.GTAP_WORKER_THREAD, [(0, 128), (0, 64), (0, 256), (148 * 2, 128)])):
    for grid, block in cfgs:
        try:
            rt = g.Runtime(kind, 0, grid_size=grid, block_size=block, max_tasks_per_worker=2048 if kind == g.GTAP_WORKER_BLOCK else 4096,
                           watchdog_ns=60_000_000_000)
        except Exception as e:  # co-residency
            print(kind, grid, block, "skip", e)
            continue
        for shape, D, mem, comp in POINTS:
            sts = [g.tree(D, buf, mem, comp, pruned=shape == "pruned", worker=kind, rt=rt)[1] for _ in range(3)]
            ms = min(s.device_ms for s in sts)
            print(f"{'thread' if kind == g.GTAP_WORKER_THREAD else 'block'} grid={sts[0].grid_size} "
                  f"block={block} {shape} D={D} mem={mem} comp={comp}: {ms:.3f} ms", flush=True)
        rt.close()
