"""GPU parity of the build options that are off (or sized) by default in the product library.

Each variant library is compiled here (paper_2604_05982_b200/build.py with -D defines, the same
nvcc sm_100a flags) and exercised in a subprocess with GTAP_LIB pointing at it, against the
oracle: the options are alternative implementations of the same task bodies / scheduler paths
(DESIGN.md §5 "Measured and rejected", the own free stack), so every result must stay bit-exact.

* GTAP_FSTACK=1, GTAP_FIB_FSTACK=1: a one-entry own free stack, so nearly every surplus free takes
  the overflow path to the home free ring (fib, trees, Cilksort, N-Queens).
* GTAP_MS_VT=15, GTAP_MS_C=256, GTAP_MS_NS=4, GTAP_MS_BITONIC_MAX=1024: the bulk-copy merge core with 480-key tiles
  fed by 1 KB chunks x 4 (default: 416-key tiles, 2 KB chunks x 2) and bitonic merges up to 1024 keys (default 512).
* GTAP_CS_KARY=0: Cilksort's plain binary split search.
* GTAP_BFS_POP_BATCH=0 / 32: single pops and the largest batch pop of the block-level leader;
  GTAP_BFS_SKIP_STALE=1: a task whose vertex improved since its spawn returns at once (measured slower);
  GTAP_BFS_TTAS=0: every scanned edge issues its atomicMin (the default reads depth[u] first).
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# runs in the subprocess: prints one JSON object of checks
_PROBE = r"""
import json, sys
import numpy as np
import torch
sys.path.insert(0, %(root)r)
import oracle, synth
import paper_2604_05982_b200 as g
res = {}
what = %(what)r
cfg = dict(grid_size=148, block_size=128, max_tasks_per_worker=4096, watchdog_ns=60_000_000_000)
if "fib" in what:
    for n in (0, 1, 2, 20, 25):
        v, st = g.fib(n, **cfg)
        ov, ot, oi = oracle.fib(n)
        res[f"fib{n}"] = (v, st.tasks, st.invocations) == (ov, ot, oi)
if "tree" in what:
    buf_cpu = synth.tree_buffer(1 << 14)
    buf = buf_cpu.to("cuda")
    for pruned, D in ((False, 12), (True, 14)):
        v, st = g.tree(D, buf, 4, 8, pruned=pruned, **cfg)
        res[f"tree{int(pruned)}"] = (v, st.tasks) == oracle.tree(D, buf_cpu.numpy().view(np.uint64), 4, 8, pruned=pruned)
if "nq" in what:
    c, st = g.nqueens(10, 4, **cfg)
    res["nq10"] = (int(c), st.tasks) == oracle.nqueens(10, 4)
for name, n in (("ms", 1 << 18), ("ms_ragged", 100003), ("ms_big", 1 << 22), ("ms_4k", 300008)):
    if "ms" not in what:
        break
    keys = synth.keys_int32(n, seed=n).numpy()
    d = torch.from_numpy(keys).cuda()
    st = g.mergesort_(d, cutoff=128, merge_mode=1, grid_size=148 * 4, block_size=128, max_tasks_per_worker=1024,
                      watchdog_ns=60_000_000_000)
    ref, tasks, inv = oracle.mergesort(keys, 128)
    res[name] = bool(np.array_equal(d.cpu().numpy(), ref)) and st.tasks == tasks
if "bfs" in what:
    rp, col = synth.rmat_csr(14, 16, seed=4)
    src = synth.bfs_sources(rp, 1, seed=4)[0]
    for grid, block, split in ((148, 64, 0), (1, 32, 0), (148 * 4, 32, 64)):
        for order in (0, 1):
            depth, st = g.bfs(rp.cuda(), col.cuda(), src, grid_size=grid, block_size=block,
                              max_tasks_per_worker=1 << 16, steal_max=32, watchdog_ns=60_000_000_000, order=order,
                              edge_split=split)
            res[f"bfs{grid}_{block}_{order}"] = bool(np.array_equal(depth.cpu().numpy(), oracle.bfs(rp, col, src)))
if "cs" in what:
    keys = synth.keys_int32(300007, seed=5).numpy()
    d = torch.from_numpy(keys).cuda()
    st = g.cilksort_(d, None, 64, 256, **cfg)
    ref = oracle.cilksort(keys, 64, 256)
    res["cs"] = bool(np.array_equal(d.cpu().numpy(), ref[0])) and st.tasks == ref[1]
print(json.dumps(res))
"""


def _variant(defines):
    sys.path.insert(0, ROOT)
    from paper_2604_05982_b200 import build as b
    return b.build(defines=defines)


def _probe(lib, what):
    env = dict(os.environ, GTAP_LIB=lib)
    code = _PROBE % {"root": ROOT, "what": what}
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("defines,what", [
    (("GTAP_FSTACK=1", "GTAP_FIB_FSTACK=1"), "fib tree nq cs"),
    (("GTAP_MS_VT=15", "GTAP_MS_C=256", "GTAP_MS_NS=4", "GTAP_MS_BITONIC_MAX=1024"), "ms"),
    (("GTAP_CS_KARY=0",), "cs"),
    (("GTAP_BFS_POP_BATCH=0",), "bfs"),
    (("GTAP_BFS_POP_BATCH=32",), "bfs"),
    (("GTAP_BFS_SKIP_STALE=1",), "bfs"),
    (("GTAP_BFS_TTAS=0",), "bfs"),
], ids=["fstack1", "ms_vt15_c256_bitonic1024", "cs_binary_split", "bfs_pop1",
        "bfs_pop32", "bfs_skip_stale", "bfs_atomic_always"])
def test_variant_parity(cuda_device, defines, what):
    lib = _variant(defines)
    res = _probe(lib, what)
    assert res and all(res.values()), res
