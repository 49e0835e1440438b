"""Scheduler invariants on the GPU (§4.3.2, SPEC S:120, S:217,
S:313-314), through the diagnostic GTAP_CHECK build of the C ABI (libgtap_gtap_check.so).

That build keeps, beside the workspace, one token per record for each of: allocated, published and
unclaimed, children of the current join epoch -- checked at every scheduler event (gtap.h
gtap_check_read). For every hot table, under schedule perturbations (one warp / one block, small and
large grids, steal seeds, steal batch sizes) the run must end with:

* every published (record, state) claimed and dispatched exactly once: publications == dispatches
  == invocations, no double publication, no dispatch of an unpublished task;
* no continuation dispatched before every child of its epoch joined; joins == non-root finished tasks;
* conservation: allocations == frees == tasks, no record still allocated, no task still published, no
  join count open; no-taskwait tables end with outstanding == 0;
* the exact oracle results (these are also the product tests' checks).

Two self-test builds inject a fault into the checker's own bookkeeping (a double publication; a lost
child join) and must fail with GTAP_E_INVARIANT and the matching violation counter: the checks can fire.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_PROBE = r"""
import json, sys
import numpy as np
import torch
sys.path.insert(0, %(root)r)
import oracle, synth
import paper_2604_05982_b200 as g
what = %(what)r
res = {}
WD = 60_000_000_000

def checked(name, kind, cfg, run, expect):
    with g.Runtime(kind, 0, watchdog_ns=WD, **cfg) as rt:
        out, st = run(rt)
        ck = rt.check_read()
    ok_res = expect(out, st)
    bad = {k: v for k, v in ck.items() if k.startswith("v_") and v}
    cons = (ck["allocs"] == ck["frees"] == st.tasks and ck["publications"] == ck["dispatches"] == st.invocations
            and ck["live_records"] == 0 and ck["published_unclaimed"] == 0 and ck["join_counts_open"] == 0)
    res[name] = dict(ok=bool(ok_res and not bad and cons), bad=bad, ck=ck, tasks=st.tasks, inv=st.invocations)
    return ck, st

T, B = g.GTAP_WORKER_THREAD, g.GTAP_WORKER_BLOCK
if "fib" in what:
    for n, cfg in ((0, dict(grid_size=1, block_size=32)), (2, dict(grid_size=148, block_size=128)),
                   (20, dict(grid_size=1, block_size=32, max_tasks_per_worker=4096)),
                   (20, dict(grid_size=148 * 4, block_size=128, steal_max=1, seed=7)),
                   (25, dict(grid_size=148 * 4, block_size=128, seed=99)),
                   (30, dict(grid_size=0, block_size=128, max_tasks_per_worker=4096))):
        ov, ot, oi = oracle.fib(n)
        def run(rt, n=n):
            t = g.Table.fib()
            rt.spawn_root(t, (n,)); rt.run(); st = rt.sync(); v = rt.root_result(0); t.close()
            return v, st
        ck, st = checked(f"fib{n}_{cfg.get('grid_size')}", T, cfg, run,
                         lambda v, st, ov=ov, ot=ot, oi=oi: (v, st.tasks, st.invocations) == (ov, ot, oi))
        # internal tasks suspend once; every non-root task joins its parent once
        res[f"fib{n}_{cfg.get('grid_size')}"]["ok"] &= ck["suspends"] == ck["continuations"] == (ot - 1) // 2 \
            and ck["joins"] == ot - 1
    # forest: 40 roots
    ns = [3 + (k %% 17) for k in range(40)]
    def runf(rt):
        t = g.Table.fib()
        for n in ns: rt.spawn_root(t, (n,))
        rt.run(); st = rt.sync(); v = [rt.root_result(i) for i in range(len(ns))]; t.close()
        return v, st
    checked("fib_forest", T, dict(grid_size=16, block_size=64, max_roots=64), runf,
            lambda v, st: v == [oracle.fib(n)[0] for n in ns])
if "epaq" in what:
    ov, ot, oi = oracle.fib(24)
    def rune(rt):
        t = g.Table.fib_cutoff(8, 3)
        rt.spawn_root(t, (24,)); rt.run(); st = rt.sync(); v = rt.root_result(0); t.close()
        return v, st
    checked("epaq", T, dict(grid_size=148, block_size=128, num_queues=3), rune, lambda v, st: v == ov)
if "ms" in what:
    for mm in (0, 1):
        for n, cfg in ((100003, dict(grid_size=148 * 4, block_size=128, max_tasks_per_worker=1024)),
                       (1 << 18, dict(grid_size=7, block_size=64, max_tasks_per_worker=4096, seed=3))):
            keys = synth.keys_int32(n, seed=n).numpy()
            d = torch.from_numpy(keys).cuda()
            ref, tasks, inv = oracle.mergesort(keys, 128)
            def runm(rt, d=d, mm=mm):
                s = torch.empty_like(d)
                t = g.Table.mergesort(d, s, 128, mm)
                rt.spawn_root(t, (0, d.numel())); rt.run(); st = rt.sync(); t.close()
                return None, st
            checked(f"ms{mm}_{n}", T, cfg, runm,
                    lambda _, st, d=d, ref=ref, tasks=tasks: bool(np.array_equal(d.cpu().numpy(), ref)) and st.tasks == tasks)
if "cs" in what:
    keys = synth.keys_int32(300007, seed=5).numpy()
    d = torch.from_numpy(keys).cuda()
    ref = oracle.cilksort(keys, 64, 256)
    def runc(rt):
        s = torch.empty_like(d)
        t = g.Table.cilksort(d, s, 64, 256)
        rt.spawn_root(t, (0, d.numel())); rt.run(); st = rt.sync(); t.close()
        return None, st
    checked("cilksort", T, dict(grid_size=148, block_size=128), runc,
            lambda _, st: bool(np.array_equal(d.cpu().numpy(), ref[0])) and st.tasks == ref[1])
if "nq" in what:
    c_ref = oracle.nqueens(10, 4)
    def runq(rt):
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        t = g.Table.nqueens(10, 4, cnt)
        rt.spawn_root(t, ()); rt.run(); st = rt.sync(); t.close()
        return int(cnt.item()), st
    ck, _ = checked("nqueens", T, dict(grid_size=148, block_size=128), runq,
                    lambda c, st: (c, st.tasks) == c_ref)
    res["nqueens"]["ok"] &= ck["outstanding"] == 0 and ck["suspends"] == 0
if "tree" in what:
    buf_cpu = synth.tree_buffer(1 << 14)
    buf = buf_cpu.to("cuda")
    for kind, kname, cfg in ((T, "thread", dict(grid_size=148, block_size=128)), (B, "block", dict(grid_size=148 * 4, block_size=64)),
                             (B, "block1", dict(grid_size=1, block_size=32))):
        for pruned, D in ((False, 10), (True, 12)):
            ref = oracle.tree(D, buf_cpu.numpy().view(np.uint64), 4, 8, pruned=pruned)
            def runt(rt, D=D, pruned=pruned, kind=kind):
                return g.tree(D, buf, 4, 8, pruned=pruned, worker=kind, rt=rt)
            checked(f"tree_{kname}_{int(pruned)}", kind, cfg, runt, lambda v, st, ref=ref: (v, st.tasks) == ref)
if "bfs" in what:
    rp, col = synth.rmat_csr(14, 16, seed=4)
    src = synth.bfs_sources(rp, 1, seed=4)[0]
    lv = oracle.bfs(rp, col, src)
    for cfg, kw in ((dict(grid_size=148, block_size=64, max_tasks_per_worker=1 << 16, steal_max=32), {}),
                    (dict(grid_size=148 * 4, block_size=64, max_tasks_per_worker=1 << 16), {}),
                    (dict(grid_size=1, block_size=32, max_tasks_per_worker=1 << 18), {}),
                    # the bench's shape: one-warp blocks (multi-task cycles), oldest-first pops, hub pieces
                    (dict(grid_size=148 * 8, block_size=32, max_tasks_per_worker=1 << 15, steal_max=32),
                     dict(order=1, edge_split=64))):
        def runb(rt, kw=kw):
            return g.bfs(rp.cuda(), col.cuda(), src, rt=rt, **kw)
        name = f"bfs_{cfg['grid_size']}_{cfg.get('steal_max', 1)}"
        ck, st = checked(name, B, cfg, runb, lambda depth, st: bool(np.array_equal(depth.cpu().numpy(), lv)))
        res[name]["ok"] &= ck["outstanding"] == 0
if "spmv" in what:
    rp, col, val, x = synth.powerlaw_csr(1 << 13, seed=2)
    y64, _ = oracle.spmv(rp, col, val, x)
    for parts in (0, 37):
        def runs(rt, parts=parts):
            return g.spmv(rp.cuda(), col.cuda(), val.cuda(), x.cuda(), None, 512, 4, parts=parts, rt=rt)
        def exps(y, st):
            e = np.abs(y.cpu().numpy().astype(np.float64) - y64) / np.maximum(np.abs(y64), 1e-30)
            return bool(np.all((y64 == 0) | (e <= 1e-5)))
        ck, _ = checked(f"spmv_{parts}", B, dict(grid_size=148, block_size=128, max_roots=64), runs, exps)
        res[f"spmv_{parts}"]["ok"] &= ck["outstanding"] == 0
if "selftest" in what:
    try:
        with g.Runtime(T, 0, grid_size=148, block_size=128, watchdog_ns=WD) as rt:
            t = g.Table.fib()
            rt.spawn_root(t, (15,)); rt.run()
            try:
                rt.sync(); code = 0
            except g.GtapError as e:
                code = e.code
            ck = rt.check_read(); t.close()
        res["selftest"] = dict(code=code, ck=ck)
    except Exception as e:
        res["selftest"] = dict(error=repr(e))
print(json.dumps(res))
"""


def _variant(defines):
    sys.path.insert(0, ROOT)
    from paper_2604_05982_b200 import build as b
    return b.build(defines=defines)


def _probe(lib, what):
    env = dict(os.environ, GTAP_LIB=lib)
    r = subprocess.run([sys.executable, "-c", _PROBE % {"root": ROOT, "what": what}], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("what", ["fib", "epaq", "ms", "cs", "nq", "tree", "bfs", "spmv"])
def test_scheduler_invariants(cuda_device, what):
    res = _probe(_variant(("GTAP_CHECK",)), what)
    assert res, res
    bad = {k: v for k, v in res.items() if not v["ok"]}
    assert not bad, bad


@pytest.mark.parametrize("mode,counter", [(1, "v_double_publish"), (2, "v_early_resume")])
def test_checker_detects_injected_faults(cuda_device, mode, counter):
    res = _probe(_variant(("GTAP_CHECK", f"GTAP_CHECK_SELFTEST={mode}")), "selftest")["selftest"]
    assert "error" not in res, res
    assert res["code"] == 12 and res["ck"][counter] >= 1, res  # GTAP_E_INVARIANT


def test_product_build_has_no_check(cuda_device):
    import paper_2604_05982_b200 as g
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=4, block_size=32) as rt:
        g.fib(5, rt=rt)
        with pytest.raises(g.GtapError) as e:
            rt.check_read()
        assert e.value.code == 11  # GTAP_E_UNSUPPORTED
