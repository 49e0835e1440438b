"""GPU tests of the runtime contract of include/gtap.h (not of a task table's arithmetic).

* roots outside the table's array are rejected at gtap_spawn_root (mergesort, Cilksort);
* a failed gtap_run drops the staged roots and the table binding, so the next run with another
  table works and never sees the stale roots;
* gtap_reset on one stream followed by gtap_run on another is ordered by the runtime;
* config.max_child_tasks (GTAP_MAX_CHILD_TASKS) is enforced at run time.
"""
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
WD = 20_000_000_000


@pytest.fixture(scope="module")
def g(cuda_device):
    import paper_2604_05982_b200 as g
    return g


def test_sort_roots_bounded_by_n(g):
    import torch
    keys = torch.zeros(1000, dtype=torch.int32, device="cuda")
    scratch = torch.zeros_like(keys)
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148, block_size=128, max_tasks_per_worker=1024,
                   watchdog_ns=WD) as r:
        for mk in (lambda: g.Table.mergesort(keys, scratch, 128, 1), lambda: g.Table.mergesort(keys, scratch, 128, 0),
                   lambda: g.Table.cilksort(keys, scratch, 64, 256)):
            t = mk()
            for bad in ((0, 1001), (500, 1 << 20), (3, 2)):
                with pytest.raises(g.GtapError) as e:
                    r.spawn_root(t, bad)
                assert e.value.code == 1
            r.spawn_root(t, (0, 1000))   # the whole array is fine
            r.spawn_root(t, (1000, 1000))
            r.reset()
            t.close()
    with pytest.raises(ValueError):
        g.Table.cilksort(keys, scratch[:999].contiguous())


def test_failed_run_drops_roots_and_table(g):
    # block 1024 exceeds the fib kernel's launch bounds: gtap_run fails with GTAP_E_INVAL
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=8, block_size=1024, max_tasks_per_worker=1024,
                   watchdog_ns=WD) as r:
        t1 = g.Table.fib()
        r.spawn_root(t1, (10,))
        with pytest.raises(g.GtapError) as e:
            r.run()
        assert e.value.code == 1
        t1.close()
        # the roots were dropped with the failure: a run now has nothing to launch
        with pytest.raises(g.GtapError):
            r.run()
        # and another table may be staged (the old binding is gone)
        t2 = g.Table.fib_cutoff(5, 1)
        r.spawn_root(t2, (12,))
        r.reset()
        t2.close()


def test_reset_and_run_on_different_streams(g):
    import torch
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148, block_size=128, max_tasks_per_worker=4096,
                   watchdog_ns=WD) as r:
        t = g.Table.fib()
        for n in (22, 23, 21, 24):
            # a long kernel on s1 delays the reset's fills; the run on s2 must still wait for them
            x = torch.randn(2048, 2048, device="cuda")
            with torch.cuda.stream(s1):
                for _ in range(8):
                    x = x @ x
                    x = x / x.abs().max()
            r.reset(s1)
            r.spawn_root(t, (n,))
            r.run(s2)
            st = r.sync()
            assert (r.root_result(0), st.tasks, st.invocations) == oracle.fib(n)
        t.close()


def test_max_child_tasks_enforced(g):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148, block_size=128, max_tasks_per_worker=1024,
                   max_child_tasks=1, watchdog_ns=WD) as r:
        with pytest.raises(g.GtapError) as e:
            g.fib(10, rt=r)
        assert e.value.code == 7   # GTAP_E_CHILD_LIMIT
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148, block_size=128, max_tasks_per_worker=1024,
                   max_child_tasks=2, watchdog_ns=WD) as r:
        v, st = g.fib(15, rt=r)
        assert (v, st.tasks, st.invocations) == oracle.fib(15)
    # block-level: SpMV splits into `fanout` children
    import torch
    rp, col, val, x = synth.powerlaw_csr(1 << 12, seed=2)
    dev = torch.device("cuda")
    with g.Runtime(g.GTAP_WORKER_BLOCK, 0, grid_size=148, block_size=256, max_tasks_per_worker=1024,
                   max_child_tasks=3, watchdog_ns=WD) as r:
        with pytest.raises(g.GtapError) as e:
            g.spmv(rp.to(dev), col.to(dev), val.to(dev), x.to(dev), nnz_cut=256, fanout=4, rt=r)
        assert e.value.code == 7


def test_die_probe_map(cuda_device):
    """gtap_ubench_die_probe: every SM gets a die label, both dies are populated, far latency > near."""
    import torch

    import paper_2604_05982_b200 as g
    from paper_2604_05982_b200 import gtap
    buf = torch.zeros(128 * 2048 // 4, dtype=torch.int32, device="cuda")
    r = gtap.ubench_die_probe(buf, 128)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    die = r["sm_die"][:nsm]
    assert set(die.tolist()) <= {0, 1} and 0 < int(die.sum()) < nsm
    assert r["far_cycles"] > r["near_cycles"] > 0
    with pytest.raises(g.GtapError):
        g.Runtime(g.GTAP_WORKER_THREAD, 0, victim_policy=2)
