"""GPU parity: fib task table vs the oracle (bit-exact value, exact task and invocation counts).

PAPER.md P:1023-1033 / P:1160-1190. Sizes: fib(0..25) (several tiles of 32-lane
warps + ragged tails), fib(40) at BASELINE configs[2]'s full size, schedule
perturbations (grid, block, seeds, steal size, pool/queue capacities), a forest,
and the failure modes (pool exhaustion, bad root) that must not hang.
"""
import pytest

import oracle

pytestmark = pytest.mark.gpu
WD = 20_000_000_000  # 20 s watchdog: a scheduler bug fails the test instead of hanging the GPU


@pytest.fixture(scope="module")
def g(cuda_device):
    import paper_2604_05982_b200 as g
    return g


@pytest.fixture(scope="module")
def rt(g):
    # a 32-lane warp holds up to ~64 live records per tree level (32 suspended + 32 pushed)
    r = g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148 * 4, block_size=128, max_tasks_per_worker=4096,
                  watchdog_ns=WD)
    yield r
    r.close()


@pytest.mark.parametrize("n", list(range(0, 26)))
def test_fib_small(g, rt, n):
    v, st = g.fib(n, rt=rt)
    ov, tasks, inv = oracle.fib(n)
    assert v == ov
    assert st.tasks == tasks and st.invocations == inv
    assert st.error_word == 0


def test_fib20_config0(g, rt):
    v, st = g.fib(20, rt=rt)
    assert (v, st.tasks, st.invocations) == (6765, 21891, 32836)  # BASELINE configs[0]


@pytest.mark.parametrize("grid,block", [(1, 32), (1, 128), (2, 32), (7, 64), (148, 32), (148 * 7, 128), (0, 256)])
def test_fib_geometry(g, grid, block):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=grid, block_size=block, max_tasks_per_worker=2048,
                   watchdog_ns=WD) as r:
        v, st = g.fib(22, rt=r)
        ov, tasks, inv = oracle.fib(22)
        assert (v, st.tasks, st.invocations) == (ov, tasks, inv)


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("steal_max", [1, 7, 32])
def test_fib_schedule_perturbation(g, seed, steal_max):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148, block_size=64, max_tasks_per_worker=2048,
                   queue_capacity=1024, steal_max=steal_max, seed=seed, watchdog_ns=WD) as r:
        v, st = g.fib(24, rt=r)
        assert (v, st.tasks, st.invocations) == oracle.fib(24)


def test_fib_few_workers_wrap(g):
    # 4 warps stealing from each other for ~2.3e5 tasks: the steal end advances far past the
    # 1024-slot ring (wraparound) and records are recycled through the free rings many times
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=4, block_size=32, max_tasks_per_worker=2048,
                   queue_capacity=1024, watchdog_ns=WD) as r:
        v, st = g.fib(25, rt=r)
        assert (v, st.tasks, st.invocations) == oracle.fib(25)
        assert st.max_pool_used <= 2048 and st.tasks > 50 * 2048


def test_fib_repeated_runs_reuse(g, rt):
    for n in (15, 3, 21, 0, 21):
        v, st = g.fib(n, rt=rt)
        assert (v, st.tasks, st.invocations) == oracle.fib(n)


def test_fib_forest(g):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148, block_size=128, max_tasks_per_worker=4096,
                   max_roots=1000, watchdog_ns=WD) as r:
        t = g.Table.fib()
        ns = [(i * 7) % 23 for i in range(1000)]
        for n in ns:
            r.spawn_root(t, (n,))
        r.run()
        st = r.sync()
        for i, n in enumerate(ns):
            assert r.root_result(i) == oracle.fib(n)[0]
        assert st.tasks == sum(oracle.fib(n)[1] for n in ns)
        t.close()


def test_fib40_full(g):
    """BASELINE configs[2]: fib(40), ~3.3e8 tasks, at the bench's launch configuration."""
    import bench
    cfg = bench.FIB_CFG
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, watchdog_ns=60_000_000_000, **cfg) as r:
        v, st = g.fib(40, rt=r)
        assert (v, st.tasks, st.invocations) == (102334155, 331160281, 496740421)


def test_pool_exhaustion_is_an_error(g):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=1, block_size=32, max_tasks_per_worker=64,
                   queue_capacity=64, watchdog_ns=WD) as r:
        with pytest.raises(g.GtapError) as e:
            g.fib(25, rt=r)
        assert e.value.code in (5, 6)  # GTAP_E_POOL_EXHAUSTED / GTAP_E_QUEUE_OVERFLOW
        # the runtime stays usable after a failed run
        v, st = g.fib(5, rt=r)
        assert v == 5


def test_bad_root_rejected(g, rt):
    t = g.Table.fib()
    with pytest.raises(g.GtapError):
        rt.spawn_root(t, (47,))  # int32 overflow (reading R17)
    t.close()


@pytest.mark.parametrize("grid,block", [(148, 128), (0, 128), (3, 64)])
def test_fib_die_aware_victims(g, grid, block):
    """victim_policy 1 (gtap_init probes the SM -> L2-die map; thieves favour victims whose deque line is near
    their die): a scheduling choice only -- values and counts stay exact."""
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=grid, block_size=block, max_tasks_per_worker=4096,
                   victim_policy=1, watchdog_ns=WD) as r:
        for n in (5, 20, 27):
            v, st = g.fib(n, rt=r)
            assert (v, st.tasks, st.invocations) == oracle.fib(n)
