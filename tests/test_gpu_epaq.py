"""GPU parity: fib with cutoff, with and without EPAQ.

EPAQ is semantics-free: the value, task count and invocation count must equal the
oracle's for 1 and for 3 queues, across cutoffs and geometries.
"""
import pytest

import oracle

pytestmark = pytest.mark.gpu
WD = 30_000_000_000


@pytest.fixture(scope="module")
def g(cuda_device):
    import paper_2604_05982_b200 as g
    return g


@pytest.fixture(scope="module")
def rt3(g):
    r = g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148 * 4, block_size=128, max_tasks_per_worker=4096,
                  num_queues=3, watchdog_ns=WD)
    yield r
    r.close()


@pytest.mark.parametrize("nq", [1, 3])
@pytest.mark.parametrize("cutoff", [0, 2, 5, 10])
@pytest.mark.parametrize("n", [0, 1, 2, 9, 10, 11, 20, 27])
def test_fib_cutoff_parity(g, rt3, nq, cutoff, n):
    v, st = g.fib_cutoff(n, cutoff, nq, rt=rt3)
    ov, tasks, inv, _ = oracle.fib_cutoff(n, cutoff)
    assert (v, st.tasks, st.invocations) == (ov, tasks, inv)


def test_epaq_queue_count_enforced(g):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148, block_size=128, max_tasks_per_worker=1024,
                   num_queues=1, watchdog_ns=WD) as r:
        with pytest.raises(g.GtapError):
            g.fib_cutoff(10, 5, 3, rt=r)


@pytest.mark.parametrize("grid,block", [(1, 32), (7, 64), (148 * 8, 128)])
def test_epaq_geometry(g, grid, block):
    # one warp holds the whole tree's live records: EPAQ changes the traversal order and footprint
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=grid, block_size=block,
                   max_tasks_per_worker=1 << 15 if grid * block <= 32 else 4096, num_queues=3, watchdog_ns=WD) as r:
        for nq in (1, 3):
            v, st = g.fib_cutoff(24, 6, nq, rt=r)
            assert (v, st.tasks, st.invocations) == oracle.fib_cutoff(24, 6)[:3]


def test_fib40_cutoff10_epaq(g):
    """The paper's EPAQ profile point: fib(40), cutoff 10, 3 queues vs 1."""
    import bench
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, num_queues=3, watchdog_ns=60_000_000_000, **bench.FIB_CFG) as r:
        ref = oracle.fib_cutoff(40, 10)[:3]
        for nq in (1, 3):
            v, st = g.fib_cutoff(40, 10, nq, rt=r)
            assert (v, st.tasks, st.invocations) == ref


@pytest.mark.parametrize("cutoff", [0, 5, 10])
@pytest.mark.parametrize("n", [2, 11, 20, 27])
def test_queue_policy_stay_parity(g, cutoff, n):
    """queue_policy 1 (stay on the class in use while it has runnable tasks, P:177-178 literal) is
    semantics-free too."""
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148 * 4, block_size=128, max_tasks_per_worker=4096,
                   num_queues=3, queue_policy=1, watchdog_ns=WD) as r:
        v, st = g.fib_cutoff(n, cutoff, 3, rt=r)
    ov, tasks, inv, _ = oracle.fib_cutoff(n, cutoff)
    assert (v, st.tasks, st.invocations) == (ov, tasks, inv)


def test_queue_policy_range(g):
    with pytest.raises(g.GtapError):
        g.Runtime(g.GTAP_WORKER_THREAD, 0, num_queues=3, queue_policy=2)
