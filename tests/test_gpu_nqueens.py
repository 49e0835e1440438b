"""GPU parity: N-Queens task table vs the oracle (exact counts)."""
import pytest

import oracle

pytestmark = pytest.mark.gpu
WD = 60_000_000_000


@pytest.fixture(scope="module")
def g(cuda_device):
    import paper_2604_05982_b200 as g
    return g


@pytest.fixture(scope="module", params=[0, 1], ids=["lane_leaf", "warp_leaf"])
def mode(request):
    return request.param


@pytest.fixture(scope="module")
def rt(g):
    r = g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148 * 4, block_size=128, max_tasks_per_worker=4096,
                  watchdog_ns=WD)
    yield r
    r.close()


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 8, 10, 12])
@pytest.mark.parametrize("cutoff", [0, 1, 3, 7])
def test_counts_and_tasks(g, rt, mode, n, cutoff):
    sol, st = g.nqueens(n, cutoff, leaf_mode=mode, rt=rt)
    osol, otasks = oracle.nqueens(n, cutoff)
    assert sol == osol
    assert st.tasks == otasks and st.invocations == otasks  # no taskwait: one invocation per task


@pytest.mark.parametrize("grid,block", [(1, 32), (13, 64), (148 * 4, 128)])
def test_geometry(g, mode, grid, block):
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=grid, block_size=block, max_tasks_per_worker=8192,
                   watchdog_ns=WD) as r:
        sol, st = g.nqueens(11, 5, leaf_mode=mode, rt=r)
        assert (sol, st.tasks) == oracle.nqueens(11, 5)


def test_n16_cutoff7(g, mode):
    """The paper's headline size: n = 16, cutoff depth 7."""
    import bench
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, watchdog_ns=WD, **bench.NQ_CFG) as r:
        sol, st = g.nqueens(16, 7, leaf_mode=mode, rt=r)
    assert sol == 14772512


def test_grid_beyond_coresidency_rejected(g):
    # a persistent grid that cannot be co-resident is refused instead of deadlocking (A3)
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148 * 64, block_size=128, max_tasks_per_worker=64) as r:
        with pytest.raises(g.GtapError):
            g.nqueens(8, 3, rt=r)
