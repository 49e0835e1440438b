"""GPU parity: Cilksort task table vs the oracle.

Bit-exact output and exact task / invocation counts (the split rule is deterministic), across
sizes, cutoffs (including ones that split every merge), adversarial inputs, and the bench size,
in both merge modes (thread: the paper's one-lane leaf sorts / merges; warp: bitonic networks run by
the task's warp; cut_merge > 1024 exercises the warp mode's lane-0 fallback).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
WD = 60_000_000_000


@pytest.fixture(scope="module")
def g(cuda_device):
    import paper_2604_05982_b200 as g
    return g


@pytest.fixture(scope="module", params=[0, 1], ids=["thread_merge", "warp_merge"])
def mode(request):
    return request.param


@pytest.fixture(scope="module")
def rt(g):
    r = g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148 * 2, block_size=128, max_tasks_per_worker=4096,
                  watchdog_ns=WD)
    yield r
    r.close()


def run(g, rt, keys_np, cuts=(64, 256), mode=1):
    import torch
    d = torch.from_numpy(keys_np).cuda()
    st = g.cilksort_(d, None, *cuts, merge_mode=mode, rt=rt)
    return d.cpu().numpy(), st


@pytest.mark.parametrize("n", [0, 1, 63, 64, 65, 1000, 4099, (1 << 16) + 3, 1 << 20])
@pytest.mark.parametrize("cuts", [(64, 256), (4, 8), (256, 2048)])
def test_sizes(g, rt, mode, n, cuts):
    keys = synth.keys_int32(n, seed=n).numpy()
    out, st = run(g, rt, keys, cuts, mode)
    ref, tasks, inv = oracle.cilksort(keys, *cuts)
    assert np.array_equal(out, ref)
    assert (st.tasks, st.invocations) == (tasks, inv)


@pytest.mark.parametrize("kind", ["sorted", "reverse", "equal", "two"])
def test_adversarial(g, rt, mode, kind):
    n = 50001
    rng = np.random.default_rng(5)
    a = {"sorted": np.arange(n), "reverse": np.arange(n, 0, -1), "equal": np.full(n, 9),
         "two": rng.integers(0, 2, n)}[kind].astype(np.int32)
    out, st = run(g, rt, a, (64, 256), mode)
    ref, tasks, inv = oracle.cilksort(a, 64, 256)
    assert np.array_equal(out, ref) and (st.tasks, st.invocations) == (tasks, inv)


def test_full_size(g, mode):
    import bench
    n = 1 << 24
    keys = synth.keys_int32(n, seed=42)
    d = keys.cuda()
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, watchdog_ns=WD, **bench.CS_CFG) as r:
        st = g.cilksort_(d, None, 64, 256, merge_mode=mode, rt=r)
    ref, tasks, inv = oracle.cilksort(keys.numpy(), 64, 256)
    assert np.array_equal(d.cpu().numpy(), ref)
    assert (st.tasks, st.invocations) == (tasks, inv)
