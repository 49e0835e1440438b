"""GPU parity: mergesort task table vs the oracle (bit-exact output, exact task counts).

PAPER.md P:59-74. Ragged sizes around the cutoff and the
32-lane tile, every cutoff the API allows at its edges, adversarial inputs,
forests, and BASELINE configs[1] (2^24 random int32) at the bench's launch
configuration. Every test runs in both merge modes: GTAP_MERGE_THREAD (the
paper's one-lane merge, TMA-staged for long runs) and GTAP_MERGE_WARP (heavy
merges run by the task's whole warp).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
WD = 30_000_000_000


@pytest.fixture(scope="module")
def g(cuda_device):
    import paper_2604_05982_b200 as g
    return g


@pytest.fixture(scope="module", params=[0, 1], ids=["thread_merge", "warp_merge"])
def mode(request):
    return request.param


@pytest.fixture(scope="module")
def rt(g):
    r = g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=148 * 2, block_size=128, max_tasks_per_worker=1024,
                  watchdog_ns=WD)
    yield r
    r.close()


def run_sort(g, rt, keys_np, cutoff=128, mode=1):
    import torch
    d = torch.from_numpy(keys_np).cuda()
    st = g.mergesort_(d, cutoff=cutoff, merge_mode=mode, rt=rt)
    return d.cpu().numpy(), st


# n % 4 == 0 and runs >= 8192 keys take the TMA-staged merge (ragged run ends -> partial chunks);
# other sizes exercise the register-window merge
@pytest.mark.parametrize("n", [0, 1, 2, 31, 127, 128, 129, 255, 256, 1000, 4097, (1 << 16) + 7, 1 << 20,
                               100004, 3 * (1 << 18) + 12, 40000])
def test_sizes(g, rt, mode, n):
    keys = synth.keys_int32(n, seed=n).numpy()
    out, st = run_sort(g, rt, keys, 128, mode)
    ref, tasks, inv = oracle.mergesort(keys, 128)
    assert np.array_equal(out, ref)
    assert (st.tasks, st.invocations) == (tasks, inv)
    if mode == 0:
        assert st.assists == 0
    else:  # every leaf and every merge ran as a warp assist
        merges, leaves = _shape(n, 128)
        assert st.assists == leaves + len(merges)


def _shape(n, cutoff):
    """(merge sizes, leaf count) of the cutoff mergesort recursion on n keys."""
    merges, leaves, stack = [], 0, [n]
    while stack:
        k = stack.pop()
        if k > cutoff:
            merges.append(k)
            stack += [k // 2, k - k // 2]
        else:
            leaves += 1
    return merges, leaves


@pytest.mark.parametrize("cutoff", [1, 2, 3, 64, 128, 255, 256])
def test_cutoffs(g, rt, mode, cutoff):
    keys = synth.keys_int32(20011, seed=cutoff).numpy()
    out, st = run_sort(g, rt, keys, cutoff, mode)
    ref, tasks, inv = oracle.mergesort(keys, cutoff)
    assert np.array_equal(out, ref)
    assert (st.tasks, st.invocations) == (tasks, inv)


@pytest.mark.parametrize("kind", ["sorted", "reverse", "equal", "two", "extremes"])
# 300007: block-assisted top merge (>= 2^17), chunk borders on ties; 300008 (n % 4 == 0): the same through the
# bulk-copy merge core
@pytest.mark.parametrize("n", [100003, 300007, 300008])
def test_adversarial(g, rt, mode, kind, n):
    rng = np.random.default_rng(7)
    a = {"sorted": np.arange(n), "reverse": np.arange(n, 0, -1), "equal": np.full(n, 3),
         "two": rng.integers(0, 2, n),
         "extremes": rng.choice(np.array([-2**31, 2**31 - 1, 0, -1]), n)}[kind].astype(np.int32)
    out, _ = run_sort(g, rt, a, 128, mode)
    assert np.array_equal(out, oracle.mergesort(a, 128)[0])


def test_forest(g, mode):
    import torch
    seg = 1 << 14
    k = 37  # total length 37 * 2^14 + 5: register-window merges
    keys = synth.keys_int32(seg * k + 5, seed=3).numpy()
    segments = [(i * seg, (i + 1) * seg) for i in range(k)] + [(seg * k, seg * k + 5)]
    d = torch.from_numpy(keys).cuda()
    st = g.mergesort_forest_(d, segments, merge_mode=mode, grid_size=148, block_size=128, max_tasks_per_worker=1024,
                             watchdog_ns=WD)
    out = d.cpu().numpy()
    tasks = 0
    for l, r in segments:
        ref, t, _ = oracle.mergesort(keys[l:r], 128)
        assert np.array_equal(out[l:r], ref)
        tasks += t
    assert st.tasks == tasks


def test_full_size_config1(g, mode):
    """BASELINE configs[1]: 2^24 random int32 keys, cutoff 128, the bench's launch configuration."""
    import torch

    import bench
    n = 1 << 24
    keys = synth.keys_int32(n, seed=42)
    d = keys.cuda()
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, watchdog_ns=60_000_000_000, **bench.MS_CFG) as r:
        st = g.mergesort_(d, cutoff=128, merge_mode=mode, rt=r)
    ref, tasks, inv = oracle.mergesort(keys.numpy(), 128)
    assert np.array_equal(d.cpu().numpy(), ref)
    assert (st.tasks, st.invocations) == (tasks, inv) == (262143, 393214)


def test_full_size_forest_c5b(g):
    """configs[4] C5b per GPU: a forest of 16 independent 2^20-key arrays (seeds 1000 + k, as bench_forest), one root per array, in
    ONE launch at the bench's launch configuration (bench.bench_forest); every array against the oracle."""
    import torch

    import bench
    k, n = bench.FOREST_WEAK_PER_GPU, bench.FOREST_EACH
    arrs = [synth.keys_int32(n, seed=1000 + j) for j in range(k)]
    d = torch.cat(arrs).cuda()
    segs = [(j * n, (j + 1) * n) for j in range(k)]
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, watchdog_ns=60_000_000_000, **dict(bench.MS_CFG, max_roots=k)) as r:
        st = g.mergesort_forest_(d, segs, cutoff=bench.MS_CUTOFF, merge_mode=bench.MS_MERGE_MODE, rt=r)
    out = d.cpu().numpy()
    tasks = inv = 0
    for j, (l, rr) in enumerate(segs):
        ref, t, i = oracle.mergesort(arrs[j].numpy(), bench.MS_CUTOFF)
        assert np.array_equal(out[l:rr], ref), j
        tasks += t
        inv += i
    assert (st.tasks, st.invocations) == (tasks, inv)


def test_forest_tma_segments(g, mode):
    import torch
    # segment lengths multiple of 4 but not of the 512-key chunk: TMA merges with partial chunks,
    # neighbouring roots writing adjacent keys concurrently
    lens = [20004 + 4 * i for i in range(24)]
    bounds = np.cumsum([0] + lens)
    keys = synth.keys_int32(int(bounds[-1]), seed=9).numpy()
    d = torch.from_numpy(keys).cuda()
    segs = [(int(bounds[i]), int(bounds[i + 1])) for i in range(len(lens))]
    g.mergesort_forest_(d, segs, merge_mode=mode, grid_size=148, block_size=128, max_tasks_per_worker=1024, watchdog_ns=WD)
    out = d.cpu().numpy()
    for l, r in segs:
        assert np.array_equal(out[l:r], np.sort(keys[l:r]))


@pytest.mark.parametrize("nseg,seg", [(2048, 1 << 15), (600, 1 << 16), (1500, 40009)])
def test_assist_board_saturation(g, nseg, seg):
    """merge_mode warp, many concurrent roots: more simultaneous merges >= 2^15 keys than GPU-wide
    board slots (1024), so requesters fall back to the block board or their own warp while slots
    open and close under them; every segment must come out sorted and the task counts exact."""
    import torch
    keys = synth.keys_int32(nseg * seg, seed=nseg).numpy()
    d = torch.from_numpy(keys).cuda()
    segs = [(i * seg, (i + 1) * seg) for i in range(nseg)]
    st = g.mergesort_forest_(d, segs, merge_mode=1, grid_size=0, block_size=128, max_tasks_per_worker=1024,
                             idle_backoff_ns=1024, watchdog_ns=WD)
    out = d.cpu().numpy().reshape(nseg, seg)
    assert np.array_equal(out, np.sort(keys.reshape(nseg, seg), axis=1))
    _, tasks, inv = oracle.mergesort(keys[:seg], 128)
    assert (st.tasks, st.invocations) == (nseg * tasks, nseg * inv)


@pytest.mark.parametrize("n", [(1 << 18) + 77, (1 << 18) + 4])   # cp.async tiles / bulk-copy merge core
@pytest.mark.parametrize("grid,block", [(1, 32), (3, 128), (148, 64)])
def test_warp_mode_small_grids(g, grid, block, n):
    """merge_mode warp with one warp / few blocks: the block and GPU-wide assists degenerate to the
    requester doing every chunk itself."""
    import torch
    keys = synth.keys_int32(n, seed=5).numpy()
    d = torch.from_numpy(keys).cuda()
    with g.Runtime(g.GTAP_WORKER_THREAD, 0, grid_size=grid, block_size=block, max_tasks_per_worker=4096,
                   watchdog_ns=WD) as r:
        st = g.mergesort_(d, cutoff=128, merge_mode=1, rt=r)
    ref, tasks, inv = oracle.mergesort(keys, 128)
    assert np.array_equal(d.cpu().numpy(), ref)
    assert (st.tasks, st.invocations) == (tasks, inv)
