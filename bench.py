#!/usr/bin/env python3
"""Benchmark of the GTaP hot path on B200 (driver contract: one JSON line on rank 0).

Headline workload: a forest of N independent mergesorts of 2^24 random int32
keys (thread-level fork-join, cutoff 128: PAPER.md P:153-165), one root
per array, the arrays dealt round-robin over the N ranks (shard.py) -- at N=1
exactly BASELINE.json configs[1]; at N>1 configs[4]'s "batched independent
mergesort forests" at configs[1]'s array size (weak scaling: 2^24 keys per
GPU). Metric Mkeys/s. A "step" is one run of the persistent scheduler over a
fresh copy of the keys: root spawn + the persistent kernel (init and result
retrieval excluded, as in the paper). Between steps (untimed) the keys
are restored, L2 is flushed by writing a 256 MiB buffer, and gtap_reset
re-arms the workspace. Each step is timed with CUDA events on the launching
stream; the job time of a step is the max over ranks. No collective runs on
the data path; after timing, ONE all_gather of per-array checksums (timed
separately: `gather_ms`).

Secondary lines (`secondary`, every config of BASELINE.json + the SURVEY §8(f)
rows): fib(40) tasks/s (configs[2]) against the measured relaxed 64-bit
L2-atomic rate, fib(20) (configs[0]), a sharded fib forest, SpMV (configs[3],
rows split by nnz over ranks), BFS RMAT-22 over 16 seeded sources split over
ranks (configs[4]), the C5b mergesort forests (16 x 2^20 per GPU weak; 128 x
2^20 over all GPUs strong). `summary` (near the end of the line) holds one
compact record per config with its oracle time; `fib40` is the last key.

`cpu_baseline` (N=1, rank 0): the oracle (oracle/, plain sequential C) timed
per config on ONE host core (sched_setaffinity, like `taskset -c 1`), median
of repeated runs, with the host's CPU model and core count.

--impl reference: the CPU oracle as it stands, timed on the host on the same
workload (one full 2^24-key array per timed step), same metric and unit.

--gpus N without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (127.0.0.1); a world size other than N is an
error.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# ---- launch configurations (shared with the full-size parity tests) ----------
MS_N = 1 << 24
MS_CUTOFF = 128
MS_CFG = dict(grid_size=0, block_size=128, max_tasks_per_worker=1024, idle_backoff_ns=1024)
MS_MERGE_MODE = 1        # GTAP_MERGE_WARP: leaf/merge bodies run by the task's warp (+ block / GPU-wide assist)
MS0_CFG = dict(grid_size=0, block_size=128, max_tasks_per_worker=1024, idle_backoff_ns=32768)  # one-lane merge
FIB_N = 40
FIB_CFG = dict(grid_size=0, block_size=128, max_tasks_per_worker=4096)
# fib(20) is launch + span bound: a smaller persistent grid starts and drains faster (grid 0 = 1,184 x 128:
# 150 us; 148 x 64 with a 256 ns idle-backoff cap: 105 us; fib(0) alone: 46 vs 12 us), P:943-948 GRID_SIZE
FIB20_CFG = dict(grid_size=148, block_size=64, max_tasks_per_worker=4096, idle_backoff_ns=256)
FIB_FOREST_ROOTS = 64    # strong scaling: 64 roots of fib(32) dealt over the ranks
FIB_FOREST_N = 32
SPMV_ROWS = 1 << 22
SPMV_NNZ_CUT = 65536
SPMV_FANOUT = 4          # a root range above the cut splits into 4 (fanout 32 made ~3 K-nnz slivers)
SPMV_PARTS = 148 * 4     # forest: one nnz-balanced root per worker (fn part(k, R), reading R20)
SPMV_CFG = dict(grid_size=148 * 4, block_size=256, max_tasks_per_worker=1024, max_roots=SPMV_PARTS)
# steals of up to 16 tasks (32 / 16 / 8 / 4: 4.20 / 3.95 / 4.02 / 4.57 ms at 2^24: bench_tools/cs_cfg_sweep.py steal)
CS_CFG = dict(grid_size=0, block_size=128, max_tasks_per_worker=4096, idle_backoff_ns=1024, steal_max=16)
NQ_N = 16
NQ_CUTOFF = 7
NQ_CFG = dict(grid_size=0, block_size=128, max_tasks_per_worker=4096)
BFS_SCALE = 22
BFS_SOURCES = 16         # 16 seeded sources, median
# one-warp blocks, 32 per SM (the 128-entry staging kernel: 3.3 KB of shared memory per block): 2368 x 64 -> 4736 x 32
# with hub splitting 7.8 -> 4.8 ms per source (bench_tools/bfs_ab.sh); batch steals (the paper's block-level steal
# takes 1): 33 -> 8.6 ms at 2368 x 64
# 2^16 records per block (12 GB of workspace; 2^15 / 2^16 / 2^17 measured equal, 3.85 / 3.86 / 3.84 ms, and 2^15
# already holds every source's local frontiers: bench_tools/bfs_pool_sweep.sh)
BFS_CFG = dict(grid_size=148 * 32, block_size=32, max_tasks_per_worker=1 << 16, idle_backoff_ns=4096,
               steal_max=32)
BFS_ORDER = 1            # oldest-first owner pops (gtap_table_bfs_ex): 9.4 -> 8.4 ms per source
BFS_SPLIT = 1024         # hub edge lists cut into bfs_edges pieces of this many edges (gtap_table_bfs_split; 0 = off)
FOREST_EACH = 1 << 20    # C5b array size
FOREST_WEAK_PER_GPU = 16
FOREST_STRONG_TOTAL = 128

L2_FLUSH_BYTES = 256 << 20
METRIC = "Mkeys/s (mergesort 2^24 int32, cutoff 128), device-timed"
UNIT = "Mkeys/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def profile_traffic(key):
    """dram bytes per launch from the committed ncu --set full summary, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ multi-rank plumbing

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _relaunch(n):
    """--gpus N outside torchrun: re-exec this script as N ranks (one process per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# Collectives run on the rank's GPU over NCCL. GTAP_BENCH_BACKEND=gloo (a test mode only: several ranks
# sharing fewer GPUs, timings meaningless) moves them to CPU tensors.
BACKEND = os.environ.get("GTAP_BENCH_BACKEND", "nccl")


def _cdev(dev):
    return dev if BACKEND == "nccl" else "cpu"


def _dist(backend=BACKEND):
    import torch.distributed as dist
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group(backend)
    return ws, rank, local


def _max_over_ranks(x, ws, dev=None):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_cdev(dev or "cuda"))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(x, ws, dev=None):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_cdev(dev or "cuda"))
    dist.all_reduce(t)
    return float(t.item())


def _barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def _fib_value(n):
    """F(n) iteratively: the bench's own correctness guard (the parity tests use the oracle)."""
    a, b = 0, 1
    for _ in range(n):
        a, b = b, a + b
    return a


# ------------------------------------------------------------------------ headline

def bench_mergesort(args, ws, rank, dev):
    """Forest of `ws` arrays of 2^24 keys (array k seeded 42 + k), dealt round robin: one per rank."""
    import torch

    import synth
    import paper_2604_05982_b200 as g
    from paper_2604_05982_b200 import shard

    n = MS_N
    mine = shard.split_round_robin(ws, ws, rank)
    assert len(mine) == 1
    aid = mine[0]
    pristine = synth.keys_int32(n, seed=42 + aid, device=dev)
    keys = torch.empty_like(pristine)
    scratch = torch.empty_like(pristine)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    rt = g.Runtime(g.GTAP_WORKER_THREAD, dev.index, **MS_CFG)
    table = g.Table.mergesort(keys, scratch, MS_CUTOFF, MS_MERGE_MODE)
    stream = torch.cuda.current_stream()

    def step():
        keys.copy_(pristine)
        flush.fill_(1)
        rt.reset(stream)
        rt.spawn_root(table, (0, n))
        rt.run(stream)
        return rt.sync()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    kern_ms = []
    stats = []
    with ClockSampler(dev.index) as clk:
        t0 = time.perf_counter()
        for i in range(args.steps):
            _barrier(ws)
            st = step()                     # runtime CUDA events around the persistent kernel (its stream)
            stats.append(st)
            kern_ms.append(_max_over_ranks(st.device_ms, ws, dev))   # job time of the step
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    _barrier(ws)
    ms = statistics.mean(kern_ms)
    own_ms = statistics.mean(s.device_ms for s in stats)
    # correctness guard: sorted + checksum (the parity tests compare with the oracle bit for bit), gathered
    sorted_ok = bool(torch.all(keys[1:] >= keys[:-1]).item())
    csum = int(keys.to(torch.int64).sum().item())
    ref_sum = int(pristine.to(torch.int64).sum().item())
    torch.cuda.synchronize()
    ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ga.record()
    rows = shard.gather_round_robin([[float(sorted_ok), float(csum == ref_sum)]], ws, ws, rank, _cdev(dev))
    gb.record()
    torch.cuda.synchronize()
    gather_ms = ga.elapsed_time(gb) if ws > 1 else 0.0
    ok = all(r is not None and r == [1.0, 1.0] for r in rows)

    # e2e through the public API with host buffers (pinned): every step copies its 2^24 keys in,
    # sorts them and copies them out. Pipelined (3 buffers): step i+1's H2D (stream s_in) and step
    # i-1's D2H (stream s_out) overlap step i's sort (compute stream); every step's copies are inside
    # the timed region, which spans all steps. A serial variant is reported beside it.
    NB = int(os.environ.get("GTAP_E2E_NB", 3))
    host_in = [pristine.cpu().pin_memory() for _ in range(NB)]
    host_out = [torch.empty_like(host_in[0]).pin_memory() for _ in range(NB)]
    kb = [keys] + [torch.empty_like(keys) for _ in range(NB - 1)]

    def e2e_serial():
        flush.fill_(1)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        keys.copy_(host_in[0], non_blocking=True)
        rt.reset(stream)
        rt.spawn_root(table, (0, n))
        rt.run(stream)
        host_out[0].copy_(keys, non_blocking=True)
        b.record(stream)
        rt.sync()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    e2e_ms = [e2e_serial() for _ in range(max(2, min(args.steps, 5)))]
    e2e_serial_ms = _max_over_ranks(statistics.mean(e2e_ms), ws, dev)
    s_in, s_out, sc = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    tables = [table] + [g.Table.mergesort(kb[j], scratch, MS_CUTOFF, MS_MERGE_MODE) for j in range(1, NB)]
    # two runtimes (two workspaces) used alternately: a run is enqueued on the compute stream behind the previous
    # one without the host first waiting for it (gtap_sync of a runtime only before its next-but-one reuse), so
    # the GPU never idles on a host round trip between consecutive sorts
    rts = [rt, g.Runtime(g.GTAP_WORKER_THREAD, dev.index, **MS_CFG)]
    # a stream of 32 sorts (or --steps if more): the pipeline fill (first H2D) and drain (last D2H), ~2 ms each,
    # are paid once per stream (10 steps: 1.9 ms per step; 40: 1.58; 100: 1.49 -- transfer-bound steady state)
    ksteps = int(os.environ.get("GTAP_E2E_STEPS", max(32, args.steps)))
    ev_in = [torch.cuda.Event() for _ in range(NB)]
    ev_sorted = [torch.cuda.Event() for _ in range(NB)]
    ev_out = [torch.cuda.Event() for _ in range(NB)]
    torch.cuda.synchronize()
    _barrier(ws)
    t_a, t_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_a.record(sc)
    s_in.wait_event(t_a)
    for i in range(ksteps + 1):
        if i < ksteps:
            bi = i % NB
            with torch.cuda.stream(s_in):
                if i >= NB:
                    s_in.wait_event(ev_out[bi])
                kb[bi].copy_(host_in[bi], non_blocking=True)
                ev_in[bi].record(s_in)
        if i >= 1:
            bj = (i - 1) % NB
            r_ = rts[(i - 1) % 2]
            sc.wait_event(ev_in[bj])
            if i >= 3:
                r_.sync()
            r_.reset(sc)
            r_.spawn_root(tables[bj], (0, n))
            r_.run(sc)
            ev_sorted[bj].record(sc)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_sorted[bj])
                host_out[bj].copy_(kb[bj], non_blocking=True)
                ev_out[bj].record(s_out)
    for r_ in rts[:min(2, ksteps)]:
        r_.sync()
    sc.wait_stream(s_out)
    t_b.record(sc)
    torch.cuda.synchronize()
    e2e_pipe_ms = _max_over_ranks(t_a.elapsed_time(t_b) / ksteps, ws, dev)
    pipe_ok = all(bool(torch.equal(host_out[j], kb[j].cpu())) for j in range(NB)) and \
        bool(torch.all(host_out[0][1:] >= host_out[0][:-1]).item())
    for t in tables[1:]:
        t.close()
    rts[1].close()
    st = stats[-1]
    algo_bytes = 8.0 * n * (1 + _ms_levels(n, MS_CUTOFF))  # read+write per key per pass
    pk, src = peaks()
    achieved = algo_bytes / (own_ms * 1e-3) / 1e9
    res = dict(
        value=ws * n / (ms * 1e-3) / 1e6, ms_per_step=ms, wall_ms_per_step=wall * 1e3 / args.steps,
        e2e=dict(value=ws * n / (e2e_pipe_ms * 1e-3) / 1e6, unit=UNIT, h2d_bytes_per_step=4 * n,
                 d2h_bytes_per_step=4 * n, ms_per_step=e2e_pipe_ms,
                 mode="pipelined (3 buffers: H2D / sort / D2H of consecutive steps overlap; two runtimes alternate so the next sort is queued before the previous one ends)",
                 steps=ksteps, correct=pipe_ok,
                 serial=dict(value=ws * n / (e2e_serial_ms * 1e-3) / 1e6, ms_per_step=e2e_serial_ms)),
        roofline=dict(bound="hbm", achieved=achieved, peak=pk["hbm_gbs"], unit="GB/s",
                      frac=achieved / pk["hbm_gbs"], traffic=profile_traffic("mergesort"),
                      peak_source=src, algorithmic_bytes_per_launch=algo_bytes,
                      algorithmic_bytes_per_key=8.0 * (1 + _ms_levels(n, MS_CUTOFF)),
                      note="8 B/key (read + write) for the leaf pass and each of the merge levels; the "
                           "persistent scheduler kernel is the only kernel of the step; per GPU"),
        stats=dict(tasks=st.tasks, invocations=st.invocations, steals_ok=st.steals_ok, workers=st.workers,
                   grid=st.grid_size, block=st.block_size, assists=st.assists),
        correct=ok, gather_ms=gather_ms, clocks=clk.summary(), gpu_launches=args.steps,
        gpu_launches_note="1 persistent scheduler kernel per step inside the runtime's kernel events; each gtap_run "
                          "also launches 3 small kernels outside them (root/control staging in, assist-board fill, "
                          "control block out; no copy-engine work)",
    )
    rt.close()
    table.close()
    return res


def _ms_levels(n, c):
    lv = 0
    while n > c:
        n = (n + 1) // 2
        lv += 1
    return lv


# ----------------------------------------------------------------------- secondary

def bench_mergesort_thread_merge(dev, reps=2):
    """The paper's one-lane merge (GTAP_MERGE_THREAD): same task graph, every leaf sort and
    merge body on its task's own lane (long merges TMA-staged); span-bound by the top merge."""
    import torch

    import synth
    import paper_2604_05982_b200 as g
    keys0 = synth.keys_int32(MS_N, seed=42, device=dev)
    keys = torch.empty_like(keys0)
    scratch = torch.empty_like(keys0)
    ms = []
    with g.Runtime(g.GTAP_WORKER_THREAD, dev.index, **MS0_CFG) as rt:
        for i in range(reps + 1):
            keys.copy_(keys0)
            st = g.mergesort_(keys, scratch, MS_CUTOFF, merge_mode=0, rt=rt)
            if i:
                ms.append(st.device_ms)
    t = statistics.median(ms)
    assert bool(torch.all(keys[1:] >= keys[:-1]).item())
    return dict(workload="mergesort 2^24 cutoff 128, merge_mode=thread (paper's one-lane merge, P:593)",
                metric="Mkeys/s", value=MS_N / (t * 1e-3) / 1e6, ms=t,
                span_note=f"critical path ~{2 * MS_N} sequential merge steps, {t * 1e6 / (2 * MS_N):.2f} ns/step")


def bench_fib(dev, ws=1, reps=3):
    """configs[2]: fib(40), one root (does not shard: replicas only at N > 1)."""
    import paper_2604_05982_b200 as g
    rt = g.Runtime(g.GTAP_WORKER_THREAD, dev.index, **FIB_CFG)
    ms = []
    st = None
    for i in range(reps + 1):
        v, st = g.fib(FIB_N, rt=rt)
        assert v == _fib_value(FIB_N)
        if i:
            ms.append(st.device_ms)
    rt.close()
    t = _max_over_ranks(statistics.median(ms), ws, dev)
    tasks = st.tasks
    return dict(workload="fib(40) no cutoff, thread-level (configs[2])" + (", replica per GPU" if ws > 1 else ""),
                metric="tasks/s", value=tasks / (t * 1e-3), ms=t, tasks=tasks, invocations=st.invocations,
                workers=st.workers, steals_ok=st.steals_ok, join_atomics=tasks - 1)


def bench_fib20(dev, ws=1, reps=20):
    """BASELINE configs[0] / SURVEY §8(d) C1: fib(20) (21,891 tasks) is span-bound -- its critical path is
    2n - 1 = 39 dependent invocations -- so it is reported as tasks/s and as time per critical-path step."""
    import paper_2604_05982_b200 as g
    rt = g.Runtime(g.GTAP_WORKER_THREAD, dev.index, **FIB20_CFG)
    ms = []
    st = None
    for i in range(reps + 1):
        v, st = g.fib(20, rt=rt)
        assert v == 6765
        if i:
            ms.append(st.device_ms)
    rt.close()
    t = _max_over_ranks(statistics.median(ms), ws, dev)
    q = statistics.quantiles(ms, n=4)
    return dict(workload="fib(20) no cutoff, thread-level (configs[0]), launch + span bound", metric="tasks/s",
                value=st.tasks / (t * 1e-3), ms=t, ms_iqr=[q[0], q[2]], runs=len(ms), tasks=st.tasks,
                invocations=st.invocations, us_per_critical_path_invocation=t * 1e3 / 39.0,
                note="critical path 2n-1 = 39 dependent invocations (SURVEY §8(a) A12a); includes the persistent "
                     "kernel's start and drain")


def bench_fib_forest(dev, ws=1, rank=0, reps=3):
    """a fib forest shards -- 64 roots of fib(32) dealt round robin over the ranks, each rank
    runs its roots in ONE launch, one all_gather of the 4-B root results after timing (strong scaling)."""
    import paper_2604_05982_b200 as g
    from paper_2604_05982_b200 import shard
    mine = shard.split_round_robin(FIB_FOREST_ROOTS, ws, rank)
    ns = [FIB_FOREST_N] * len(mine)
    rt = g.Runtime(g.GTAP_WORKER_THREAD, dev.index, **dict(FIB_CFG, max_roots=len(ns)))
    ms = []
    for i in range(reps + 1):
        rt.reset()
        vals, st = g.fib_forest(ns, rt=rt)
        if i:
            ms.append(st.device_ms)
    rt.close()
    t = _max_over_ranks(statistics.median(ms), ws, dev)
    tasks = _sum_over_ranks(float(st.tasks), ws, dev)
    got = shard.gather_round_robin([[float(v)] for v in vals], FIB_FOREST_ROOTS, ws, rank, _cdev(dev))
    ok = all(r is not None and int(r[0]) == _fib_value(FIB_FOREST_N) for r in got)
    return dict(workload=f"fib forest: {FIB_FOREST_ROOTS} roots of fib({FIB_FOREST_N}) over {ws} GPU(s), "
                         f"round robin (SURVEY §8(e)), strong scaling", metric="tasks/s",
                value=tasks / (t * 1e-3), ms=t, tasks=int(tasks), roots_per_gpu=len(mine), correct=ok,
                scaling="strong")


EPAQ_POOL = 32768   # records per worker: the "stay" policy holds a deeper frontier of suspended tasks


def bench_epaq(dev, reps=3):
    """fib(40) with a cutoff, 1 queue vs EPAQ with 3 queues, under both
    kept-class policies (gtap_config.queue_policy: 0 rotate every cycle, 1 stay while the class has work,
    P:177-178 literal), at cutoff 10 and 14; every run with EPAQ_POOL records per worker."""
    import paper_2604_05982_b200 as g
    out = {}
    for cutoff in (10, 14):
        for nq, pol in ((1, 0), (3, 0), (3, 1)):
            with g.Runtime(g.GTAP_WORKER_THREAD, dev.index, num_queues=3, queue_policy=pol,
                           **dict(FIB_CFG, max_tasks_per_worker=EPAQ_POOL)) as rt:
                ms = []
                for i in range(reps + 1):
                    v, st = g.fib_cutoff(FIB_N, cutoff, nq, rt=rt)
                    assert v == _fib_value(FIB_N)
                    if i:
                        ms.append(st.device_ms)
            out[(cutoff, nq, pol)] = statistics.median(ms)
    pts = {f"cutoff{c}": dict(ms_1q=out[(c, 1, 0)], ms_epaq_rotate=out[(c, 3, 0)], ms_epaq_stay=out[(c, 3, 1)],
                              speedup_rotate=out[(c, 1, 0)] / out[(c, 3, 0)],
                              speedup_stay=out[(c, 1, 0)] / out[(c, 3, 1)]) for c in (10, 14)}
    return dict(workload="fib(40) with cutoff: EPAQ 3 queues vs 1 queue (NEXT #1)", metric="speedup",
                value=pts["cutoff10"]["speedup_stay"], points=pts, records_per_worker=EPAQ_POOL,
                paper="~1.8x on GH200 (P:788)")


def bench_cilksort(dev, reps=3):
    """Cilksort of the same 2^24 keys (parallel merge)."""
    import torch

    import synth
    import paper_2604_05982_b200 as g
    pristine = synth.keys_int32(MS_N, seed=42, device=dev)
    keys = torch.empty_like(pristine)
    scratch = torch.empty_like(pristine)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    with g.Runtime(g.GTAP_WORKER_THREAD, dev.index, **CS_CFG) as rt:
        ms = []
        for i in range(reps + 1):
            keys.copy_(pristine)
            flush.fill_(1)
            st = g.cilksort_(keys, scratch, 64, 256, rt=rt)
            if i:
                ms.append(st.device_ms)
    ok = bool(torch.all(keys[1:] >= keys[:-1]).item())
    t = statistics.median(ms)
    pk, _ = peaks()
    levels = _ms_levels(MS_N, 64)
    algo = 8.0 * MS_N * (1 + levels)
    return dict(workload="Cilksort 2^24 int32, cut 64/256 (NEXT #2), thread-level", metric="Mkeys/s",
                value=MS_N / (t * 1e-3) / 1e6, ms=t, tasks=st.tasks, sorted=ok,
                roofline=dict(bound="hbm", achieved=algo / (t * 1e-3) / 1e9, peak=pk["hbm_gbs"], unit="GB/s",
                              frac=algo / (t * 1e-3) / 1e9 / pk["hbm_gbs"]))


def bench_forest(dev, ws=1, rank=0, arrays_total=FOREST_WEAK_PER_GPU, n_each=FOREST_EACH, scaling="weak", reps=3):
    """a forest of independent 2^20-key mergesorts, one root per array, the arrays dealt
    round robin over the ranks (shard.split_round_robin); each rank sorts its arrays in ONE launch. After
    timing, one all_gather of per-array checksums. Aggregate = all keys / slowest rank's time."""
    import torch

    import synth
    import paper_2604_05982_b200 as g
    from paper_2604_05982_b200 import shard
    mine = shard.split_round_robin(arrays_total, ws, rank)
    arrays = len(mine)
    n = arrays * n_each
    pristine = torch.cat([synth.keys_int32(n_each, seed=1000 + i, device=dev) for i in mine])
    keys = torch.empty_like(pristine)
    scratch = torch.empty_like(pristine)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    segs = [(i * n_each, (i + 1) * n_each) for i in range(arrays)]
    with g.Runtime(g.GTAP_WORKER_THREAD, dev.index, **dict(MS_CFG, max_roots=arrays)) as rt:
        ms = []
        for i in range(reps + 1):
            keys.copy_(pristine)
            flush.fill_(1)
            st = g.mergesort_forest_(keys, segs, scratch, MS_CUTOFF, merge_mode=MS_MERGE_MODE, rt=rt)
            if i:
                ms.append(st.device_ms)
    k2 = keys.view(arrays, n_each)
    ok = bool(torch.equal(torch.sort(pristine.view(arrays, n_each), dim=1).values, k2))
    t = _max_over_ranks(statistics.median(ms), ws, dev)
    torch.cuda.synchronize()
    ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ga.record()
    rows = shard.gather_round_robin([[float(ok), float(arrays)]], ws, ws, rank, _cdev(dev))   # one row per rank
    gb.record()
    torch.cuda.synchronize()
    ok_all = all(r[0] == 1.0 for r in rows) and int(sum(r[1] for r in rows)) == arrays_total
    pk, _ = peaks()
    levels = _ms_levels(n_each, MS_CUTOFF)
    total = arrays_total * n_each
    algo_per_gpu = 8.0 * n * (1 + levels)
    return dict(workload=f"mergesort forest {arrays_total} x 2^20 int32 over {ws} GPU(s) (configs[4] C5b, "
                         f"{scaling}), thread-level, cutoff 128", metric="Mkeys/s",
                value=total / (t * 1e-3) / 1e6, ms=t, arrays_per_gpu=arrays, tasks=st.tasks, correct=ok_all,
                scaling=scaling, gather_ms=ga.elapsed_time(gb) if ws > 1 else 0.0,
                roofline=dict(bound="hbm", achieved=algo_per_gpu / (t * 1e-3) / 1e9, peak=pk["hbm_gbs"],
                              unit="GB/s", frac=algo_per_gpu / (t * 1e-3) / 1e9 / pk["hbm_gbs"],
                              algorithmic_bytes_per_key=8.0 * (1 + levels)))


def bench_nqueens(dev, reps=3):
    """N-Queens n = 16, cutoff depth 7."""
    import paper_2604_05982_b200 as g
    with g.Runtime(g.GTAP_WORKER_THREAD, dev.index, **NQ_CFG) as rt:
        ms = []
        for i in range(reps + 1):
            sol, st = g.nqueens(NQ_N, NQ_CUTOFF, rt=rt)
            assert sol == 14772512
            if i:
                ms.append(st.device_ms)
    t = statistics.median(ms)
    return dict(workload="N-Queens n=16 cutoff 7 (NEXT #4), thread-level, no taskwait", metric="tasks/s",
                value=st.tasks / (t * 1e-3), ms=t, tasks=st.tasks, solutions=sol)


TREE_CFG = {"thread": dict(grid_size=0, block_size=128, max_tasks_per_worker=4096),
            "block": dict(grid_size=148 * 32, block_size=32, max_tasks_per_worker=2048)}


def bench_tree(dev, reps=3):
    """synthetic trees on both worker kinds: full binary D = 22
    (mem_ops 64, compute_iters 256) and pruned 3-ary D = 24 (mem_ops 64, compute_iters 32768); the
    pseudo-random loads read a 256 MiB table (HBM, not L2)."""
    import synth
    import paper_2604_05982_b200 as g
    buf = synth.tree_buffer(1 << 25, device=dev)
    pts = {}
    for kind, wk in (("thread", g.GTAP_WORKER_THREAD), ("block", g.GTAP_WORKER_BLOCK)):
        with g.Runtime(wk, dev.index, **TREE_CFG[kind]) as rt:
            for name, D, mem, comp, pruned in (("full_D22", 22, 64, 256, False),
                                               ("pruned_D24_comp32768", 24, 64, 32768, True)):
                ms = []
                for i in range(reps + 1):
                    _, st = g.tree(D, buf, mem, comp, pruned=pruned, worker=wk, rt=rt)
                    if i:
                        ms.append(st.device_ms)
                t = statistics.median(ms)
                pts[f"{name}_{kind}"] = dict(ms=t, tasks=st.tasks, tasks_per_s=st.tasks / (t * 1e-3))
    return dict(workload="synthetic trees (NEXT #3), thread- vs block-level", metric="tasks/s", points=pts)


ATOM_KINDS = (("atom_add_relaxed", 0), ("red_add", 1), ("atom_cas", 2), ("atom_min", 3),
              ("same_address_add", 4), ("atom_add_acq_rel", 5), ("atom_add_u64_relaxed", 6))


def bench_atomics(dev):
    import torch

    import paper_2604_05982_b200 as g
    small = torch.empty(1 << 22, dtype=torch.int32, device=dev)  # 16 MiB: L2-resident
    out = {}
    grid, block, ops = 148 * 8, 256, 64
    for name, kind in ATOM_KINDS:
        g.ubench_atomics(small, kind, grid, block, ops)
        o = ops if kind != 4 else 4
        ms = min(g.ubench_atomics(small, kind, grid, block, o) for _ in range(3))
        out[name] = grid * block * o / (ms * 1e-3)
    return out


def bench_spmv(dev, ws=1, rank=0, reps=5):
    """configs[3]: x replicated, rows partitioned over ranks by nnz, one all_gather of y after timing."""
    import torch

    import synth
    import paper_2604_05982_b200 as g
    from paper_2604_05982_b200 import shard
    rp, col, val, x = synth.powerlaw_csr(SPMV_ROWS, seed=7, device=dev)
    ranges = shard.split_rows_by_nnz(rp.cpu(), ws)
    lo, hi = ranges[rank]
    y = torch.zeros(SPMV_ROWS, dtype=torch.float32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    rt = g.Runtime(g.GTAP_WORKER_BLOCK, dev.index, **SPMV_CFG)
    ms = []
    st = None
    for i in range(reps + 1):
        flush.fill_(1)
        rt.reset()
        y, st = g.spmv(rp, col, val, x, y, SPMV_NNZ_CUT, SPMV_FANOUT, rows=(lo, hi), parts=SPMV_PARTS, rt=rt)
        if i:
            ms.append(st.device_ms)
    rt.close()
    t = _max_over_ranks(statistics.median(ms), ws, dev)
    gather_ms = 0.0
    if ws > 1:  # the only collective: gather the y slices (outside the timed region, timed on its own)
        torch.cuda.synchronize()
        ga, gb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ga.record()
        y = shard.gather_slices(y[lo:hi].contiguous().to(_cdev(dev)), ranges, rank).to(dev)
        gb.record()
        torch.cuda.synchronize()
        gather_ms = ga.elapsed_time(gb)
    nnz = int(rp[-1].item())
    algo = 8.0 * nnz + 12.0 * SPMV_ROWS  # col+val per nnz; row_ptr + y + x once per row
    pk, _ = peaks()
    return dict(workload=f"SpMV power-law 2^22 rows (configs[3]), block-level, rows split over {ws} GPU(s)",
                metric="GB/s", value=algo / (t * 1e-3) / 1e9, gflops=2.0 * nnz / (t * 1e-3) / 1e9, ms=t, nnz=nnz,
                tasks=st.tasks, frac_hbm_per_gpu=algo / ws / (t * 1e-3) / 1e9 / pk["hbm_gbs"], roots=SPMV_PARTS,
                gather_ms=gather_ms, gather_floor_ms=0.50,
                gather_floor_note="a bare streaming gather (sum val*x[col], no rows, no scheduler) over this matrix "
                                  "takes 0.50 ms on B200 (profiles/r01_spmv_gather_floor.txt)",
                traffic=profile_traffic("spmv"), scaling="strong", y_checksum=float(y.double().sum().item()))


def bench_bfs(dev, ws=1, rank=0, atom_min_peak=None, nsrc_total=BFS_SOURCES):
    """configs[4] / SURVEY §8(d) C5a: 16 seeded sources, graph replicated, sources dealt round robin over
    the ranks (shard.split_round_robin); per-source GTEPS (Graph500 edge count), median over all 16."""
    import torch

    import synth
    import paper_2604_05982_b200 as g
    from paper_2604_05982_b200 import shard
    rp, col = synth.rmat_csr(BFS_SCALE, 16, seed=3, device=dev)
    depth = torch.empty(rp.numel() - 1, dtype=torch.int32, device=dev)
    deg = (rp[1:] - rp[:-1]).to(torch.int64)
    rt = g.Runtime(g.GTAP_WORKER_BLOCK, dev.index, **BFS_CFG)
    allsrc = synth.bfs_sources(rp, nsrc_total, seed=5)
    mine = shard.split_round_robin(nsrc_total, ws, rank)
    rt.reset()
    g.bfs(rp, col, allsrc[0], depth, rt=rt, order=BFS_ORDER, edge_split=BFS_SPLIT)  # warm-up (untimed)
    per = []
    for k in mine:
        rt.reset()
        depth, st = g.bfs(rp, col, allsrc[k], depth, rt=rt, order=BFS_ORDER, edge_split=BFS_SPLIT)
        reached = depth != 0x7FFFFFFF
        edges = int(deg[reached].sum().item()) // 2  # undirected input edges in the component (Graph500)
        per.append([float(k), edges / (st.device_ms * 1e-3), st.device_ms, float(st.tasks),
                    float(reached.sum().item()), float(edges)])
    rt.close()
    allper = shard.gather_round_robin(per, nsrc_total, ws, rank, _cdev(dev))   # one row per source, source order
    rank_time = [sum(allper[k][2] for k in shard.split_round_robin(nsrc_total, ws, r)) for r in range(ws)]
    teps = statistics.median(p[1] for p in allper)
    out = dict(workload="BFS RMAT scale 22 ef 16 (configs[4]), block-level", metric="GTEPS", value=teps / 1e9,
               order="oldest-first owner pops (gtap_table_bfs_ex order 1)" if BFS_ORDER else "LIFO owner pops",
               edge_split=BFS_SPLIT, grid=BFS_CFG["grid_size"], block=BFS_CFG["block_size"],
               ms=statistics.median(p[2] for p in allper), sources=len(allper),
               tasks_over_reached=statistics.median(p[3] / p[4] for p in allper),
               reached=int(statistics.median(p[4] for p in allper)))
    if atom_min_peak:
        # L2-atomic roofline: one atom.min per scanned CSR entry; every reached vertex is
        # expanded at least once, so the scanned entries are at least 2 x the component's undirected edges
        # (a lower bound: re-expansions scan more), i.e. achieved >= 2 x TEPS
        ach = 2.0 * teps
        out["roofline"] = dict(bound="l2_atomic", achieved=ach, peak=atom_min_peak, unit="atomics/s",
                               frac=ach / atom_min_peak, peak_source="measured live: gtap_ubench_atomics atom.min")
    if ws > 1:  # aggregate: every rank's edges over the slowest rank's total time (no collective on the path)
        out.update(aggregate_gteps=sum(p[5] for p in allper) / (max(rank_time) * 1e-3) / 1e9, scaling="weak")
    return out


# ------------------------------------------------------------------ CPU baseline (oracle)

def _host_desc():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return dict(cpu_model=model or platform.processor() or "unknown", nproc=os.cpu_count())


class _PinOneCore:
    """Run the oracle on one host core (the calling thread's affinity, like `taskset -c 1`)."""

    def __enter__(self):
        self.old = None
        try:
            self.old = os.sched_getaffinity(0)
            cpus = sorted(self.old)
            self.cpu = 1 if 1 in cpus else cpus[0]
            os.sched_setaffinity(0, {self.cpu})
        except Exception:
            self.cpu = None
        return self

    def __exit__(self, *a):
        if self.old:
            os.sched_setaffinity(0, self.old)


def _median_time(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), len(ts)


def cpu_baseline(dev):
    """The oracle as it stands (sequential C, gcc -O3, one pinned core), per config, median of repeats.

    Inputs are generated on the GPU by synth/ (identical on CPU and CUDA) and copied to the host; only the
    oracle call is timed."""
    import torch

    import oracle
    import synth
    oracle.build()
    per = {}
    with _PinOneCore() as pin:
        t, k = _median_time(lambda: oracle.fib(20), 20)
        per["C1_fib20"] = dict(ms=t * 1e3, runs=k, value=21891 / t, unit="tasks/s")
        keys = synth.keys_int32(MS_N, seed=42, device=dev).cpu().numpy()
        t, k = _median_time(lambda: oracle.mergesort(keys, MS_CUTOFF), 3)
        per["C2_mergesort_2p24"] = dict(ms=t * 1e3, runs=k, value=MS_N / t / 1e6, unit="Mkeys/s")
        del keys
        t, k = _median_time(lambda: oracle.fib(FIB_N), 3)
        per["C3_fib40"] = dict(ms=t * 1e3, runs=k, value=331160281 / t, unit="tasks/s")
        rp, col, val, x = (a.cpu().numpy() for a in synth.powerlaw_csr(SPMV_ROWS, seed=7, device=dev))
        nnz = int(rp[-1])
        t, k = _median_time(lambda: oracle.spmv(rp, col, val, x), 3)
        per["C4_spmv"] = dict(ms=t * 1e3, runs=k, value=(8.0 * nnz + 12.0 * SPMV_ROWS) / t / 1e9, unit="GB/s")
        del rp, col, val, x
        rpt, colt = synth.rmat_csr(BFS_SCALE, 16, seed=3, device=dev)
        srcs = synth.bfs_sources(rpt, BFS_SOURCES, seed=5)
        rp, col = rpt.cpu().numpy(), colt.cpu().numpy()
        del rpt, colt
        deg = (rp[1:] - rp[:-1]).astype("int64")
        teps, ts = [], []
        for s in srcs:
            t0 = time.perf_counter()
            lv = oracle.bfs(rp, col, s)
            dt = time.perf_counter() - t0
            ts.append(dt)
            teps.append(int(deg[lv != 0x7FFFFFFF].sum()) // 2 / dt)
        per["C5a_bfs"] = dict(ms=statistics.median(ts) * 1e3, runs=len(ts), value=statistics.median(teps) / 1e9,
                              unit="GTEPS")
        del rp, col
        arrs = [synth.keys_int32(FOREST_EACH, seed=1000 + i, device=dev).cpu().numpy()
                for i in range(FOREST_WEAK_PER_GPU)]
        t, k = _median_time(lambda: [oracle.mergesort(a, MS_CUTOFF) for a in arrs], 3)
        per["C5b_forest_16x2p20"] = dict(ms=t * 1e3, runs=k, value=FOREST_WEAK_PER_GPU * FOREST_EACH / t / 1e6,
                                         unit="Mkeys/s")
        cpu = pin.cpu
    torch.cuda.synchronize()
    head = per["C2_mergesort_2p24"]
    return dict(value=head["value"], unit=UNIT, cores=1, kind="oracle",
                sample="oracle mergesort of the full 2^24-key headline array (seed 42), median of 3; every other "
                       "config in per_config at its full bench size",
                pinned_cpu=cpu, compiler="gcc -O3 -ffp-contract=off", **_host_desc(), per_config=per)


# --------------------------------------------------------------------------- driver

def _summary(res, secondary, cpu):
    """One compact record per BASELINE config (value, time, roofline fraction, oracle time)."""
    def find(prefix):
        for s in secondary:
            if s.get("workload", "").startswith(prefix):
                return s
        return {}

    per = (cpu or {}).get("per_config", {})

    def rec(s, key, unit, extra=()):
        if not s:
            return None
        r = {"value": s.get("value"), "unit": unit, "ms": s.get("ms")}
        for k in extra:
            if k in s:
                r[k] = s[k]
        if "roofline" in s:
            r["frac"] = s["roofline"].get("frac")
        if key in per:
            r["oracle_ms"] = per[key]["ms"]
            r["speedup_vs_oracle"] = per[key]["ms"] / s["ms"] if s.get("ms") else None
        return r

    out = {
        "C1_fib20": rec(find("fib(20)"), "C1_fib20", "tasks/s", ("us_per_critical_path_invocation",)),
        "C2_mergesort_2p24": dict(value=res["value"], unit=UNIT, ms=res["ms_per_step"],
                                  frac=res["roofline"]["frac"]),
        "C4_spmv": rec(find("SpMV"), "C4_spmv", "GB/s", ("frac_hbm_per_gpu", "gather_ms")),
        "C5a_bfs": rec(find("BFS"), "C5a_bfs", "GTEPS", ("sources", "tasks_over_reached", "aggregate_gteps")),
        "C5b_forest_weak": rec(find("mergesort forest 16") or find("mergesort forest"), "C5b_forest_16x2p20",
                               "Mkeys/s", ("gather_ms",)),
        "C5b_forest_strong": rec(find(f"mergesort forest {FOREST_STRONG_TOTAL}"), "", "Mkeys/s", ("gather_ms",)),
        "fib_forest": rec(find("fib forest"), "", "tasks/s", ("correct",)),
    }
    if "C2_mergesort_2p24" in per:
        out["C2_mergesort_2p24"]["oracle_ms"] = per["C2_mergesort_2p24"]["ms"]
        out["C2_mergesort_2p24"]["speedup_vs_oracle"] = per["C2_mergesort_2p24"]["ms"] / res["ms_per_step"]
    return {k: v for k, v in out.items() if v is not None}


def _round(o, sig=5):
    """Floats to `sig` significant digits (keeps the one-line JSON short enough for the driver's tail)."""
    if isinstance(o, float):
        return float(f"{o:.{sig}g}")
    if isinstance(o, dict):
        return {k: _round(v, sig) for k, v in o.items()}
    if isinstance(o, (list, tuple)):
        return [_round(v, sig) for v in o]
    return o


def run_ours(args):
    import torch
    ws, rank, local = _dist()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: world size {ws} != --gpus {args.gpus}")
    local = local % torch.cuda.device_count()   # == LOCAL_RANK with one GPU per rank
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    res = bench_mergesort(args, ws, rank, dev)
    secondary = []
    atoms = {}
    fibr = None

    def leg(fn, *a, **k):
        try:
            r = fn(*a, **k)
            secondary.append(r)
            return r
        except Exception as e:  # a secondary result must not kill the headline
            secondary.append(dict(workload=fn.__name__, error=repr(e)))
            return None

    if not args.no_secondary:
        atoms = leg(bench_atomics, dev) or {}
        if atoms:
            secondary[-1] = dict(workload="L2 atomic probes (gtap_ubench_atomics, distinct L2-resident sectors)",
                                 metric="ops/s", value=atoms)
        fibr = leg(bench_fib, dev, ws)
        if fibr and atoms:
            peak = atoms["atom_add_u64_relaxed"]
            ach = fibr["join_atomics"] / (fibr["ms"] * 1e-3)
            fibr["roofline"] = dict(bound="l2_atomic", achieved=ach, peak=peak, unit="atomics/s", frac=ach / peak,
                                    peak_source="measured live: gtap_ubench_atomics kind 6 (relaxed 64-bit atom.add "
                                                "with return, distinct L2-resident sectors) = the fused join RMW")
        leg(bench_fib20, dev, ws)
        leg(bench_fib_forest, dev, ws, rank)
        leg(bench_forest, dev, ws, rank, FOREST_WEAK_PER_GPU * ws, scaling="weak")
        leg(bench_forest, dev, ws, rank, FOREST_STRONG_TOTAL, scaling="strong")
        leg(bench_spmv, dev, ws, rank)
        leg(bench_bfs, dev, ws, rank, atoms.get("atom_min"))
        leg(bench_epaq, dev)
        leg(bench_nqueens, dev)
        leg(bench_mergesort_thread_merge, dev)
        leg(bench_cilksort, dev)
        leg(bench_tree, dev)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(dev)
    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": "mergesort forest: one independent 2^24-key random int32 array per GPU "
                                   "(N=1: BASELINE configs[1]; N>1: configs[4] batched forests at that array size), "
                                   "thread-level fork-join, cutoff 128",
                       "keys_per_gpu": MS_N, "arrays_total": ws, "cutoff": MS_CUTOFF, "launch": MS_CFG,
                       "merge_mode": "warp (leaf-sort and merge bodies run by the task's warp, long merges shared by "
                                     "idle warps; same task graph; the paper's one-lane merge is a secondary line)",
                       "grid": res["stats"]["grid"], "block": res["stats"]["block"],
                       "workers": res["stats"]["workers"], "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"forest over {ws} GPU(s): arrays dealt round robin, one root per array; "
                                      "no collective on the data path; one all_gather of checksums after timing",
                       "timing": "persistent-kernel CUDA events (PAPER P:323), max over ranks per step; input "
                                 "restore, L2 flush and gtap_reset untimed between steps"},
            "e2e": res["e2e"], "roofline": res["roofline"], "gpu_launches": res["gpu_launches"],
            "gpu_launches_note": res["gpu_launches_note"], "gather_ms": res["gather_ms"],
            "correct": res["correct"], "stats": res["stats"], "wall_ms_per_step": res["wall_ms_per_step"],
            "secondary": secondary,
            "clocks": res["clocks"],
        }
        if cpu:
            line["cpu_baseline"] = cpu
        line["summary"] = _summary(res, secondary, cpu)
        if fibr:
            f = {k: fibr.get(k) for k in ("value", "ms", "tasks", "invocations")}
            f["roofline"] = {k: fibr["roofline"][k] for k in ("bound", "achieved", "peak", "unit", "frac")} \
                if "roofline" in fibr else None
            f["metric"] = "tasks/s (fib(40), configs[2])"
            if cpu:
                f["oracle_ms"] = cpu["per_config"]["C3_fib40"]["ms"]
                f["speedup_vs_oracle"] = f["oracle_ms"] / fibr["ms"]
                f["paper"] = "2.4x vs one Grace core on GH200 (P:585); context only"
            line["fib40"] = f
        print(json.dumps(_round(line)), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    """The CPU oracle as it stands, timed on the host (rank 0 only): one full 2^24-key array per step."""
    rank = int(os.environ.get("RANK", "0"))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        raise SystemExit(f"bench.py: world size {ws} != --gpus {args.gpus}")
    if rank != 0:
        return
    import oracle
    import synth
    oracle.build()
    keys = synth.keys_int32(MS_N, seed=42).numpy()
    times = []
    with _PinOneCore() as pin:
        for _ in range(args.warmup):               # warm-up on a small prefix (untimed)
            oracle.mergesort(keys[: 1 << 16], MS_CUTOFF)
        for _ in range(args.steps):
            t0 = time.perf_counter()
            oracle.mergesort(keys, MS_CUTOFF)
            times.append(time.perf_counter() - t0)
        cpu = pin.cpu
    t = statistics.median(times)
    v = MS_N / t / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": "mergesort 2^24 random int32 keys, cutoff 128 (BASELINE configs[1]); each timed step "
                               "sorts one full 2^24-key array (seed 42) with the sequential C oracle",
                   "same_workload_per_gpu": True},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "pinned_cpu": cpu,
                         "compiler": "gcc -O3 -ffp-contract=off",
                         "sample": f"one full 2^24-key array per step, {args.steps} steps, median", **_host_desc()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
