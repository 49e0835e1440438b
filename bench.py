#!/usr/bin/env python3
"""Benchmark of the GTaP hot path on B200 (driver contract: one JSON line on rank 0).

Workload (N=1): BASELINE.json configs[1] -- mergesort of 2^24 random int32 keys,
thread-level fork-join with cutoff 128, metric
Mkeys/s. A "step" is one run of the persistent scheduler over a fresh copy of
the keys: root spawn + the persistent kernel (init and result retrieval are
excluded, as in the paper). Between steps (untimed) the keys are
restored, L2 is flushed by writing a 256 MiB buffer, and gtap_reset re-arms
the workspace. Each step is timed with CUDA events on the launching stream.

Secondary results in the same line (`secondary`): fib(40) tasks/s
(configs[2]) against the measured L2-atomic rate, SpMV (configs[3]) GB/s
against HBM, BFS RMAT-22 (configs[4]) GTEPS. Multi-GPU (torchrun): every rank
runs an independent replica of the workload (weak scaling, no collective on
the data path); one all_gather of per-rank checksums after timing.

--impl reference: the CPU oracle (oracle/, plain sequential C) timed on the
host on a bounded sample of the same workload, same metric and unit.
"""
from __future__ import annotations

import argparse
import json
import os
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
SPMV_ROWS = 1 << 22
SPMV_NNZ_CUT = 65536
SPMV_FANOUT = 32
SPMV_PARTS = 148 * 8     # forest: one nnz-balanced root per worker (fn part(k, R), reading R20)
SPMV_CFG = dict(grid_size=148 * 8, block_size=128, max_tasks_per_worker=1024, max_roots=SPMV_PARTS)
CS_CFG = dict(grid_size=0, block_size=128, max_tasks_per_worker=4096, idle_backoff_ns=1024)
NQ_N = 16
NQ_CUTOFF = 7
NQ_CFG = dict(grid_size=0, block_size=128, max_tasks_per_worker=4096)
BFS_SCALE = 22
BFS_CFG = dict(grid_size=148 * 16, block_size=64, max_tasks_per_worker=1 << 18, idle_backoff_ns=1024,
               steal_max=32)  # batch steals (the paper's block-level steal takes 1): 33 -> 8.6 ms

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


# ----------------------------------------------------------------------------- ours

def _dist():
    import torch.distributed as dist
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group("nccl")
    return ws, rank, local


def _max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def bench_mergesort(args, ws, rank, dev):
    import torch

    import synth
    import paper_2604_05982_b200 as g

    n = MS_N
    pristine = synth.keys_int32(n, seed=42 + rank, device=dev)
    keys = torch.empty_like(pristine)
    scratch = torch.empty_like(pristine)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    rt = g.Runtime(g.GTAP_WORKER_THREAD, dev.index, **MS_CFG)
    table = g.Table.mergesort(keys, scratch, MS_CUTOFF, MS_MERGE_MODE)
    stream = torch.cuda.current_stream()

    def step(timed_events=None):
        keys.copy_(pristine)
        flush.fill_(1)
        rt.reset(stream)
        rt.spawn_root(table, (0, n))
        if timed_events:
            timed_events[0].record(stream)
        rt.run(stream)
        if timed_events:
            timed_events[1].record(stream)
        return rt.sync()

    for _ in range(args.warmup):
        step()
    _barrier(ws)
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    stats = []
    with ClockSampler(dev.index) as clk:
        t0 = time.perf_counter()
        for i in range(args.steps):
            stats.append(step(evs[i]))
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    _barrier(ws)
    ev_ms = [a.elapsed_time(b) for a, b in evs]           # torch events around gtap_run (incl. root/ctl H2D)
    kern_ms = [s.device_ms for s in stats]                 # runtime events around the persistent kernel only
    ms = statistics.mean(kern_ms)
    ms_max = _max_over_ranks(ms, ws)
    # correctness guard: sorted + checksum (the parity tests compare with the oracle bit for bit)
    ok = bool(torch.all(keys[1:] >= keys[:-1]).item()) and \
        int(keys.to(torch.int64).sum().item()) == int(pristine.to(torch.int64).sum().item())
    # e2e through the public API with host buffers (pinned): every step copies its 2^24 keys in,
    # sorts them and copies them out. (1) serial: H2D -> reset/spawn/run -> D2H -> sync, one step at
    # a time; (2) pipelined (double-buffered): step i+1's H2D (copy engine, stream s_in) and step
    # i-1's D2H (other copy engine, stream s_out) overlap step i's sort (compute stream); each
    # step's copies are inside the timed region, which spans all steps.
    NB = 3                                              # device/host buffers in flight
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
        host_out[0].copy_(keys, non_blocking=True)   # enqueued behind the kernel, before the host waits
        b.record(stream)
        rt.sync()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    e2e_ms = [e2e_serial() for _ in range(max(2, min(args.steps, 5)))]
    e2e_serial_ms = _max_over_ranks(statistics.mean(e2e_ms), ws)
    s_in, s_out, sc = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()  # sc: compute
    tables = [table] + [g.Table.mergesort(kb[j], scratch, MS_CUTOFF, MS_MERGE_MODE) for j in range(1, NB)]
    ksteps = max(6, args.steps)
    ev_in = [torch.cuda.Event() for _ in range(NB)]
    ev_sorted = [torch.cuda.Event() for _ in range(NB)]
    ev_out = [torch.cuda.Event() for _ in range(NB)]
    torch.cuda.synchronize()
    t_a, t_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_a.record(sc)
    s_in.wait_event(t_a)
    for i in range(ksteps + 1):
        if i < ksteps:                                  # H2D of step i
            bi = i % NB
            with torch.cuda.stream(s_in):
                if i >= NB:
                    s_in.wait_event(ev_out[bi])         # buffer bi's previous result copied out
                kb[bi].copy_(host_in[bi], non_blocking=True)
                ev_in[bi].record(s_in)
        if i >= 1:                                      # sort step i-1, then its D2H
            bj = (i - 1) % NB
            sc.wait_event(ev_in[bj])
            if i >= 2:
                rt.sync()                               # the previous run's stats (host waits here)
            rt.reset(sc)
            rt.spawn_root(tables[bj], (0, n))
            rt.run(sc)
            ev_sorted[bj].record(sc)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_sorted[bj])
                host_out[bj].copy_(kb[bj], non_blocking=True)
                ev_out[bj].record(s_out)
    rt.sync()
    sc.wait_stream(s_out)
    t_b.record(sc)
    torch.cuda.synchronize()
    e2e_pipe_ms = _max_over_ranks(t_a.elapsed_time(t_b) / ksteps, ws)
    pipe_ok = all(bool(torch.equal(host_out[j], kb[j].cpu())) for j in range(NB)) and \
        bool(torch.all(host_out[0][1:] >= host_out[0][:-1]).item())
    for t in tables[1:]:
        t.close()
    e2e_ms_max = e2e_pipe_ms
    st = stats[-1]
    algo_bytes = 8.0 * n * (1 + _ms_levels(n, MS_CUTOFF))  # read+write per key per pass
    pk, src = peaks()
    achieved = algo_bytes / (ms * 1e-3) / 1e9
    res = dict(
        value=ws * n / (ms_max * 1e-3) / 1e6, ms_per_step=ms_max, wall_ms_per_step=wall * 1e3 / args.steps,
        event_ms_per_step=statistics.mean(ev_ms),
        e2e=dict(value=ws * n / (e2e_ms_max * 1e-3) / 1e6, unit=UNIT, h2d_bytes_per_step=4 * n,
                 d2h_bytes_per_step=4 * n, ms_per_step=e2e_ms_max,
                 mode="pipelined (3 buffers: H2D / sort / D2H of consecutive steps overlap)",
                 steps=ksteps, correct=pipe_ok,
                 serial=dict(value=ws * n / (e2e_serial_ms * 1e-3) / 1e6, ms_per_step=e2e_serial_ms)),
        roofline=dict(bound="hbm", achieved=achieved, peak=pk["hbm_gbs"], unit="GB/s",
                      frac=achieved / pk["hbm_gbs"], traffic=profile_traffic("mergesort"),
                      peak_source=src, algorithmic_bytes_per_launch=algo_bytes,
                      algorithmic_bytes_per_key=8.0 * (1 + _ms_levels(n, MS_CUTOFF)),
                      note="8 B/key (read + write) for the leaf pass and each of the merge levels; the "
                           "persistent scheduler kernel is the only kernel of the step"),
        stats=dict(tasks=st.tasks, invocations=st.invocations, steals_ok=st.steals_ok, workers=st.workers,
                   grid=st.grid_size, block=st.block_size, assists=st.assists),
        correct=ok, clocks=clk.summary(), gpu_launches=args.steps,
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
                metric="Mkeys/s", value=MS_N / (t * 1e-3) / 1e6, ms=t, launch=MS0_CFG,
                span_note=f"critical path ~{2 * MS_N} sequential merge steps, {t * 1e6 / (2 * MS_N):.2f} ns/step")


def bench_fib(dev, reps=3):
    import torch

    import paper_2604_05982_b200 as g
    rt = g.Runtime(g.GTAP_WORKER_THREAD, dev.index, **FIB_CFG)
    ms = []
    st = None
    for i in range(reps + 1):
        v, st = g.fib(FIB_N, rt=rt)
        assert v == 102334155
        if i:
            ms.append(st.device_ms)
    rt.close()
    t = statistics.median(ms)
    tasks = st.tasks
    return dict(workload="fib(40) no cutoff, thread-level (configs[2])", metric="tasks/s", value=tasks / (t * 1e-3),
                ms=t, tasks=tasks, invocations=st.invocations, workers=st.workers, steals_ok=st.steals_ok,
                join_atomics=tasks - 1)


def bench_fib20(dev, reps=20):
    """BASELINE configs[0] / SURVEY §8(d) C1: fib(20) (21,891 tasks) is span-bound -- its critical path is
    2n - 1 = 39 dependent invocations -- so it is reported as tasks/s and as time per critical-path step."""
    import paper_2604_05982_b200 as g
    # a short idle backoff: at fib(20) idle warps polling for the few runnable tasks are on the critical
    # path (8192 ns cap: 0.198 ms, 1024 ns: 0.145 ms; fib(40) prefers 8192, bench_tools/fib_backoff.py)
    rt = g.Runtime(g.GTAP_WORKER_THREAD, dev.index, **dict(FIB_CFG, idle_backoff_ns=1024))
    ms = []
    st = None
    for i in range(reps + 1):
        v, st = g.fib(20, rt=rt)
        assert v == 6765
        if i:
            ms.append(st.device_ms)
    rt.close()
    t = statistics.median(ms)
    return dict(workload="fib(20) no cutoff, thread-level (configs[0]), launch + span bound", metric="tasks/s",
                value=st.tasks / (t * 1e-3), ms=t, tasks=st.tasks, invocations=st.invocations,
                us_per_critical_path_invocation=t * 1e3 / 39.0,
                note="critical path 2n-1 = 39 dependent invocations (SURVEY §8(a) A12a); includes the persistent "
                     "kernel's start and drain", launch=dict(FIB_CFG, idle_backoff_ns=1024))


def bench_epaq(dev, cutoff=10, reps=3):
    """fib(40) with cutoff 10, 1 queue vs EPAQ with 3 queues."""
    import paper_2604_05982_b200 as g
    out = {}
    for nq in (1, 3):
        with g.Runtime(g.GTAP_WORKER_THREAD, dev.index, num_queues=3, **FIB_CFG) as rt:
            ms = []
            for i in range(reps + 1):
                v, st = g.fib_cutoff(FIB_N, cutoff, nq, rt=rt)
                assert v == 102334155
                if i:
                    ms.append(st.device_ms)
        out[nq] = (statistics.median(ms), st.tasks)
    return dict(workload=f"fib(40) cutoff {cutoff}: EPAQ 3 queues vs 1 queue (NEXT #1)", metric="speedup",
                value=out[1][0] / out[3][0], ms_1q=out[1][0], ms_3q=out[3][0], tasks=out[3][1],
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


def bench_forest(dev, reps=3, arrays=16, n_each=1 << 20):
    """SURVEY §8(a) C5b on one GPU: a forest of 16 independent 2^20-key mergesorts (one root per array,
    the per-GPU shard of the 8-GPU weak-scaling configuration; BASELINE configs[4])."""
    import torch

    import synth
    import paper_2604_05982_b200 as g
    n = arrays * n_each
    pristine = torch.cat([synth.keys_int32(n_each, seed=1000 + i, device=dev) for i in range(arrays)])
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
    ok = bool(torch.all(k2[:, 1:] >= k2[:, :-1]).item()) and bool(
        torch.equal(torch.sort(pristine.view(arrays, n_each), dim=1).values, k2))
    t = statistics.median(ms)
    pk, _ = peaks()
    levels = _ms_levels(n_each, MS_CUTOFF)
    algo = 8.0 * n * (1 + levels)
    return dict(workload=f"mergesort forest {arrays} x 2^20 int32 per GPU (configs[4] C5b), thread-level, cutoff 128",
                metric="Mkeys/s", value=n / (t * 1e-3) / 1e6, ms=t, tasks=st.tasks, sorted=ok,
                roofline=dict(bound="hbm", achieved=algo / (t * 1e-3) / 1e9, peak=pk["hbm_gbs"], unit="GB/s",
                              frac=algo / (t * 1e-3) / 1e9 / pk["hbm_gbs"],
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
    return dict(workload="synthetic trees (NEXT #3), thread- vs block-level", metric="tasks/s",
                configs={k: dict(v) for k, v in TREE_CFG.items()}, points=pts)


def bench_atomics(dev):
    import torch

    import paper_2604_05982_b200 as g
    buf = torch.empty(1 << 26, dtype=torch.int32, device=dev)  # 256 MiB: words spread over L2 + HBM
    small = torch.empty(1 << 22, dtype=torch.int32, device=dev)  # 16 MiB: L2-resident
    out = {}
    grid, block, ops = 148 * 8, 256, 64
    for name, kind in (("atom_add_relaxed", 0), ("red_add", 1), ("atom_cas", 2), ("atom_min", 3),
                       ("same_address_add", 4), ("atom_add_acq_rel", 5)):
        b = small
        g.ubench_atomics(b, kind, grid, block, ops)
        ms = min(g.ubench_atomics(b, kind, grid, block, ops if kind != 4 else 4) for _ in range(3))
        nops = grid * block * (ops if kind != 4 else 4)
        out[name] = nops / (ms * 1e-3)
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
    t = _max_over_ranks(statistics.median(ms), ws)
    if ws > 1:  # the only collective: gather the y slices (outside the timed region)
        y = shard.gather_slices(y[lo:hi].contiguous(), ranges, rank)
    nnz = int(rp[-1].item())
    algo = 8.0 * nnz + 12.0 * SPMV_ROWS  # col+val per nnz; row_ptr + y + x once per row
    pk, _ = peaks()
    return dict(workload=f"SpMV power-law 2^22 rows (configs[3]), block-level, rows split over {ws} GPU(s)",
                metric="GB/s", value=algo / (t * 1e-3) / 1e9, gflops=2.0 * nnz / (t * 1e-3) / 1e9, ms=t, nnz=nnz,
                tasks=st.tasks, frac_hbm_per_gpu=algo / ws / (t * 1e-3) / 1e9 / pk["hbm_gbs"], roots=SPMV_PARTS,
                gather_floor_ms=0.50, gather_floor_note="a bare streaming gather (sum val*x[col], no rows, no "
                "scheduler) over this matrix takes 0.50 ms on B200: the random 32-B x sectors bound any CSR "
                "SpMV here (profiles/r01_spmv_gather_floor.txt)",
                traffic=profile_traffic("spmv"), scaling="strong", y_checksum=float(y.double().sum().item()))


def bench_bfs(dev, nsrc=4, ws=1, rank=0, atom_min_peak=None):
    import torch

    import synth
    import paper_2604_05982_b200 as g
    rp, col = synth.rmat_csr(BFS_SCALE, 16, seed=3, device=dev)
    depth = torch.empty(rp.numel() - 1, dtype=torch.int32, device=dev)
    rt = g.Runtime(g.GTAP_WORKER_BLOCK, dev.index, **BFS_CFG)
    # multi-GPU: the graph is replicated and the sources are split over the ranks; source 0
    # of every rank's list is a warm-up
    allsrc = synth.bfs_sources(rp, nsrc * ws, seed=5)
    srcs = [allsrc[rank * nsrc]] + allsrc[rank * nsrc: (rank + 1) * nsrc]
    res = []
    for i, s in enumerate(srcs):
        rt.reset()
        depth, st = g.bfs(rp, col, s, depth, rt=rt)
        if i == 0:
            continue
        reached = depth != 0x7FFFFFFF
        deg = (rp[1:] - rp[:-1]).to(torch.int64)
        edges = int(deg[reached].sum().item()) // 2  # undirected input edges in the component (Graph500)
        res.append((edges / (st.device_ms * 1e-3), st.device_ms, st.tasks, int(reached.sum().item())))
    rt.close()
    teps = statistics.median(r[0] for r in res)
    out = dict(workload="BFS RMAT scale 22 ef 16 (configs[4]), block-level", metric="GTEPS", value=teps / 1e9,
               ms=statistics.median(r[1] for r in res), tasks=[r[2] for r in res], reached=[r[3] for r in res],
               sources=len(res))
    if atom_min_peak:
        # L2-atomic roofline: one atom.min per scanned CSR entry; every reached vertex is
        # expanded at least once, so the scanned entries are at least 2 x the component's undirected edges
        # (a lower bound: re-expansions scan more), i.e. achieved >= 2 x TEPS
        ach = 2.0 * teps
        out["roofline"] = dict(bound="l2_atomic", achieved=ach, peak=atom_min_peak, unit="atomics/s",
                               frac=ach / atom_min_peak, peak_source="measured live: gtap_ubench_atomics atom.min",
                               note="achieved counts only the first expansion of each reached vertex (lower bound)")
    if ws > 1:  # aggregate: every rank's edges over the slowest rank's total time (no collective on the path)
        import torch.distributed as dist
        t = torch.tensor([sum(r[1] for r in res), sum(r[0] * r[1] * 1e-3 for r in res)], dtype=torch.float64,
                         device=dev)
        allv = [torch.zeros_like(t) for _ in range(ws)]
        dist.all_gather(allv, t)
        tmax = max(float(v[0]) for v in allv)
        edges = sum(float(v[1]) for v in allv)
        out.update(aggregate_gteps=edges / (tmax * 1e-3) / 1e9, sources_total=nsrc * ws, scaling="weak")
    return out


def cpu_baseline(sample_n=1 << 22, budget_s=12.0):
    """The oracle as it stands (sequential C mergesort), on the host, bounded sample."""
    import oracle
    import synth
    keys = synth.keys_int32(sample_n, seed=11).numpy()
    oracle.mergesort(keys[:1024], MS_CUTOFF)
    t_tot, reps = 0.0, 0
    while t_tot < budget_s and reps < 50:
        t0 = time.perf_counter()
        oracle.mergesort(keys, MS_CUTOFF)
        t_tot += time.perf_counter() - t0
        reps += 1
    # context for the paper's only fib ratio (GPU 2.4x faster than one CPU core at fib(40))
    t0 = time.perf_counter()
    oracle.fib(FIB_N)
    fib_s = time.perf_counter() - t0
    return dict(value=sample_n * reps / t_tot / 1e6, unit=UNIT, cores=1, kind="oracle",
                sample=f"{reps} x oracle mergesort of 2^{sample_n.bit_length() - 1} seeded int32 keys, cutoff 128",
                fib40_oracle_ms=fib_s * 1e3)


def run_ours(args):
    import torch
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    res = bench_mergesort(args, ws, rank, dev)
    secondary = []
    atom_min_peak = None
    if not args.no_secondary:
        try:
            atoms = bench_atomics(dev)
            fibr = bench_fib(dev)
            peak_atom = atoms["atom_add_acq_rel"]
            atom_min_peak = atoms.get("atom_min")
            fibr["roofline"] = dict(bound="l2_atomic", achieved=fibr["join_atomics"] / (fibr["ms"] * 1e-3),
                                    peak=peak_atom, unit="atomics/s",
                                    frac=fibr["join_atomics"] / (fibr["ms"] * 1e-3) / peak_atom,
                                    peak_source="measured live: gtap_ubench_atomics kind 5 (atom.acq_rel.add, "
                                                "distinct L2-resident sectors)")
            secondary.append(fibr)
            secondary.append(bench_fib20(dev))
            secondary.append(dict(workload="L2 atomic probes", metric="ops/s", value=atoms))
            secondary.append(bench_epaq(dev))
            secondary.append(bench_nqueens(dev))
            secondary.append(bench_mergesort_thread_merge(dev))
            secondary.append(bench_cilksort(dev))
            secondary.append(bench_forest(dev))
            secondary.append(bench_tree(dev))
        except Exception as e:  # secondary results must not kill the main line
            secondary.append(dict(workload="fib40/atomics", error=repr(e)))
        try:
            secondary.append(bench_spmv(dev, ws, rank))
        except Exception as e:
            secondary.append(dict(workload="bench_spmv", error=repr(e)))
        try:
            secondary.append(bench_bfs(dev, ws=ws, rank=rank, atom_min_peak=atom_min_peak))
        except Exception as e:
            secondary.append(dict(workload="bench_bfs", error=repr(e)))
    # the only collective: gather per-rank checksums after timing
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([1.0 if res["correct"] else 0.0], device=dev)
        allv = [torch.zeros_like(t) for _ in range(ws)]
        dist.all_gather(allv, t)
        res["correct"] = all(bool(v.item()) for v in allv)
    if rank == 0:
        pk, src = peaks()
        line = {
            "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": "mergesort 2^24 random int32 keys, thread-level fork-join, cutoff 128 "
                                   "(BASELINE configs[1])",
                       "keys_per_gpu": MS_N, "cutoff": MS_CUTOFF, "launch": MS_CFG,
                       "merge_mode": "warp (GTAP_MERGE_WARP: thread-level tasks, leaf-sort and merge bodies run "
                                     "by the task's warp, long merges shared by idle warps; same task graph -- "
                                     "the paper's one-lane merge is the secondary 'merge_mode=thread' line)",
                       "grid": res["stats"]["grid"], "block": res["stats"]["block"],
                       "workers": res["stats"]["workers"], "l2": "flushed between steps (256 MiB write)",
                       "parallelism": f"replicas x{ws} (independent roots per GPU)",
                       "timing": "persistent-kernel CUDA events (PAPER P:323); input restore, L2 flush and "
                                 "gtap_reset untimed between steps"},
            "e2e": res["e2e"], "roofline": res["roofline"], "gpu_launches": res["gpu_launches"],
            "gpu_launches_note": res["gpu_launches_note"],
            "clocks": res["clocks"], "correct": res["correct"], "stats": res["stats"],
            "wall_ms_per_step": res["wall_ms_per_step"], "event_ms_per_step": res["event_ms_per_step"],
            "secondary": secondary,
        }
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline()
            for s in line.get("secondary", []):
                if s.get("workload", "").startswith("fib(40) no cutoff") and "ms" in s:
                    s["speedup_vs_cpu_oracle"] = line["cpu_baseline"]["fib40_oracle_ms"] / s["ms"]
                    s["paper_speedup_vs_cpu_seq"] = "2.4x on GH200 vs one Grace core (P:585); context only"
                if s.get("workload", "").startswith("mergesort 2^24 cutoff 128, merge_mode=thread") and "value" in s:
                    s["speedup_vs_cpu_oracle"] = s["value"] / line["cpu_baseline"]["value"]
                    s["paper_note"] = "paper: up to 103x slower than 72-core OpenMP at n = 1e7 (P:592); context only"
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference(args):
    """The CPU oracle as it stands, timed on the host (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle
    import synth
    sample_n = 1 << 21
    keys = synth.keys_int32(sample_n, seed=11).numpy()
    for _ in range(args.warmup):
        oracle.mergesort(keys[: 1 << 16], MS_CUTOFF)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.mergesort(keys, MS_CUTOFF)
        times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    v = sample_n / t / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": "mergesort 2^24 random int32 keys, cutoff 128 (BASELINE configs[1]); "
                               "each step sorts a bounded 2^21-key sample"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"2^21 seeded int32 keys per step, {args.steps} steps"},
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
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
