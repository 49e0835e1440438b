"""Pipelined e2e of the bench (3 buffers, H2D / sort / D2H on separate streams): per-run kernel
time (gtap stats) vs the step time, with and without the copies, to see whether the copies slow the
sort (L2 pollution by the DMA traffic) or host round trips leave bubbles."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402

n = bench.MS_N
NB = 3
pristine = synth.keys_int32(n, seed=42, device="cuda")
scratch = torch.empty_like(pristine)
kb = [torch.empty_like(pristine) for _ in range(NB)]
host_in = [pristine.cpu().pin_memory() for _ in range(NB)]
host_out = [torch.empty_like(host_in[0]).pin_memory() for _ in range(NB)]
rt = g.Runtime(g.GTAP_WORKER_THREAD, 0, **bench.MS_CFG)
tables = [g.Table.mergesort(kb[j], scratch, bench.MS_CUTOFF, bench.MS_MERGE_MODE) for j in range(NB)]
s_in, s_out, sc = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def run(copies, ksteps=8):
    ev_in = [torch.cuda.Event() for _ in range(NB)]
    ev_sorted = [torch.cuda.Event() for _ in range(NB)]
    ev_out = [torch.cuda.Event() for _ in range(NB)]
    dev_ms = []
    torch.cuda.synchronize()
    t_a, t_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_a.record(sc)
    s_in.wait_event(t_a)
    for i in range(ksteps + 1):
        if i < ksteps:
            bi = i % NB
            with torch.cuda.stream(s_in):
                if i >= NB:
                    s_in.wait_event(ev_out[bi])
                if copies:
                    kb[bi].copy_(host_in[bi], non_blocking=True)
                else:
                    kb[bi].copy_(pristine, non_blocking=True)
                ev_in[bi].record(s_in)
        if i >= 1:
            bj = (i - 1) % NB
            sc.wait_event(ev_in[bj])
            if i >= 2:
                dev_ms.append(rt.sync().device_ms)
            rt.reset(sc)
            rt.spawn_root(tables[bj], (0, n))
            rt.run(sc)
            ev_sorted[bj].record(sc)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_sorted[bj])
                if copies:
                    host_out[bj].copy_(kb[bj], non_blocking=True)
                ev_out[bj].record(s_out)
    dev_ms.append(rt.sync().device_ms)
    sc.wait_stream(s_out)
    t_b.record(sc)
    torch.cuda.synchronize()
    return t_a.elapsed_time(t_b) / ksteps, statistics.mean(dev_ms)


for copies in (True, False, True, False):
    step, k = run(copies)
    print(f"copies={copies!s:5s} step {step:.3f} ms  kernel {k:.3f} ms  -> {n / step / 1e3:.0f} Mkeys/s", flush=True)

# copies only: 64 MB H2D and 64 MB D2H on two streams at once (no sort), 8 rounds
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s_in)
s_out.wait_event(a)
for i in range(8):
    with torch.cuda.stream(s_in):
        kb[i % NB].copy_(host_in[i % NB], non_blocking=True)
    with torch.cuda.stream(s_out):
        host_out[(i + 1) % NB].copy_(kb[(i + 1) % NB], non_blocking=True)
s_in.wait_stream(s_out)
b.record(s_in)
torch.cuda.synchronize()
t = a.elapsed_time(b) / 8
print(f"concurrent H2D + D2H of 64 MB each: {t:.3f} ms per pair -> {2 * 4 * n / t / 1e6:.1f} GB/s aggregate", flush=True)
