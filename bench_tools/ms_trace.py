"""Timeline of one 2^24 mergesort (merge_mode 1 by default) from the GTAP_MS_TRACE build.

usage: python bench_tools/ms_trace.py [merge_mode] [idle_backoff_ns]
Per (kind, size): count, first start / last end (ms from the first record), mean duration.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("GTAP_LIB", os.path.join(ROOT, "paper_2604_05982_b200", "libgtap_gtap_ms_trace.so"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_05982_b200 as g  # noqa: E402
import synth  # noqa: E402
from paper_2604_05982_b200 import gtap  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
backoff = int(sys.argv[2]) if len(sys.argv) > 2 else bench.MS_CFG["idle_backoff_ns"]
KIND = {0: "lane merge", 1: "TMA merge", 2: "leaf sort", 3: "warp assist", 4: "block assist", 5: "GPU assist",
        6: "GPU chunk", 7: "block chunk", 8: "chunk split"}
n = 1 << 24
keys = synth.keys_int32(n, seed=42, device="cuda")
scratch = torch.empty_like(keys)
L = gtap.lib()
cap = 1 << 20
buf = np.zeros((cap, 4), np.uint64)
cnt = ctypes.c_uint32()
with g.Runtime(g.GTAP_WORKER_THREAD, 0, **dict(bench.MS_CFG, idle_backoff_ns=backoff)) as rt:
    for _ in range(2):
        k2 = keys.clone()
        L.gtap_ms_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.byref(cnt))
        st = g.mergesort_(k2, scratch, 128, merge_mode=mode, rt=rt)
        L.gtap_ms_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.byref(cnt))
m = min(int(cnt.value), cap)
t0, t1 = buf[:m, 0].astype(np.int64), buf[:m, 1].astype(np.int64)
sz = (buf[:m, 2] >> np.uint64(32)).astype(np.int64)
kind = (buf[:m, 3] & np.uint64(255)).astype(np.int64)
base = t0.min()
print(f"mode={mode} backoff={backoff} kernel_ms={st.device_ms:.3f} records={m} span_ms={(t1.max() - base) / 1e6:.3f}")
for k in sorted(set(kind.tolist())):
    for size in sorted(set(sz[kind == k].tolist()), reverse=True):
        sel = (kind == k) & (sz == size)
        if sel.sum() < 1:
            continue
        d = (t1[sel] - t0[sel]) / 1e3
        print(f"{KIND[k]:12s} size={size:9d} n={sel.sum():6d} start={(t0[sel].min() - base) / 1e6:7.3f} "
              f"end={(t1[sel].max() - base) / 1e6:7.3f} ms  dur_us mean={d.mean():8.1f} max={d.max():8.1f}")

# scheduler share: warp time outside task bodies = 1 - (leaf sorts + warp-assisted merges + GPU-wide chunks, kinds
# 2, 3, 6, 7) / (workers x span); requester records 4 / 5 overlap their own chunk records and are excluded
body = float(((t1 - t0)[np.isin(kind, [2, 3, 6, 7])]).sum())
W = st.workers
span = float(t1.max() - base)
print(f"workers {W}: task-body share of warp time {body / (W * span):.3f}, scheduler + idle {1 - body / (W * span):.3f} "
      f"(span {span / 1e6:.3f} ms)")

# timeline: average number of warps busy per 50 us bin, by record class (requester records 4/5 excluded:
# their warps' chunk work is recorded as kinds 6/7)
BIN = 50_000
nb = int((t1.max() - base) // BIN) + 1
cls = {"leaf": [2], "warp merge": [3], "chunks": [6, 7]}
print("bin_us " + " ".join(f"{c:>11s}" for c in cls) + "   leaf_starts")
for b in range(nb):
    lo, hi = base + b * BIN, base + (b + 1) * BIN
    row = []
    for c, ks in cls.items():
        sel = np.isin(kind, ks)
        ov = np.clip(np.minimum(t1[sel], hi) - np.maximum(t0[sel], lo), 0, None)
        row.append(ov.sum() / BIN)
    ls = ((kind == 2) & (t0 >= lo) & (t0 < hi)).sum()
    print(f"{b * 50:6d} " + " ".join(f"{v:11.1f}" for v in row) + f"   {ls}")

# top-level merge: which warps merged its chunks, how many each, gaps between a warp's chunks
wid = (buf[:m, 3] >> np.uint64(32)).astype(np.int64)
top = (kind == 5) & (sz == sz[kind == 5].max()) if (kind == 5).any() else None
if top is not None and top.any():
    ts, te = t0[top].min(), t1[top].max()
    ch = (kind == 6) & (t0 >= ts) & (t1 <= te)
    ws = wid[ch]
    uw, cnts = np.unique(ws, return_counts=True)
    print(f"top merge {sz[top].max()} keys: {(te - ts) / 1e3:.1f} us, chunks {ch.sum()}, distinct warps {len(uw)}, "
          f"chunks/warp hist {np.bincount(cnts).tolist()}")
    first = np.array([t0[ch][ws == w].min() - ts for w in uw]) / 1e3
    print(f"  first chunk start after open: p10 {np.percentile(first, 10):.1f} p50 {np.percentile(first, 50):.1f} "
          f"p90 {np.percentile(first, 90):.1f} max {first.max():.1f} us")
    gaps = []
    for w in uw:
        sel = ch & (wid == w)
        a, b = np.sort(t0[sel]), np.sort(t1[sel])
        gaps += list((a[1:] - b[:-1]) / 1e3)
    if gaps:
        g_ = np.array(gaps)
        print(f"  gap between a warp's chunks: p50 {np.percentile(g_, 50):.2f} p90 {np.percentile(g_, 90):.2f} max {g_.max():.2f} us")
    d = (t1[ch] - t0[ch]) / 1e3
    print(f"  chunk dur p10 {np.percentile(d, 10):.1f} p50 {np.percentile(d, 50):.1f} p90 {np.percentile(d, 90):.1f} max {d.max():.1f} us")
    last = np.array([t1[ch][ws == w].max() for w in uw])
    print(f"  last chunk end before close: p10 {(te - np.percentile(last, 90)) / 1e3:.1f} p50 {(te - np.percentile(last, 50)) / 1e3:.1f} us")

# GPU-wide phase: per 20 us bin, warps merging chunks (busy) vs chunks open but unclaimed (demand); a bin with
# idle warps AND unclaimed chunks loses time to discovery, one with idle warps and no demand to the DAG
# (parents waiting for their last chunks / join-to-open latency)
req = np.where(kind == 5)[0]
if len(req):
    spl = np.where(kind == 8)[0]
    spos, st0 = (buf[spl, 2] & np.uint64(0xFFFFFFFF)).astype(np.int64), t0[spl]
    rpos = (buf[req, 2] & np.uint64(0xFFFFFFFF)).astype(np.int64)
    claims = []   # per slot: sorted claim times
    for i, j in enumerate(req):
        sel = (spos >= rpos[i]) & (spos < rpos[i] + sz[j]) & (st0 >= t0[j]) & (st0 <= t1[j])
        claims.append(np.sort(st0[sel]))
    BIN2 = 20_000
    g0 = t0[req].min()
    print("GPU phase (20 us bins): t_us  busy_chunk_warps  unclaimed_chunks  open_slots")
    for t in range(int(g0), int(t1.max()), BIN2):
        tm = t + BIN2 // 2
        openm = (t0[req] <= tm) & (t1[req] > tm)
        un = 0
        for i in np.where(openm)[0]:
            nch = (sz[req[i]] + 4095) // 4096
            un += nch - int(np.searchsorted(claims[i], tm))
        ch = (kind == 6)
        busy = ((t0[ch] <= tm) & (t1[ch] > tm)).sum() + ((kind == 8) & (t0 <= tm) & (t1 > tm)).sum()
        print(f"  {(t - base) / 1e3:8.0f} {busy:6d} {un:7d} {openm.sum():5d}")
    # join-to-open: a parent slot opens after the later of its two children's slots closed
    ends = {(int(rpos[i]), int(sz[j])): t1[j] for i, j in enumerate(req)}
    lat = {}
    for i, j in enumerate(req):
        s, p = int(sz[j]), int(rpos[i])
        c1, c2 = ends.get((p, s // 2)), ends.get((p + s // 2, s - s // 2))
        if c1 is not None and c2 is not None:
            lat.setdefault(s, []).append((t0[j] - max(c1, c2)) / 1e3)
    for s in sorted(lat):
        v = np.array(lat[s])
        print(f"  join->open size {s:9d}: n {len(v):4d} p50 {np.percentile(v, 50):6.2f} p90 {np.percentile(v, 90):6.2f} us")
