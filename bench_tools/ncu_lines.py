"""Per-source-line / per-region warp-stall breakdown from an ncu report's source page.

usage: ncu -i REP --page source --csv --print-source cuda,sass > x.csv; python bench_tools/ncu_lines.py x.csv [file:lo-hi ...]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
regions = []
for a in sys.argv[2:]:
    f, rg = a.split(":")
    lo, hi = rg.split("-")
    regions.append((f, int(lo), int(hi)))
hdr = None
f = None
per = collections.defaultdict(collections.Counter)
tot = collections.Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        idx = {h: i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
        continue
    if hdr is None or r[0] in ("", "Function Name") or r[2] != "-":
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    key = f"{f}:other"
    for (rf, lo, hi) in regions:
        if rf == f and lo <= ln <= hi:
            key = f"{rf}:{lo}-{hi}"
    for h, i in idx.items():
        try:
            v = float(r[i] or 0)
        except ValueError:
            v = 0
        per[key][h] += v
        tot[h] += v
T = sum(tot.values())
print(f"total samples {T:.0f}")
for k, c in sorted(per.items(), key=lambda kv: -sum(kv[1].values())):
    s = sum(c.values())
    if s < 0.01 * T:
        continue
    top = ", ".join(f"{h[6:]} {100 * v / s:.0f}%" for h, v in c.most_common(5))
    print(f"{100 * s / T:5.1f}% {k:32s} {top}")
