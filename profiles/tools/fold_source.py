"""Fold `ncu -i REP --page source --csv --print-source cuda,sass` output per CUDA
source line: share of SASS instructions executed and of warp stall samples.
usage: python fold_source.py SOURCE.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
path = None
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or len(r) < 8:
        continue
    try:
        ie = float(r[hdr.index("Instructions Executed")])
        st = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    k = (path, int(r[0]))
    a = agg.setdefault(k, [0.0, 0.0, r[1].strip()[:90]])
    a[0] += ie
    a[1] += st
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {ti:.0f}, stall samples {ts:.0f}")
for (f, ln), (ie, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f:16s} {ln:5d} {100 * ie / ti:5.1f}% {100 * st / ts:5.1f}%  {src}")
