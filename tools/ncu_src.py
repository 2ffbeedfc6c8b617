"""Per (file, line) totals from an ncu source page exported with
  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass -k regex:<kernel> > s.csv
python tools/ncu_src.py s.csv [topN] [sort: inst|stall]
Prints warp instructions executed and stall samples per CUDA source line."""
import csv
import os
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
key = sys.argv[3] if len(sys.argv) > 3 else "inst"
agg = defaultdict(lambda: [0, 0, ""])
fname, hdr, cur = "?", None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        i_st = hdr.index("Warp Stall Sampling (All Samples)")
        i_ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        cur = (fname, int(r[0])) if r[0].isdigit() else None
        if cur is not None:
            agg[cur][2] = r[1].strip()[:80]
        continue
    if cur is None:
        continue
    try:
        agg[cur][0] += int(r[i_st] or 0)
        agg[cur][1] += int(r[i_ie] or 0)
    except ValueError:
        pass
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total: stall samples {ts}, warp instructions {ti}")
k = 1 if key == "inst" else 0
for (f, ln), (s, ie, src) in sorted(agg.items(), key=lambda kv: -kv[1][k])[:top]:
    print(f"{f:16s}{ln:5d}  inst {100 * ie / ti:5.1f}%  stall {100 * s / ts:5.1f}%  {src}")
