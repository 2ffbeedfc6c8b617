"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA line:
stall samples and warp-level instructions executed.  Usage:
  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
  python tools/ncu_lines.py s.csv [topN]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
agg = defaultdict(lambda: [0, 0, 0, ""])
cur = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        i_st = hdr.index("Warp Stall Sampling (All Samples)")
        i_ie = hdr.index("Instructions Executed")
        i_ti = hdr.index("Thread Instructions Executed")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] not in ("", None):
        cur = int(r[0]) if r[0].isdigit() else cur
        if cur is not None:
            agg[cur][3] = r[1][:90]
        continue
    if cur is None:
        continue
    try:
        agg[cur][0] += int(r[i_st] or 0)
        agg[cur][1] += int(r[i_ie] or 0)
        agg[cur][2] += int(r[i_ti] or 0)
    except ValueError:
        pass
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
for ln, (s, ie, ti, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:5d} stall {100*s/tot_s:5.1f}%  inst {100*ie/tot_i:5.1f}%  thr/inst {ti/max(ie,1):5.1f}  {src}")
