"""Stall reasons per CUDA source line from an ncu source page CSV
(ncu -i X --page source --csv --print-source cuda,sass > s.csv).
python tools/ncu_stalls.py s.csv [topN]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
hdr = None
agg = defaultdict(lambda: defaultdict(float))
src = {}
cur = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] not in ("", None):
        cur = int(r[0]) if r[0].isdigit() else cur
        if cur is not None:
            src[cur] = r[1][:70]
        continue
    if cur is None:
        continue
    for i in cols:
        try:
            agg[cur][hdr[i][6:]] += float(r[i] or 0)
        except ValueError:
            pass
tot = defaultdict(float)
for a in agg.values():
    for k, v in a.items():
        tot[k] += v
T = sum(tot.values()) or 1
print("overall:", ", ".join(f"{k} {v / T * 100:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:10]))
for ln in sorted(agg, key=lambda l: -sum(agg[l].values()))[:top]:
    a = agg[ln]
    s = sum(a.values()) or 1
    print(f"{ln:5d} {s / T * 100:5.1f}% {src.get(ln, '')[:60]:60s} | " +
          ", ".join(f"{k} {v / s * 100:.0f}%" for k, v in sorted(a.items(), key=lambda x: -x[1])[:4]))
