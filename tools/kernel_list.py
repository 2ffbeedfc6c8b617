"""Print ncu per-kernel times for a few steps of a workload (launch list)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
            per[name].append(float(d["Metric Value"]) / 1e3)
for k, v in per.items():
    print(f"{k:40s} n={len(v):3d} mean={sum(v)/len(v):8.2f} us  min={min(v):8.2f} max={max(v):8.2f}")
