"""Per-workload DRAM traffic of step_main / step_rare for bench.py's `traffic`.

Reads gpurun_out/launches_<wl>.csv (ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --clock-control none on
tools/prof_step.py <wl> 100 3) for each workload given, merges
"<wl>:<kernel>:ncu_us" / ":dram_bytes_per_launch" / "<wl>:step_main:
dram_bytes_per_env" into profiles/ncu_summary.json (other keys kept), copies
each launch list to profiles/<tag>_launches_<wl>.csv and the summary to
gpurun_out/ncu_summary.json.

python tools/ncu_workloads.py <tag> <wl> [<wl> ...]
"""
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from make_profiles import launches  # noqa: E402

import bench  # noqa: E402

G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def main():
    tag, wls = sys.argv[1], sys.argv[2:]
    path = os.path.join(P, "ncu_summary.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for wl in wls:
        src = os.path.join(G, f"launches_{wl}.csv")
        if not os.path.exists(src):
            print("missing", src)
            continue
        shutil.copy(src, os.path.join(P, f"{tag}_launches_{wl}.csv"))
        for k, m in launches(src).items():
            if not m.get("dram__bytes_read.sum"):
                continue
            t = sum(m["gpu__time_duration.sum"]) / len(m["gpu__time_duration.sum"])
            dr = (sum(m["dram__bytes_read.sum"]) + sum(m["dram__bytes_write.sum"])) / len(m["dram__bytes_read.sum"])
            out[f"{wl}:{k}:ncu_us"] = t
            out[f"{wl}:{k}:dram_bytes_per_launch"] = dr
            if k == "step_main":
                out[f"{wl}:step_main:dram_bytes_per_env"] = dr / bench.WORKLOADS[wl][2]
    out["note_workloads"] = (f"round {tag}: the same ncu launch-list pass on tools/prof_step.py <wl> 100 3 for "
                             "each workload key (steady state at the workload's bench size)")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    os.makedirs(G, exist_ok=True)
    shutil.copy(path, os.path.join(G, "ncu_summary.json"))
    print(json.dumps({k: v for k, v in out.items() if k.split(":")[0] in wls}, indent=1))


if __name__ == "__main__":
    main()
