"""Summarise a GPU round's captures (gpurun_out/) into profiles/ (tracked).

python tools/make_profiles.py <round-tag>
Reads gpurun_out/{launches.csv, prof_c3_full.ncu-rep, prof_roll_full.ncu-rep,
prof_image_full.ncu-rep, bench.json, bench_ref.json}; writes
profiles/<tag>_launches_c3.csv, <tag>_ncu_c3_full_summary.txt,
<tag>_ncu_rollout_summary.txt, <tag>_ncu_image_summary.txt,
<tag>_bench_c3.json, <tag>_bench_ref.json and refreshes
profiles/ncu_summary.json (the per-launch DRAM traffic bench.py reports).
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"


def run(*cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


def raw_summary(rep):
    return run(sys.executable, os.path.join(ROOT, "tools", "ncu_raw.py"), rep)


def line_summary(rep, top=25):
    src = run("ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass")
    tmp = os.path.join(G, "_src.csv")
    with open(tmp, "w") as fh:
        fh.write(src)
    return run(sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), tmp, str(top)) + \
        run(sys.executable, os.path.join(ROOT, "tools", "ncu_stalls.py"), tmp, "10")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(lambda: defaultdict(list))
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "").split("<")[0]
            v = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
                     "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}.get(unit, 1)
            per[name][d["Metric Name"]].append(v * scale)
    return per


def main():
    out = {}
    if os.path.exists(os.path.join(G, "launches.csv")):
        shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"{tag}_launches_c3.csv"))
        per = launches(os.path.join(G, "launches.csv"))
        step = 0.0
        for k, m in per.items():
            t = sum(m["gpu__time_duration.sum"]) / len(m["gpu__time_duration.sum"])
            dr = (sum(m["dram__bytes_read.sum"]) + sum(m["dram__bytes_write.sum"])) / len(m["dram__bytes_read.sum"])
            out[f"c3:{k}:ncu_us"] = t
            out[f"c3:{k}:dram_bytes_per_launch"] = dr
            step += t
        out["c3:step"] = step
        if "c3:step_main:ncu_us" in out:
            out["c3:step_main:dram_bytes_per_env"] = out["c3:step_main:dram_bytes_per_launch"] / (1 << 20)
            out["c3:step_share_step_main"] = out["c3:step_main:ncu_us"] / step
        out["note"] = (f"round {tag}: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                       "--clock-control none on tools/prof_step.py c3 100 3 (steady state, 2^20 envs; ncu serialises "
                       "the kernels, so step_rare's time is standalone: in bench.py it overlaps the next step_main)")
        with open(os.path.join(P, "ncu_summary.json"), "w") as fh:
            json.dump(out, fh, indent=1)
    for rep, name in (("prof_c3_full", "ncu_c3_full_summary"), ("prof_roll_full", "ncu_rollout_summary"),
                      ("prof_image_full", "ncu_image_summary")):
        path = os.path.join(G, rep + ".ncu-rep")
        if os.path.exists(path):
            with open(os.path.join(P, f"{tag}_{name}.txt"), "w") as fh:
                fh.write(raw_summary(path))
                fh.write("\n== source lines (stall samples / warp instructions) ==\n")
                fh.write(line_summary(path))
    for f, name in (("bench.json", "bench_c3.json"), ("bench_ref.json", "bench_ref.json")):
        path = os.path.join(G, f)
        if os.path.exists(path):
            lines = [l for l in open(path) if l.strip().startswith("{")]
            if lines:
                with open(os.path.join(P, f"{tag}_{name}"), "w") as fh:
                    fh.write(lines[-1])
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
