"""Summarise a GPU session's captures (tools/gpu_session.sh <tag>, in
gpurun_out/) into profiles/ (tracked).

python tools/make_profiles.py <tag>
Writes profiles/<tag>_bench_<wl>.json (the bench lines), <tag>_launches_*.csv
(ncu launch lists: the driver's bench command over its timed window, and
tools/prof_step.py <wl> 100 3 per workload), <tag>_ncu_<what>_summary.txt
(raw metrics + per-source-line instructions / stalls of each --set full
capture) and refreshes profiles/ncu_summary.json (the per-launch DRAM traffic
bench.py reports as roofline.traffic).
"""
import csv
import glob
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
WL_ENVS = {"c1": 1024, "c2": 1 << 16, "c3": 1 << 20, "c4": 1 << 19, "doorkey": 1 << 20}


def run(*cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


def launches(path):
    """{kernel: {metric: [values per launch, in us / bytes]}} of an ncu CSV launch list."""
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
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
                     "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}.get(d["Metric Unit"], 1)
            per[name][d["Metric Name"]].append(v * scale)
    return per


def window_launches(path, before=10, steps=20):
    """The launches of the driver's timed window in a launch list of
    `bench.py --steps 20 --warmup 5`: the 20 steps around the budget-reset
    burst (the longest step_main before the statistics reduction), 10 before
    it, the burst step and 9 after, with every kernel launched between."""
    rows = list(csv.reader(open(path)))
    hdr, seq = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "").split("<")[0]
            seq.append((name, float(d["Metric Value"].replace(",", "")) / 1e3))  # ns -> us
    end = next((i for i, (k, _) in enumerate(seq) if "reduce" in k), len(seq))
    mains = [i for i, (k, _) in enumerate(seq[:end]) if k == "step_main"]
    burst = max(mains, key=lambda i: seq[i][1])
    b = mains.index(burst)
    first, last = mains[max(0, b - before)], mains[min(len(mains) - 1, b - before + steps - 1)]
    stop = next((i for i in range(last + 1, end) if seq[i][0] in ("step_main", "validate_kernel", "prebuild_kernel")),
                end)
    per = defaultdict(lambda: defaultdict(list))
    for k, t in seq[first:stop]:
        per[k]["gpu__time_duration.sum"].append(t)
    return per


def full_summary(rep, kernel_regex=None, top=30):
    out = run(sys.executable, os.path.join(ROOT, "tools", "ncu_raw.py"), rep)
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel_regex:
        cmd += ["-k", f"regex:{kernel_regex}"]
    src = run(*cmd)
    tmp = os.path.join(G, "_src.csv")
    with open(tmp, "w") as fh:
        fh.write(src)
    out += f"\n== per source line ({kernel_regex or 'all kernels'}): warp instructions / stall samples ==\n"
    out += run(sys.executable, os.path.join(ROOT, "tools", "ncu_src.py"), tmp, str(top), "inst")
    out += "\n== stall reasons ==\n" + run(sys.executable, os.path.join(ROOT, "tools", "ncu_stalls.py"), tmp, "8")
    return out


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    os.makedirs(P, exist_ok=True)
    # bench lines
    for path in sorted(glob.glob(os.path.join(G, f"{tag}_bench_*.json"))):
        lines = [ln for ln in open(path) if ln.strip().startswith("{")]
        if lines:
            with open(os.path.join(P, os.path.basename(path)), "w") as fh:
                fh.write(lines[-1])
    # launch lists: the driver's command, and the per-workload steady-state pass
    summary_path = os.path.join(P, "ncu_summary.json")
    summ = {}
    src = os.path.join(G, f"{tag}_launches_bench_c3_k20.csv")
    if os.path.exists(src):
        shutil.copy(src, os.path.join(P, os.path.basename(src)))
        per = window_launches(src)
        tot = sum(sum(m["gpu__time_duration.sum"]) for m in per.values())
        summ["bench_c3_k20:share"] = {k: sum(m["gpu__time_duration.sum"]) / tot for k, m in per.items()}
        summ["bench_c3_k20:launches"] = {k: len(m["gpu__time_duration.sum"]) for k, m in per.items()}
        summ["bench_c3_k20:mean_us"] = {k: sum(m["gpu__time_duration.sum"]) / len(m["gpu__time_duration.sum"])
                                       for k, m in per.items()}
    for wl, nenv in WL_ENVS.items():
        src = os.path.join(G, f"launches_{wl}.csv")
        if not os.path.exists(src):
            continue
        shutil.copy(src, os.path.join(P, f"{tag}_launches_{wl}.csv"))
        for k, m in launches(src).items():
            if not m.get("dram__bytes_read.sum"):
                continue
            t = sum(m["gpu__time_duration.sum"]) / len(m["gpu__time_duration.sum"])
            dr = (sum(m["dram__bytes_read.sum"]) + sum(m["dram__bytes_write.sum"])) / len(m["dram__bytes_read.sum"])
            summ[f"{wl}:{k}:ncu_us"] = t
            summ[f"{wl}:{k}:dram_bytes_per_launch"] = dr
            if k == "step_main":
                summ[f"{wl}:step_main:dram_bytes_per_env"] = dr / nenv
    summ["note"] = (f"round {tag} (tools/gpu_session.sh): <wl>:<kernel>:* from ncu --metrics gpu__time_duration.sum,"
                    "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none on tools/prof_step.py <wl> 100 3 "
                    "(steady state, the workload's bench size; ncu serialises the kernels); bench_c3_k20:* from the "
                    "launch list of the driver's command (python bench.py --steps 20 --warmup 5) over its timed "
                    "window: each kernel's share of the serialised device time")
    with open(summary_path, "w") as fh:
        json.dump(summ, fh, indent=1)
    # --set full captures
    for rep, what, regex in (("c3_steady", "c3_step_main_steady", "step_main"),
                             ("c3_steady", "c3_step_rare_steady", "step_rare"),
                             ("c3_burst", "c3_step_main_burst", "step_main"),
                             ("c3_prebuild", "c3_prebuild", "prebuild"),
                             ("c3_rollout", "c3_rollout", "rollout"),
                             ("image", "image", "image_kernel")):
        path = os.path.join(G, f"{tag}_{rep}.ncu-rep")
        if os.path.exists(path):
            with open(os.path.join(P, f"{tag}_ncu_{what}_summary.txt"), "w") as fh:
                fh.write(full_summary(path, regex))
    print(json.dumps(summ, indent=1)[:3000])


if __name__ == "__main__":
    main()
