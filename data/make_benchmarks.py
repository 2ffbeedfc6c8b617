"""Materialise the benchmark rulesets used by bench.py and the GPU tests.

Run in the build container with the REFERENCE generator (out of scope to
port: offline CPU data prep, SURVEY.md §2 "Task generator"):

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python /root/repo/data/make_benchmarks.py

Writes data/<config>-<M>.xmgb in the reference's .xmgb v1 format
(ref docs/format.md) via the reference's own save_benchmark, seed 42
(ref benchgen.py:77-98).  "*-1m-style" configs of BASELINE.json are these
presets; env i runs row i mod M.
"""
import os
import sys

from rulegrid.benchgen import CONFIGS, generate_benchmark
from rulegrid.benchio import Benchmark, save_benchmark

OUT = os.path.dirname(os.path.abspath(__file__))
SIZES = {"trivial": 65536, "small": 4096, "medium": 65536, "high": 65536}

for name, m in SIZES.items():
    if len(sys.argv) > 1 and name not in sys.argv[1:]:
        continue
    tasks = generate_benchmark(CONFIGS[name], m)
    path = os.path.join(OUT, f"{name}-{m}.xmgb")
    save_benchmark(path, Benchmark(tuple(tasks), name, CONFIGS[name].random_seed))
    print(path, os.path.getsize(path), flush=True)
