"""Device time per step in windows of a long run (fill / steady / burst / refill).
python tools/step_windows.py <run> [steps]   (runs from tools/quick_time.RUNS)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import benchmark_file  # noqa: E402
from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions  # noqa
from quick_time import RUNS  # noqa: E402

name = sys.argv[1]
env_name, config, n, _ = RUNS[name]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1100
spare = False
_, params = make(env_name)
vec = VecEnv(params, n, load_benchmark(benchmark_file(config)) if config else None, reuse_outputs=True)
vec.reset(key_from_seed(0))
acts = random_actions(policy_keys(key_from_seed(1), n, device="cuda"), 0, steps)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
torch.cuda.synchronize()
ev[0].record()
for t in range(steps):
    vec.step(acts[t], True, False)
    ev[t + 1].record()
torch.cuda.synchronize()
dt = np.array([ev[t].elapsed_time(ev[t + 1]) * 1e3 for t in range(steps)])
b = params.step_budget
wins = [(0, 20), (20, 170), (170, b - 2), (b - 2, b + 2), (b + 2, b + 40), (b + 40, min(b + 200, steps)),
        (min(b + 200, steps), steps)]
print(f"{name} spare={int(spare)} n={n} budget={b} total {dt.sum() / 1e3:.2f} ms mean {dt.mean():.1f} us/step")
for lo, hi in wins:
    if hi > lo:
        print(f"  steps [{lo:5d},{hi:5d}): mean {dt[lo:hi].mean():8.1f} us  median {np.median(dt[lo:hi]):8.1f}  max {dt[lo:hi].max():8.1f}")
