"""Drive a workload to a given step for profiling (ncu -k regex:step_).

python tools/prof_step.py <workload> <pre_steps> <steps> [n]
Each step launches step_main and step_rare (validation off), after one reset
launch of step_rare, so `ncu -k regex:step_ -s <1 + 2*pre_steps> -c <2*k>`
captures k steps of the tail.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_12044_b200 import key_from_seed, policy_keys, random_actions  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 100
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n = int(sys.argv[4]) if len(sys.argv) > 4 else bench.WORKLOADS[wl][2]
dev = torch.device("cuda", 0)
params, bm, vec = bench.make_workload(wl, dev, n, 0)
vec.reset(key_from_seed(0))
acts = random_actions(policy_keys(key_from_seed(1), n, device=dev), 0, pre + steps)
for t in range(pre + steps):
    vec.step(acts[t], validate=False)
torch.cuda.synchronize()
print("done", wl, n, pre, steps)
