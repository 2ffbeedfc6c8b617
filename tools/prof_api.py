"""Drive VecEnv.step through the public API (validation on) for profiling."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_12044_b200 import key_from_seed, policy_keys, random_actions  # noqa: E402

wl, pre, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
n = bench.WORKLOADS[wl][2]
dev = torch.device("cuda", 0)
params, bm, vec = bench.make_workload(wl, dev, n, 0)
vec.reset(key_from_seed(0))
acts = random_actions(policy_keys(key_from_seed(1), n, device=dev), 0, pre + steps)
for t in range(pre + steps):
    vec.step(acts[t])
torch.cuda.synchronize()
print("done")
