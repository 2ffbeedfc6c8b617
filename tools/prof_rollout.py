"""Fused-rollout timing / profiling driver.

python tools/prof_rollout.py <workload> <pre_steps> <chunk> <launches> [records 0|1] [n]
Advances `pre_steps` with one stats-only rollout, then times `launches`
rollout launches of `chunk` steps each (CUDA events per launch) and prints
them.  Under ncu: `-k regex:rollout -s 1 -c 1` captures the first timed one.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_12044_b200 import key_from_seed, policy_keys  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
pre = int(sys.argv[2]) if len(sys.argv) > 2 else 100
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 32
launches = int(sys.argv[4]) if len(sys.argv) > 4 else 4
records = int(sys.argv[5]) if len(sys.argv) > 5 else 1
n = int(sys.argv[6]) if len(sys.argv) > 6 else bench.WORKLOADS[wl][2]
dev = torch.device("cuda", 0)
params, bm, vec = bench.make_workload(wl, dev, n, 0)
vec.reset(key_from_seed(0))
pk = policy_keys(key_from_seed(1), n, device=dev)
vec.rollout(pre, policy_keys=pk, t0=0, record=())
rec = ("observations", "rewards", "discounts", "step_types") if records else ()
from paper_2312_12044_b200.vecenv import Trajectory  # noqa: E402
v = params.view_size
traj = Trajectory(torch.zeros((chunk, n, v, v, 2), dtype=torch.uint8, device=dev),
                  torch.zeros((chunk, n), dtype=torch.float32, device=dev),
                  torch.zeros((chunk, n), dtype=torch.float32, device=dev),
                  torch.zeros((chunk, n), dtype=torch.int8, device=dev)) if records else None
torch.cuda.synchronize()
t = pre
times = []
for i in range(launches):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    traj = vec.rollout(chunk, policy_keys=pk, t0=t, record=rec, out=traj)
    b.record()
    torch.cuda.synchronize()
    times.append(a.elapsed_time(b))
    t += chunk
print(f"{wl} n={n} pre={pre} chunk={chunk} records={records}: ms/launch",
      " ".join(f"{x:.3f}" for x in times), "| us/step", " ".join(f"{1e3 * x / chunk:.1f}" for x in times),
      "| Gsteps/s", " ".join(f"{n * chunk / x / 1e6:.2f}" for x in times))
