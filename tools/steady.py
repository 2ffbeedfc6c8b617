"""Device time per VecEnv.step in a burst-free steady-state window and in a
window across the synchronized budget reset (development timing; knobs via
the XMG_* environment variables).
python tools/steady.py <workload> [pre] [steps] [envs]"""
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
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
n = int(sys.argv[4]) if len(sys.argv) > 4 else bench.WORKLOADS[wl][2]
dev = torch.device("cuda", 0)
params, bm, vec = bench.make_workload(wl, dev, n, 0)
b = params.step_budget
total = max(pre + steps, b + 12)
acts = random_actions(policy_keys(key_from_seed(1), n, device=dev), 0, total)


def window(t0, k):
    vec.reset(key_from_seed(0))
    for t in range(t0):
        vec.step(acts[t])
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for t in range(t0, t0 + k):
        vec.step(acts[t])
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / k


knobs = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("XMG_"))
st = window(pre, steps)
bu = window(b - 10, 20)
print(f"{wl} n={n} {knobs or 'default'}: steady [{pre},{pre + steps}) {st:.1f} us/step "
      f"({n / st / 1e3:.3f} G/s); burst [{b - 10},{b + 10}) {bu:.1f} us/step ({n / bu / 1e3:.3f} G/s)", flush=True)
