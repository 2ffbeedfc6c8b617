"""Debug: run a golden case step by step and check that every pending counter
is back to zero after each (synchronised) step."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from helpers import fixture_params, fixture_rulesets, load_golden  # noqa: E402
from paper_2312_12044_b200 import Key, VecEnv  # noqa: E402

case = sys.argv[1]
fx = load_golden(case)
params = fixture_params(fx)
n = len(fx["goals"])
rulesets = fixture_rulesets(fx) if params.scenario == "xland" else None
vec = VecEnv(params, n, rulesets)
vec.reset(Key(int(fx["key"][0]), int(fx["key"][1])))
acts = torch.from_numpy(fx["actions"]).cuda()
kq = 128
qcap = max((n + 127) // 128 * 128 // 128 * 128, 128)
nch = (n + 127) // 128 * 4
for t in range(len(fx["actions"])):
    w = vec._work.cpu().numpy().view(np.uint32)
    pend = w[len(w) - 2 * nch: len(w) - nch]
    dirty = w[len(w) - nch:]
    if pend.any():
        print(f"before step {t + 1}: pending {pend} dirty {dirty} epoch {vec.epoch}", flush=True)
        cnts = w[:4 * kq].reshape(2, 2, kq)
        print("counts parity0 put", np.nonzero(cnts[0, 0])[0], cnts[0, 0][cnts[0, 0] > 0],
              "reset", np.nonzero(cnts[0, 1])[0], cnts[0, 1][cnts[0, 1] > 0])
        print("counts parity1 put", np.nonzero(cnts[1, 0])[0], cnts[1, 0][cnts[1, 0] > 0],
              "reset", np.nonzero(cnts[1, 1])[0], cnts[1, 1][cnts[1, 1] > 0])
        print("actions prev", fx["actions"][t - 1], "step_type prev", fx["step_type"][t - 1])
        break
    ts = vec.step(acts[t])
    torch.cuda.synchronize()
print("done", t)
