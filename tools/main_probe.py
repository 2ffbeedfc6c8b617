"""step_main / step_rare standalone times (xmg_profile, serialised) at a
workload's steady state, with and without observations (development).
python tools/main_probe.py [workload]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_12044_b200 import _lib, key_from_seed, policy_keys, random_actions  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
dev = torch.device("cuda", 0)
n = bench.WORKLOADS[wl][2]
params, bm, vec = bench.make_workload(wl, dev, n, 0)
acts = random_actions(policy_keys(key_from_seed(1), n, device=dev), 0, 200)
L = _lib.lib()
for obs in (True, False):
    vec.reset(key_from_seed(0))
    for t in range(100):
        vec.step(acts[t], compute_obs=obs, validate=False)
    torch.cuda.synchronize()
    L.xmg_profile(1)
    for t in range(100, 150):
        vec.step(acts[t], compute_obs=obs, validate=False)
    L.xmg_profile(0)
    m, r, k = C.c_double(), C.c_double(), C.c_int64()
    L.xmg_profile_read(C.byref(m), C.byref(r), C.byref(k))
    print(f"{os.environ.get('XMG_LIB', 'default')[-22:]:22s} {wl} obs={obs}: step_main {1e3 * m.value / k.value:.1f} us, "
          f"step_rare {1e3 * r.value / k.value:.1f} us", flush=True)
