"""Steady-state step cost decomposition (development): device time per
VecEnv.step over steps [100, 300) with and without validation, plus the
serialised step_main / step_rare / prebuild times (xmg_profile).  Knobs via
XMG_* environment variables (XMG_PDL=0, XMG_AHEAD_EVERY=..., ...).
python tools/overhead.py [workload]"""
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
acts = random_actions(policy_keys(key_from_seed(1), n, device=dev), 0, 300)
L = _lib.lib()
knobs = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("XMG_")) or "default"
for validate in (True, False):
    vec.reset(key_from_seed(0))
    for t in range(100):
        vec.step(acts[t], validate=validate)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for t in range(100, 300):
        vec.step(acts[t], validate=validate)
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) * 1e3 / 200
    vec.reset(key_from_seed(0))
    for t in range(100):
        vec.step(acts[t], validate=validate)
    torch.cuda.synchronize()
    L.xmg_profile(1)
    for t in range(100, 164):
        vec.step(acts[t], validate=validate)
    L.xmg_profile(0)
    m, r, k = C.c_double(), C.c_double(), C.c_int64()
    L.xmg_profile_read(C.byref(m), C.byref(r), C.byref(k))
    print(f"{knobs:28s} {wl} validate={validate!s:5s}: {us:.1f} us/step; serialised step_main "
          f"{1e3 * m.value / k.value:.1f} us, step_rare {1e3 * r.value / k.value:.1f} us", flush=True)
