"""Device time of one reset-ahead batch (xmg_prebuild) at a workload's size:
python tools/time_prebuild.py [workload] [classes] [reps]
(XMG_LIB selects a library variant)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_12044_b200 import _lib, key_from_seed  # noqa: E402
from paper_2312_12044_b200.vecenv import STAGE_BITS  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
dev = torch.device("cuda", 0)
params, bm, vec = bench.make_workload(wl, dev, bench.WORKLOADS[wl][2], 0)
every, classes = C.c_int64(), C.c_int64()
_lib.lib().xmg_ahead_plan(C.byref(vec._desc), vec.num_envs, C.byref(every), C.byref(classes))
B = int(sys.argv[2]) if len(sys.argv) > 2 else classes.value
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
vec.reset(key_from_seed(0))
stream = torch.cuda.current_stream(dev).cuda_stream
L = _lib.lib()
times = []
for r in range(reps + 1):
    vec.agent[:, 0] &= ~STAGE_BITS
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    _lib.check(L.xmg_prebuild(vec._desc_ref, vec._state_ref, r % B, B, vec.num_envs, stream), "xmg_prebuild")
    e.record()
    torch.cuda.synchronize()
    if r:
        times.append(s.elapsed_time(e) * 1e3)
    assert int(((vec.agent[r % B::B, 0] >> 18) & 3).min()) == 2
builds = (vec.num_envs + B - 1) // B
t = sorted(times)[len(times) // 2]
print(f"{os.environ.get('XMG_LIB', 'default')[-24:]:24s} {wl} every={every.value} classes={B}: batch of {builds} "
      f"builds {t:.1f} us = {t * 1e3 / builds:.2f} ns/build", flush=True)
