"""Per-warp phase times of step_rare from a -DXMG_TRACE build (XMG_LIB=...)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_12044_b200 import _lib, key_from_seed, policy_keys, random_actions  # noqa: E402

wl, pre = sys.argv[1], int(sys.argv[2])
n = bench.WORKLOADS[wl][2]
dev = torch.device("cuda", 0)
params, bm, vec = bench.make_workload(wl, dev, n, 0)
vec.reset(key_from_seed(0))
acts = random_actions(policy_keys(key_from_seed(1), n, device=dev), 0, pre + 1)
for t in range(pre):
    vec.step(acts[t], validate=False)
torch.cuda.synchronize()
L = _lib.lib()
L.xmg_debug_trace_clear()
torch.cuda.synchronize()
vec.step(acts[pre], validate=False)
torch.cuda.synchronize()
rows = 1 << 16
buf = np.zeros((rows, 24), np.uint64)
L.xmg_debug_trace.argtypes = [C.c_void_p, C.c_int64]
L.xmg_debug_trace(buf.ctypes.data, rows)
act = buf[:, 0] > 0
t0 = buf[act, 0].min()
work = act & (buf[:, 2] > 0)
print(f"warps started {act.sum()}, with work {work.sum()}")
st = (buf[work, 0].astype(np.int64) - int(t0)) / 1e3
p1 = (buf[work, 1].astype(np.int64) - int(t0)) / 1e3
p2 = (buf[work, 2].astype(np.int64) - int(t0)) / 1e3
cnt = buf[work, 3]
print(f"start max {st.max():.1f} us; PUT phase end: median {np.median(p1):.1f} max {p1.max():.1f}; "
      f"all done: median {np.median(p2):.1f} max {p2.max():.1f} us")
put_dur = p1 - st
res_dur = p2 - p1
print(f"PUT phase duration: median {np.median(put_dur):.1f} p90 {np.percentile(put_dur, 90):.1f} max {put_dur.max():.1f}")
print(f"reset phase duration: median {np.median(res_dur):.1f} p90 {np.percentile(res_dur, 90):.1f} max {res_dur.max():.1f}")
for i in np.argsort(-(p2 - st))[:6]:
    print(f"  start {st[i]:.1f} put_end {p1[i]:.1f} end {p2[i]:.1f} cnt_put {int(cnt[i]) & 0xffffffff} "
          f"cnt_reset {int(cnt[i]) >> 32}")
sub = work & (buf[:, 4] > 0) & (buf[:, 5] > 0) & (buf[:, 6] > 0)
if sub.any():
    b0 = buf[sub, 0].astype(np.int64)
    pf = (buf[sub, 4].astype(np.int64) - b0) / 1e3
    e1 = (buf[sub, 5].astype(np.int64) - buf[sub, 4].astype(np.int64)) / 1e3
    rest = (buf[sub, 6].astype(np.int64) - buf[sub, 5].astype(np.int64)) / 1e3
    for nm, x in (("prefetch", pf), ("first env", e1), ("rest of batch", rest)):
        print(f"{nm:14s}: median {np.median(x):.2f} p90 {np.percentile(x, 90):.2f} max {x.max():.2f} us")
rs = work & (buf[:, 7] > 0) & (buf[:, 2] > buf[:, 1])
if rs.any():
    kd = (buf[rs, 7].astype(np.int64) - buf[rs, 1].astype(np.int64)) / 1e3
    bd = (buf[rs, 2].astype(np.int64) - buf[rs, 7].astype(np.int64)) / 1e3
    print(f"reset keys    : median {np.median(kd):.2f} max {kd.max():.2f}; build+obs: median {np.median(bd):.2f} max {bd.max():.2f} us")
wb = work & (buf[:, 8] > 0) & (buf[:, 14] > 0)
if wb.any():
    names = ["keys/setup", "free list", "draws", "rank/place", "copy out", "obs"]
    prev = buf[wb, 8].astype(np.int64)
    for k in range(1, 7):
        cur = buf[wb, 8 + k].astype(np.int64)
        dt = (cur - prev) / 1e3
        print(f"build {names[k - 1]:11s}: median {np.median(dt):.2f} max {dt.max():.2f} us")
        prev = cur
wr = work & (buf[:, 11] > 0) & (buf[:, 16] > 0) & (buf[:, 21] > 0)
if wr.any():
    names = ["doors", "a-words..", "zero+hist", "scan", "scatter", "ranks"]
    cols = [11, 16, 17, 18, 19, 20, 21]
    for k in range(1, len(cols)):
        dt = (buf[wr, cols[k]].astype(np.int64) - buf[wr, cols[k - 1]].astype(np.int64)) / 1e3
        print(f"rank {names[k - 1]:10s}: median {np.median(dt):.2f} max {dt.max():.2f} us")
