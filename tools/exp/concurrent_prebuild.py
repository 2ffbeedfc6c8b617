"""Timing experiment (unsafe: races are ignored): the steady-state step with
the reset-ahead batches launched on a side stream, concurrent with the steps,
against batches launched in line (the library default) and no batches.
Run with XMG_AHEAD_EVERY=100000 so xmg_step itself launches none in the window.
python tools/exp/concurrent_prebuild.py [every] [prio]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_12044_b200 import _lib, key_from_seed, policy_keys, random_actions  # noqa: E402

every = int(sys.argv[1]) if len(sys.argv) > 1 else 16
prio = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dev = torch.device("cuda", 0)
n = bench.WORKLOADS["c3"][2]
params, bm, vec = bench.make_workload("c3", dev, n, 0)
acts = random_actions(policy_keys(key_from_seed(1), n, device=dev), 0, 300)
L = _lib.lib()
B = max(1, (params.step_budget - 2) // every)
side = torch.cuda.Stream(device=dev, priority=prio)
for mode in ("none", "inline", "side"):
    vec.reset(key_from_seed(0))
    for t in range(100):
        vec.step(acts[t])
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = torch.cuda.current_stream(dev)
    s.record()
    for t in range(100, 300):
        if t % every == 0 and mode != "none":
            st = side if mode == "side" else main
            if mode == "side":
                side.wait_stream(main)  # the batch starts after the steps before it were enqueued
            _lib.check(L.xmg_prebuild(vec._desc_ref, vec._state_ref, (t // every) % B, B, n, st.cuda_stream),
                       "xmg_prebuild")
        vec.step(acts[t])
    e.record()
    main.wait_stream(side)
    torch.cuda.synchronize()
    print(f"every={every} prio={prio} {mode:6s}: {s.elapsed_time(e) * 1e3 / 200:.1f} us/step", flush=True)
