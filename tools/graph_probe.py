"""Small-batch step cost breakdown (development): host time per call and
device time per step of the graph path vs the two-kernel path.
python tools/graph_probe.py <workload> [steps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2312_12044_b200 import key_from_seed, policy_keys, random_actions  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
dev = torch.device("cuda", 0)
n = bench.WORKLOADS[wl][2]
for graph in (True, False):
    params, bm, vec = bench.make_workload(wl, dev, n, 0, graph=graph)
    vec.reset(key_from_seed(0))
    acts = random_actions(policy_keys(key_from_seed(1), n, device=dev), 0, steps + 20)
    for t in range(20):
        vec.step(acts[t])
    torch.cuda.synchronize()
    # host cost per call with the staging copy, and with in-place actions
    t0 = time.perf_counter()
    for t in range(20, 20 + steps):
        vec.step(acts[t])
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    line = f"{wl} n={n} graph={graph}: host {1e6 * (t1 - t0) / steps:.1f} us/call, wall {1e6 * (t2 - t0) / steps:.1f} us/step"
    if graph:
        buf = vec.action_buffer
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for t in range(steps):
            vec.step(buf)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        line += f"; in-place actions: host {1e6 * (t1 - t0) / steps:.1f} us/call, wall {1e6 * (t2 - t0) / steps:.1f} us/step"
    print(line, flush=True)
