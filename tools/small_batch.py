"""Per-call step cost across batch sizes: VecEnv.step (step_main + step_rare,
validated or not) against a one-step block in the fused kernel
(VecEnv.steps(actions[t:t+1]), xmg_rollout with T = 1).
python tools/small_batch.py [c3|doorkey] [log2 sizes...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from helpers import benchmark_file  # noqa: E402
from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions  # noqa

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
sizes = [int(x) for x in sys.argv[2:]] or [10, 12, 14, 16, 18, 20]
env_name, config = {"c3": ("XLand-MiniGrid-R4-13x13", "medium"), "doorkey": ("MiniGrid-DoorKey-8x8", None)}[wl]
_, params = make(env_name)
bm = load_benchmark(benchmark_file(config)) if config else None
steps = 300
for lg in sizes:
    n = 1 << lg
    res = {}
    for mode in ("step", "step_nv", "fused1"):
        vec = VecEnv(params, n, bm, reuse_outputs=True)
        vec.reset(key_from_seed(0))
        acts = random_actions(policy_keys(key_from_seed(1), n, device="cuda"), 0, steps + 10)
        for t in range(10):
            vec.step(acts[t])
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for t in range(10, 10 + steps):
            if mode == "step":
                vec.step(acts[t])
            elif mode == "step_nv":
                vec.step(acts[t], validate=False)
            else:
                vec.steps(acts[t:t + 1], validate=False)
        e.record()
        torch.cuda.synchronize()
        vec.check()
        res[mode] = s.elapsed_time(e) / steps * 1e3
    print(f"{wl} n=2^{lg}: " + "  ".join(f"{k} {v:7.1f} us" for k, v in res.items()), flush=True)
