"""Small workload touching every kernel, for compute-sanitizer
(memcheck / racecheck / synccheck):
  compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from helpers import benchmark_file  # noqa: E402
from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions  # noqa
from paper_2312_12044_b200.render import image_observations  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
for env_name, cfg in (("XLand-MiniGrid-R4-13x13", "medium"), ("MiniGrid-DoorKey-8x8", None)):
    _, params = make(env_name)
    bm = load_benchmark(benchmark_file(cfg)) if cfg else None
    vec = VecEnv(params, n, bm)
    vec.enable_stats()
    vec.reset(key_from_seed(0))
    pk = policy_keys(key_from_seed(1), n, device=vec.device)
    acts = random_actions(pk, 0, 40)
    for t in range(20):
        ts = vec.step(acts[t])
    vec.steps(acts[20:30].contiguous(), compute_obs=(n * 50) % 16 == 0)
    vec.rollout(10, policy_keys=pk, t0=30)
    image_observations(ts.observations[:64])
    vec.check()
torch.cuda.synchronize()
print("sanitize workload done")
