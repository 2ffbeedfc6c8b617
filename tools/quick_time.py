"""Quick device timing of VecEnv.step (CUDA events) for development.
python tools/quick_time.py [names...]  (default: all)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from helpers import benchmark_file  # noqa: E402
from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions  # noqa

RUNS = {
    "c3": ("XLand-MiniGrid-R4-13x13", "medium", 1 << 20, 600),
    "c3nv": ("XLand-MiniGrid-R4-13x13", "medium", 1 << 20, 600),
    "c2": ("XLand-MiniGrid-R1-9x9", "trivial", 1 << 16, 600),
    "r1big": ("XLand-MiniGrid-R1-9x9", "trivial", 1 << 20, 600),
    "c4": ("XLand-MiniGrid-R9-25x25", "high", 1 << 19, 1900),
    "doorkey": ("MiniGrid-DoorKey-8x8", None, 1 << 20, 400),
    "empty": ("MiniGrid-Empty-8x8", None, 1 << 20, 400),
}


def run(name):
    env_name, config, n, steps = RUNS[name]
    validate = name != "c3nv"
    _, params = make(env_name)
    vec = VecEnv(params, n, load_benchmark(benchmark_file(config)) if config else None, reuse_outputs=True)
    vec.reset(key_from_seed(0))
    acts = random_actions(policy_keys(key_from_seed(1), n, device="cuda"), 0, steps)
    for t in range(5):
        vec.step(acts[t], True, validate)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for t in range(steps):
        vec.step(acts[t], True, validate)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(f"{os.environ.get('XMG_LIB', 'default')[-20:]:20s} {name:8s} {env_name:26s} n={n:8d} steps={steps}: "
          f"{ms / steps * 1e3:8.1f} us/step {n * steps / ms * 1e3 / 1e9:7.3f} G env-steps/s", flush=True)


if __name__ == "__main__":
    for nm in (sys.argv[1:] or RUNS):
        run(nm)
