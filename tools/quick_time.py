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




def burst(name="c3", around=506, k=4):
    """Per-step device times around the synchronized budget reset."""
    env_name, config, n, _ = RUNS[name]
    _, params = make(env_name)
    vec = VecEnv(params, n, load_benchmark(benchmark_file(config)) if config else None, reuse_outputs=True)
    vec.reset(key_from_seed(0))
    acts = random_actions(policy_keys(key_from_seed(1), n, device="cuda"), 0, around + k)
    for t in range(around - 1):
        vec.step(acts[t], True, False)
    times = []
    for t in range(around - 1, around - 1 + k):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        vec.step(acts[t], True, False)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) * 1e3)
    print(f"{os.environ.get('XMG_LIB', 'default')[-20:]:20s} burst {name}: steps {around - 1}..{around + k - 2} us: "
          + " ".join(f"{x:.0f}" for x in times), flush=True)


if __name__ == "__main__":  # noqa
    for nm in (sys.argv[1:] or RUNS):
        if nm.startswith("burst:"):
            burst(nm.split(":")[1])
        else:
            run(nm)
