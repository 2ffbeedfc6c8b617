"""Quick device timing of VecEnv.step (CUDA events) for development."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from helpers import benchmark_file

def run(env_name, config, n, steps, validate=True, compute_obs=True):
    _, params = make(env_name)
    vec = VecEnv(params, n, load_benchmark(benchmark_file(config)) if config else None, reuse_outputs=True)
    vec.reset(key_from_seed(0))
    acts = random_actions(policy_keys(key_from_seed(1), n, device="cuda"), 0, steps)
    for t in range(5): vec.step(acts[t], compute_obs, validate)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for t in range(steps): vec.step(acts[t], compute_obs, validate)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(f"{env_name:28s} {config or '-':8s} n={n:9d} steps={steps} validate={validate} obs={compute_obs}: "
          f"{ms/steps*1e3:8.1f} us/step  {n*steps/ms*1e3/1e9:7.3f} G env-steps/s", flush=True)

if __name__ == "__main__":
    run("XLand-MiniGrid-R4-13x13", "medium", 1 << 20, 600)
    run("XLand-MiniGrid-R4-13x13", "medium", 1 << 20, 600, validate=False)
    run("XLand-MiniGrid-R1-9x9", "trivial", 1 << 16, 600)
    run("XLand-MiniGrid-R1-9x9", "trivial", 1 << 20, 600)
    run("XLand-MiniGrid-R9-25x25", "high", 1 << 19, 1900)
    run("MiniGrid-DoorKey-8x8", None, 1 << 20, 400)
    run("MiniGrid-Empty-8x8", None, 1 << 20, 400)
