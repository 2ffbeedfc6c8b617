"""The sharded (N > 1) product path on the GPU: two ranks (gloo, both on
cuda:0 — one GPU is all this pool offers) each run their contiguous shard of
the global batch through VecEnv(global_offset=...) with reset-ahead and the
in-kernel statistics, sum the statistics with parallel.all_reduce_stats and
take the max time with parallel.all_reduce_max, exactly as bench.py does.
The summed statistics and every shard's final state must equal the same
envs of one full-batch VecEnv (ref harness.py:169-181: slices of one global
split_batch).  And `bench.py --gpus 2` re-launches itself under
torch.distributed.run and reports both ranks."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.multiprocessing as mp

from .helpers import benchmark_file

pytestmark = pytest.mark.gpu

N_GLOBAL, STEPS = 8192, 520
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions
    from paper_2312_12044_b200.parallel import all_reduce_max, all_reduce_stats, shard_range
    _, params = make("XLand-MiniGrid-R4-13x13")
    bm = load_benchmark(benchmark_file("medium"))
    off, n = shard_range(N_GLOBAL, rank, world)
    vec = VecEnv(params, n, bm, device="cuda:0", global_offset=off)
    vec.enable_stats()
    vec.reset(key_from_seed(0))
    acts = random_actions(policy_keys(key_from_seed(1), n, offset=off, device="cuda:0"), 0, STEPS)
    for t in range(STEPS):
        vec.step(acts[t])
    vec.check()
    tot = all_reduce_stats(vec.episode_stats().cpu())
    tmax = all_reduce_max(torch.tensor([float(rank + 1)], dtype=torch.float64))
    torch.save({"off": off, "grids": vec.grids.cpu(), "words": vec.state_words().cpu(), "rng": vec.rng.cpu(),
                "tot": tot, "tmax": tmax}, os.path.join(out_dir, f"rank{rank}.pt"))
    dist.destroy_process_group()


def test_two_rank_shards_equal_the_global_batch(tmp_path):
    from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    _, params = make("XLand-MiniGrid-R4-13x13")
    full = VecEnv(params, N_GLOBAL, load_benchmark(benchmark_file("medium")), device="cuda:0")
    full.enable_stats()
    full.reset(key_from_seed(0))
    acts = random_actions(policy_keys(key_from_seed(1), N_GLOBAL, device="cuda:0"), 0, STEPS)
    for t in range(STEPS):
        full.step(acts[t])
    want = full.episode_stats().cpu()
    for rank in range(2):
        r = torch.load(os.path.join(tmp_path, f"rank{rank}.pt"))
        sl = slice(r["off"], r["off"] + r["grids"].shape[0])
        assert torch.equal(r["grids"], full.grids[sl].cpu())
        assert torch.equal(r["words"], full.state_words()[sl].cpu())
        assert torch.equal(r["rng"], full.rng[sl].cpu())
        assert torch.equal(r["tot"][1:], want[1:])  # trials and lengths: integer sums
        assert abs(float(r["tot"][0]) - float(want[0])) <= 1e-9 * max(1.0, abs(float(want[0])))
        assert float(r["tmax"][0]) == 2.0


def test_bench_gpus_2_launches_two_ranks():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", "c2",
                          "--steps", "8", "--warmup", "3", "--no-e2e", "--no-fused", "--no-block", "--no-image",
                          "--no-windows"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_envs"] == 2 * d["config"]["envs_per_gpu"]
    assert d["value"] > 0
