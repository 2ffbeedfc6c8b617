"""world_size-2 gloo test of the sharded (N > 1) path on CPU.

Each rank runs its contiguous shard of a random-policy rollout (the CPU
oracle stands in for the GPU kernels here; the kernels' shard parity is
test_parity_gpu.py::test_shards_reproduce_the_global_batch) with keys and
task rows derived from GLOBAL env indices, then the episode statistics are
summed with the same all-reduce bench.py uses.  The totals must equal one
process running every env."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from .helpers import benchmark_file, oracle_from_table

N_GLOBAL, STEPS = 96, 520


def _run_shard(offset, count, table, params):
    import torch

    from oracle import oracle as O
    ids = (np.arange(count) + offset) % table.num_tasks
    ora = oracle_from_table(params, table, ids)
    root = O.key_from_seed(0)
    ora.reset_with_keys(*O.split_batch(root, count, offset))
    keys = [O.fold_in(O.key_from_seed(1), offset + i) for i in range(count)]
    pk0 = np.array([k[0] for k in keys], np.uint64)
    pk1 = np.array([k[1] for k in keys], np.uint64)
    ret, trials = ora.rollout_random(pk0, pk1, 0, STEPS)
    return torch.tensor([ret.sum(), float(trials.sum())], dtype=torch.float64)


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2312_12044_b200 import load_benchmark, make
    from paper_2312_12044_b200.parallel import all_reduce_stats, shard_range
    _, params = make("XLand-MiniGrid-R1-9x9")
    table = load_benchmark(benchmark_file("trivial")).task_table()
    off, cnt = shard_range(N_GLOBAL, rank, world)
    stats = all_reduce_stats(_run_shard(off, cnt, table, params))
    if rank == 0:
        np.save(out_path, stats.numpy())
    dist.destroy_process_group()


def test_two_rank_shards_sum_to_the_global_run(tmp_path):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "stats.npy")
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    from paper_2312_12044_b200 import load_benchmark, make
    _, params = make("XLand-MiniGrid-R1-9x9")
    table = load_benchmark(benchmark_file("trivial")).task_table()
    whole = _run_shard(0, N_GLOBAL, table, params).numpy()
    sharded = np.load(out)
    assert whole[1] > 0
    np.testing.assert_allclose(sharded, whole, rtol=0, atol=1e-9)


def test_shard_range_partitions():
    from paper_2312_12044_b200.parallel import shard_range, shard_task_ids
    covered = []
    for r in range(3):
        off, cnt = shard_range(100, r, 3)
        covered.extend(range(off, off + cnt))
    assert covered == list(range(100))
    assert shard_task_ids(5, 4, 6).tolist() == [5, 0, 1, 2]
