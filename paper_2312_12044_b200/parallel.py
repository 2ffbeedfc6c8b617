"""Multi-GPU plumbing: env-range sharding and the one statistics collective.

Envs are independent (ref vecenv.py:1-17), so N GPUs run N shards with no
per-step communication: rank g owns the contiguous global env range
[g*n, (g+1)*n) and derives every per-env key and task row from the GLOBAL
index (split_batch(root, n, offset), task = (offset + i) % M), which makes a
shard's trajectories identical to the same envs of a single-GPU run -- the
property the reference tests for its process pool (ref
tests/test_harness.py:105-122).  After a run one all-reduce (NCCL on GPUs,
gloo in the CPU tests) sums the episode statistics (ref RolloutStats,
harness.py:103-143).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_range(global_envs: int, rank: int, world: int) -> tuple[int, int]:
    """(offset, count) of rank's contiguous share; the last rank takes the remainder."""
    if not 0 <= rank < world:
        raise ValueError("rank outside [0, world)")
    per = global_envs // world
    off = rank * per
    return off, (global_envs - off if rank == world - 1 else per)


def shard_task_ids(offset: int, count: int, num_tasks: int) -> np.ndarray:
    """Task-table rows of a shard: env i (global) runs row i mod M."""
    return ((np.arange(count, dtype=np.int64) + offset) % num_tasks).astype(np.int32)


def all_reduce_stats(stats: torch.Tensor) -> torch.Tensor:
    """Sum a small statistics tensor over all ranks (in place); no-op when
    torch.distributed is not initialised."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM)
    return stats


def all_reduce_max(x: torch.Tensor) -> torch.Tensor:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
    return x
