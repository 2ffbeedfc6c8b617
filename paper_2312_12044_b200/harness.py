"""Throughput and scaling harness over the GPU engine.

GPU counterparts of the reference's measurement entry points
(ref harness.py:149-276): ``bench_throughput`` (random-policy env-steps per
second for each batch size, the minimum over repeats) and ``bench_scaling``
(along the grid-size or rule-count axis, with the reference's fixed
``scaling_ruleset`` workload and trial length), plus ``write_csv``.

Differences by design: time is measured on the device with CUDA events
around the steps (not ``time.perf_counter`` around a process pool), the
``workers`` argument of the reference is accepted and ignored (one GPU runs
the whole batch; shard across GPUs with ``VecEnv(global_offset=...)``), and
the random actions are Philox words of per-env policy keys generated on the
device (``random_actions``) rather than NumPy PCG64 draws.  ``mode`` picks
the engine path being timed: ``"step"`` (one ``VecEnv.step`` per step, the
reference's loop), ``"steps"`` (64 steps per host call) or ``"rollout"``
(the fused kernel, statistics only).
"""

from __future__ import annotations

import csv
from typing import Iterable, Sequence

import torch

from .core import Color, Tile, fold_in, key_from_seed, pack_entity
from .env import EnvParams, make
from .ruleset import Ruleset
from .vecenv import VecEnv, policy_keys, random_actions

GRID_SIZE_VALUES = (9, 13, 17, 25)        # ref harness.py:44
NUM_RULES_VALUES = (1, 3, 6, 12, 24)      # ref harness.py:45
SCALING_TRIAL_STEPS = 256                 # ref harness.py:52
MODES = ("step", "steps", "rollout")


def _timed_sps(params: EnvParams, num_envs: int, num_steps: int, seed: int, rep: int, mode: str,
               rulesets=None, device=None) -> float:
    """env-steps/s of one timed run: reset, then ``num_steps`` random-policy
    steps, CUDA events on the current stream."""
    vec = VecEnv(params, num_envs, rulesets, device=device, reuse_outputs=True)
    root = fold_in(key_from_seed(seed), rep)
    vec.reset(root)
    keys = policy_keys(fold_in(root, 1), num_envs, device=vec.device)
    acts = random_actions(keys, 0, num_steps) if mode != "rollout" else None
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(vec.device)
    start.record()
    if mode == "step":
        for t in range(num_steps):
            vec.step(acts[t])
    elif mode == "steps":
        for t0 in range(0, num_steps, 64):
            vec.steps(acts[t0:t0 + 64], validate=False,
                      compute_obs=(num_envs * 2 * params.view_size ** 2) % 16 == 0)
    else:
        vec.rollout(num_steps, policy_keys=keys, record=())
    end.record()
    torch.cuda.synchronize(vec.device)
    vec.check()
    return num_envs * num_steps / (start.elapsed_time(end) / 1e3)


def _bench_params(params: EnvParams, num_envs_list: Sequence[int], num_steps: int, repeats: int, seed: int,
                  mode: str, device=None) -> list[tuple[int, float]]:
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}, got {mode!r}")
    rows = []
    for n in num_envs_list:
        samples = [_timed_sps(params, n, num_steps, seed, rep, mode, device=device) for rep in range(max(1, repeats))]
        rows.append((n, min(samples)))
    return rows


def bench_throughput(env_name: str, num_envs_list: Sequence[int], num_steps: int = 512, repeats: int = 3,
                     workers: int = 1, seed: int = 0, mode: str = "step", device=None) -> list[tuple[int, float]]:
    """Random-policy env-steps per second for each batch size: (num_envs,
    sps) rows, sps the minimum over ``repeats`` timed runs (ref
    harness.py:204-218)."""
    _, params = make(env_name)
    return _bench_params(params, num_envs_list, num_steps, repeats, seed, mode, device)


def scaling_ruleset(num_rules: int) -> Ruleset:
    """The reference's replicated-NEAR workload (ref harness.py:224-246): one
    TILE_NEAR rule copied ``num_rules`` times whose second input never
    exists, so no copy fires and the dynamics are identical across rule
    counts; the goal object is never placed, so trials end on the budget."""
    a = pack_entity(Tile.BALL, Color.RED)
    b = pack_entity(Tile.SQUARE, Color.GREEN)
    out = pack_entity(Tile.PYRAMID, Color.BLUE)
    prize = pack_entity(Tile.HEX, Color.PURPLE)
    movers = tuple(pack_entity(Tile.BALL, c) for c in (Color.RED, Color.YELLOW, Color.PURPLE, Color.WHITE))
    return Ruleset(goal=(1, prize, 0, 0), rules=((3, a, b, out),) * num_rules, init_objects=movers)


def bench_scaling(axis: str, values: Sequence[int], num_envs: int = 1024, num_steps: int = 256, repeats: int = 3,
                  workers: int = 1, seed: int = 0, mode: str = "step", device=None) -> list[tuple[int, float]]:
    """Env-steps per second along one axis, (value, sps) rows (ref
    harness.py:249-275): ``grid_size`` varies a square single-room grid,
    ``num_rules`` replicates the NEAR rule on a 16x16 grid; both with the
    fixed trial length SCALING_TRIAL_STEPS."""
    rows = []
    for value in values:
        if axis == "grid_size":
            params = EnvParams(height=value, width=value, ruleset=scaling_ruleset(1), max_steps=SCALING_TRIAL_STEPS)
        elif axis == "num_rules":
            params = EnvParams(height=16, width=16, ruleset=scaling_ruleset(value), max_steps=SCALING_TRIAL_STEPS)
        else:
            raise ValueError(f"axis must be 'grid_size' or 'num_rules', got {axis!r}")
        (_, sps), = _bench_params(params, [num_envs], num_steps, repeats, seed, mode, device)
        rows.append((value, sps))
    return rows


def write_csv(path, header: Sequence[str], rows: Iterable[tuple]) -> None:
    """ref harness.py:278-282."""
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(header)
        writer.writerows(rows)
