"""The paper's ``xminigrid`` names over the batched GPU engine.

``BASELINE.json:north_star`` names the API of the paper's JAX package
(``xminigrid.make(env_id) -> (env, env_params)``, ``env.reset`` /
``env.step`` over a batch of TimeSteps, ``load_benchmark`` /
``sample_ruleset``, ``GymAutoResetWrapper``).
The mounted reference exports the same capabilities as ``rulegrid.*``
(SURVEY.md 0.1 #1); this module is the thin alias layer over them:

    env, env_params = xminigrid.make("XLand-MiniGrid-R4-13x13")
    env = GymAutoResetWrapper(env)                      # auto-reset is built in
    benchmark = xminigrid.load_benchmark("trivial")     # registered name or a path
    ruleset = benchmark.sample_ruleset(key)             # ref benchio.py:57-58
    env_params = env_params.replace(ruleset=ruleset)
    timestep = env.reset(env_params, keys)              # keys: (N, 2) episode keys
    timestep = env.step(env_params, timestep, actions)  # actions: (N,)

Differences from JAX, by design: the batch is explicit (no ``vmap``), keys
are (N, 2) tensors of episode keys (``split_batch`` makes them), and the
state is device-resident and advanced in place: ``timestep.state`` is the
``VecEnv`` that owns it, so a TimeStep is a view of the latest step, not an
immutable value.  Per-env rulesets come from ``reset(..., rulesets=...)``
(a Benchmark / TaskTable with optional ``task_ids``, or a list).
Semantics are those of ``rulegrid.VecEnv`` (GymAutoReset: a LAST record
carries the next trial's first observation).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .core import Key, key_from_seed
from .env import EnvParams, StepType, registered_environments
from .env import make as _make
from .ruleset import Benchmark, load_benchmark as _load_path, load_named, registered_benchmarks
from .vecenv import VecEnv, split_batch

__all__ = ["make", "registered_environments", "load_benchmark", "registered_benchmarks", "GymAutoResetWrapper",
           "Environment", "TimeStep", "EnvParams", "StepType", "split_batch", "key_from_seed"]


@dataclass(eq=False)
class TimeStep:
    """Batched TimeStep (paper's ``xminigrid.types.TimeStep``): device
    tensors of the latest record plus the VecEnv owning the state."""
    state: VecEnv
    step_type: torch.Tensor    # (N,) int8: FIRST 0 / MID 1 / LAST 2
    reward: torch.Tensor       # (N,) float32
    discount: torch.Tensor     # (N,) float32
    observation: torch.Tensor  # (N, v, v, 2) uint8

    def first(self) -> torch.Tensor:
        return self.step_type == int(StepType.FIRST)

    def mid(self) -> torch.Tensor:
        return self.step_type == int(StepType.MID)

    def last(self) -> torch.Tensor:
        return self.step_type == int(StepType.LAST)


class Environment:
    """``env`` of ``xminigrid.make``: reset / step over a batch."""

    num_actions = 6

    def __init__(self, device=None):
        self.device = device

    def observation_shape(self, params: EnvParams) -> tuple[int, int, int]:
        return (params.view_size, params.view_size, 2)

    def reset(self, params: EnvParams, keys, rulesets=None, task_ids=None) -> TimeStep:
        """Reset N envs from their episode keys ((N, 2) tensor / array of
        (hi, lo) words, or one Key for N = 1); ref VecEnv.reset_with_keys."""
        if isinstance(keys, Key):
            keys = np.array([[keys.hi, keys.lo]], np.uint64)
        if isinstance(keys, torch.Tensor):
            k = keys.to(torch.int64)
            k0, k1 = k[:, 0], k[:, 1]
        else:
            k = np.asarray(keys, np.uint64).reshape(-1, 2)
            k0, k1 = k[:, 0], k[:, 1]
        n = int(k0.shape[0])
        vec = VecEnv(params, n, rulesets, device=self.device, task_ids=task_ids)
        ts = vec.reset_with_keys(k0, k1)
        return TimeStep(vec, ts.step_types, ts.rewards, ts.discounts, ts.observations)

    def step(self, params: EnvParams, timestep: TimeStep, actions) -> TimeStep:
        """One step of every env (auto-reset included), ref VecEnv.step."""
        vec = timestep.state
        if vec.params != params:
            raise ValueError("step() params differ from the ones this batch was reset with "
                             "(the state binds them at reset)")
        ts = vec.step(actions)
        return TimeStep(vec, ts.step_types, ts.rewards, ts.discounts, ts.observations)


def GymAutoResetWrapper(env: Environment) -> Environment:  # noqa: N802 (the paper's name)
    """Auto-reset is part of every step here (ref vecenv.py:9-11, 359-361):
    the wrapper is the identity."""
    return env


def make(env_id: str, device=None) -> tuple[Environment, EnvParams]:
    """``xminigrid.make``: (env, env_params) for a registered id (30 ids,
    ref registry.py:9-51)."""
    _, params = _make(env_id)
    return Environment(device), params


def load_benchmark(name_or_path) -> Benchmark:
    """A registered benchmark name (``load_named``: $XMINIGRID_DATA or
    ~/.xland_minigrid) or a path to an ``.xmgb`` file (ref benchio.py:110-206)."""
    import os
    if os.path.exists(str(name_or_path)):
        return _load_path(name_or_path)
    return load_named(str(name_or_path))
