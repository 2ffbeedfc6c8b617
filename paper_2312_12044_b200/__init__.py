"""B200-native batched XLand-MiniGrid environment step (arXiv 2312.12044).

Host-side mirror of the reference ``rulegrid`` API for the batched step
(make / EnvParams / VecEnv / load_benchmark / sample_ruleset / keys) over the
sm_100a kernels of libxmg.so (C ABI: include/xmg.h).  The paper's
``xminigrid`` names (make / GymAutoResetWrapper / load_benchmark / batched
reset and step) are in :mod:`paper_2312_12044_b200.xminigrid`; the fused
rollout is ``VecEnv.rollout``, observation images are in
:mod:`paper_2312_12044_b200.render`, the JSON-lines server in
:mod:`paper_2312_12044_b200.bridge`.
"""

from ._lib import NativeLibraryError, build
from .core import (AgentState, Color, Direction, Entity, FormatError, Grid, GridFull, InvalidAction, InvalidCode,
                   InvalidEncoding, InvalidProportion, Key, LayoutTooSmall, Position, Tile, UnknownBenchmark,
                   UnknownEnvironment, fold_in, key_from_seed, pack_entity, random_words, randint, split,
                   unpack_entity)
from .env import Action, Environment, EnvParams, StepType, make, registered_environments
from .layouts import Layout, plan_layout
from .ruleset import (EMPTY_RULESET, MAX_INIT_OBJECTS, MAX_RULES, Benchmark, Ruleset, TaskTable, load_benchmark,
                      load_named, registered_benchmarks, save_benchmark)
from .vecenv import EnvState, Trajectory, VecEnv, VecTimeStep, philox, policy_keys, random_actions, split_batch

__version__ = "0.1.0"

__all__ = [
    "Action", "AgentState", "Benchmark", "Color", "Direction", "EMPTY_RULESET", "Entity", "EnvParams", "EnvState",
    "Environment", "FormatError", "Grid", "GridFull", "InvalidAction", "InvalidCode", "InvalidEncoding",
    "InvalidProportion", "Key", "Layout", "LayoutTooSmall", "MAX_INIT_OBJECTS", "MAX_RULES", "NativeLibraryError",
    "Position", "Ruleset", "StepType", "TaskTable", "Tile", "Trajectory", "UnknownBenchmark", "UnknownEnvironment", "VecEnv",
    "VecTimeStep", "build", "fold_in", "key_from_seed", "load_benchmark", "load_named", "make", "pack_entity",
    "philox", "plan_layout", "policy_keys", "random_actions", "random_words", "randint", "registered_benchmarks",
    "registered_environments", "save_benchmark", "split", "split_batch", "unpack_entity",
]
