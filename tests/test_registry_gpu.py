"""Every registered environment id (ref registry.py:9-51) through the GPU
engine against the oracle: 512 envs under the on-device random policy, past
the first synchronized budget reset where the budget allows, all outputs
every step and the final state bit-exact."""
import numpy as np
import pytest

from .helpers import benchmark_file, oracle_from_table
from .test_parity_gpu import _assert_state

pytestmark = pytest.mark.gpu

# rule-count family -> the benchmark whose tasks it runs here (R1 trivial,
# R2 small, R4 / R6 medium, R9 high)
_CONFIG = {"R1": "trivial", "R2": "small", "R4": "medium", "R6": "medium", "R9": "high"}


def _ids():
    from paper_2312_12044_b200.env import registered_environments
    return registered_environments()


@pytest.mark.parametrize("env_name", _ids())
def test_every_registered_env_vs_oracle(env_name):
    from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions
    from paper_2312_12044_b200.ruleset import TaskTable
    _, params = make(env_name)
    n = 512
    steps = min(params.step_budget + 5, 1100)
    config = _CONFIG[env_name.split("-")[2]] if env_name.startswith("XLand") else None
    if config:
        bm = load_benchmark(benchmark_file(config))
        vec = VecEnv(params, n, bm)
        ora = oracle_from_table(params, bm.task_table(), vec._ids_host)
    else:
        vec = VecEnv(params, n)
        ora = oracle_from_table(params, TaskTable(np.zeros((1, 4), np.uint32), 0, 0, 0), np.zeros(n, np.int64))
    root = key_from_seed(11)
    np.testing.assert_array_equal(vec.reset(root).observations.cpu().numpy(), ora.reset(root))
    acts = random_actions(policy_keys(key_from_seed(12), n, device=vec.device), 0, steps)
    ah = acts.cpu().numpy()
    lasts = 0
    for t in range(steps):
        ts = vec.step(acts[t])
        o, r, d, s = ora.step(ah[t])
        obs, rew, disc, st = ts.numpy()
        np.testing.assert_array_equal(st, s, err_msg=f"{env_name} step_type t={t}")
        np.testing.assert_array_equal(rew, r.astype(np.float32), err_msg=f"{env_name} reward t={t}")
        np.testing.assert_array_equal(disc, d.astype(np.float32), err_msg=f"{env_name} discount t={t}")
        np.testing.assert_array_equal(obs, o, err_msg=f"{env_name} obs t={t}")
        lasts += int((s == 2).sum())
    _assert_state(vec, ora.grids, ora.agent(), ora.rng, ora.step_count, f"{env_name} final")
    vec.check()
    assert lasts > 0, "no trial ended: the auto-reset path was not exercised"


@pytest.mark.parametrize("env_name", _ids())
def test_every_registered_env_rollout_and_steps_equal_step(env_name):
    """The fused rollout (xmg_rollout) and the block path (xmg_steps) against
    per-call steps on twin batches, for every registered id: records and final
    state identical (the per-call path is pinned to the oracle above)."""
    import torch
    from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions
    _, params = make(env_name)
    n = 336  # ragged: not a multiple of a warp or a CTA (n * 50 a multiple of 16 for the block path)
    steps = min(params.step_budget + 5, 600)
    config = _CONFIG[env_name.split("-")[2]] if env_name.startswith("XLand") else None
    bm = load_benchmark(benchmark_file(config)) if config else None
    a, b, c = (VecEnv(params, n, bm) for _ in range(3))
    for v in (a, b, c):
        v.reset(key_from_seed(21))
    keys = policy_keys(key_from_seed(22), n, device=a.device)
    acts = random_actions(keys, 0, steps)
    tr = a.rollout(steps, policy_keys=keys)
    blk = b.steps(acts, compute_obs=(n * 2 * params.view_size ** 2) % 16 == 0)
    for t in range(steps):
        ts = c.step(acts[t])
        for name in ("observations", "rewards", "discounts", "step_types"):
            ref = getattr(ts, name)
            torch.testing.assert_close(getattr(tr, name)[t], ref, rtol=0, atol=0,
                                       msg=f"{env_name} rollout {name} t={t}")
            got = getattr(blk, name)
            if got is not None:
                torch.testing.assert_close(got[t], ref, rtol=0, atol=0, msg=f"{env_name} steps {name} t={t}")
    for v in (a, b):
        assert torch.equal(v.grids, c.grids) and torch.equal(v.state_words(), c.state_words()) and torch.equal(v.rng, c.rng)
    for v in (a, b, c):
        v.check()
