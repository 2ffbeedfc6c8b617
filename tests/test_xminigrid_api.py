"""The paper's xminigrid-style names (paper_2312_12044_b200.xminigrid) over
the batched engine: CPU checks of the host API, GPU equality with VecEnv."""
import numpy as np
import pytest
import torch

from .helpers import benchmark_file


def test_make_replace_benchmark_cpu():
    from paper_2312_12044_b200 import xminigrid as X
    env, params = X.make("XLand-MiniGrid-R4-13x13")
    assert X.GymAutoResetWrapper(env) is env
    assert env.observation_shape(params) == (5, 5, 2) and env.num_actions == 6
    bm = X.load_benchmark(benchmark_file("medium"))
    rs = bm.sample_ruleset(X.key_from_seed(3))
    p2 = params.replace(ruleset=rs)
    assert p2.ruleset == rs and p2.height == 13 and params.ruleset != rs
    assert len(X.registered_environments()) == 30
    with pytest.raises(KeyError):
        X.load_benchmark("no-such-benchmark")


@pytest.mark.gpu
def test_reset_step_equal_vecenv():
    from paper_2312_12044_b200 import VecEnv, key_from_seed, policy_keys, random_actions
    from paper_2312_12044_b200 import xminigrid as X
    env, params = X.make("XLand-MiniGrid-R4-13x13")
    env = X.GymAutoResetWrapper(env)
    bm = X.load_benchmark(benchmark_file("medium"))
    params = params.replace(ruleset=bm.sample_ruleset(key_from_seed(5)))
    n = 1024
    keys = X.split_batch(key_from_seed(0), n, device="cuda")
    ts = env.reset(params, keys)
    ref = VecEnv(params, n)
    rts = ref.reset(key_from_seed(0))
    assert torch.equal(ts.observation, rts.observations) and bool(ts.first().all())
    acts = random_actions(policy_keys(key_from_seed(1), n, device="cuda"), 0, 600)
    for t in range(600):
        ts = env.step(params, ts, acts[t])
        r = ref.step(acts[t])
        assert torch.equal(ts.observation, r.observations) and torch.equal(ts.reward, r.rewards)
        assert torch.equal(ts.step_type, r.step_types) and torch.equal(ts.discount, r.discounts)
    assert bool(ts.last().any()) or bool(ts.mid().all())
    with pytest.raises(ValueError):
        env.step(params.replace(view_size=7), ts, acts[0])
    # per-env tasks from a benchmark table
    ts2 = env.reset(params, keys[:64], rulesets=bm, task_ids=np.arange(64) * 7)
    assert ts2.observation.shape == (64, 5, 5, 2)
