"""GPU parity of the fused rollout kernel (xmg_rollout).

The rollout is T VecEnv.step calls in one kernel; it must be bit-identical to
them (and therefore to the oracle): every record of every step (observation,
reward, discount, step type), the final state (grids, pose, pocket, step
count, goal / task word, rng key) and the episode statistics.
"""
import numpy as np
import pytest
import torch

from .helpers import benchmark_file, oracle_from_table

pytestmark = pytest.mark.gpu


def _pair(env_name, config, n, resample=False, see=None, **kw):
    from paper_2312_12044_b200 import VecEnv, load_benchmark, make
    _, params = make(env_name)
    if see is not None:
        from dataclasses import replace
        params = replace(params, see_through_walls=see)
    bm = load_benchmark(benchmark_file(config)) if config else None
    a = VecEnv(params, n, bm, resample_tasks=resample, **kw)
    b = VecEnv(params, n, bm, resample_tasks=resample, **kw)
    return params, bm, a, b


def _same_state(a, b, msg):
    torch.testing.assert_close(a.grids, b.grids, rtol=0, atol=0, msg=f"grids {msg}")
    assert torch.equal(a.state_words(), b.state_words()), f"agent word {msg}"
    assert torch.equal(a.rng, b.rng), f"rng {msg}"


@pytest.mark.parametrize("env_name,config,n,steps,resample,see,fused", [
    ("XLand-MiniGrid-R4-13x13", "medium", 4096, 600, False, None, None),
    ("XLand-MiniGrid-R4-13x13", "medium", 2048, 530, False, None, False),   # the per-call rollout path
    ("XLand-MiniGrid-R1-9x9", "trivial", 4096, 300, False, None, None),
    ("XLand-MiniGrid-R9-25x25", "high", 1024, 400, False, None, None),    # auto: per-call kernels
    ("XLand-MiniGrid-R9-25x25", "high", 1024, 400, False, None, True),    # the fused kernel, 25x25 grids
    ("XLand-MiniGrid-R4-13x13", "medium", 1000, 520, True, None, None),     # resample-on-reset, ragged tail
    ("XLand-MiniGrid-R2-13x13", "small", 999, 300, False, False, None),     # occluded view, odd n
    ("MiniGrid-DoorKey-8x8", None, 2048, 250, False, None, None),
    ("MiniGrid-UnlockPickUp", None, 1024, 400, False, None, None),
    ("MiniGrid-FourRooms", None, 512, 300, False, None, None),
    ("MiniGrid-Empty-8x8", None, 333, 200, False, None, None),
])
def test_rollout_equals_steps(env_name, config, n, steps, resample, see, fused):
    from paper_2312_12044_b200 import key_from_seed, policy_keys, random_actions
    params, bm, a, b = _pair(env_name, config, n, resample, see)
    root = key_from_seed(7)
    a.reset(root)
    b.reset(root)
    sa, sb = a.enable_stats(), b.enable_stats()
    pk = policy_keys(key_from_seed(1), n, device=a.device)
    acts = random_actions(pk, 0, steps)
    tr = b.rollout(steps, policy_keys=pk, fused=fused)
    for t in range(steps):
        ts = a.step(acts[t])
        assert torch.equal(ts.observations, tr.observations[t]), f"obs t={t}"
        assert torch.equal(ts.rewards, tr.rewards[t]), f"reward t={t}"
        assert torch.equal(ts.discounts, tr.discounts[t]), f"discount t={t}"
        assert torch.equal(ts.step_types, tr.step_types[t]), f"step type t={t}"
    a.check()
    _same_state(a, b, "after rollout")
    torch.testing.assert_close(sa.sum(0), sb.sum(0), rtol=1e-12, atol=1e-9)
    assert float(sa[:, 1].sum()) == float(sb[:, 1].sum())  # trial counts exact


def test_rollout_vs_oracle_and_interleaving():
    """Rollout chunks interleaved with single steps (the rollout consumes no
    epoch) against the oracle on the same keys, tasks and actions."""
    from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions
    _, params = make("XLand-MiniGrid-R4-13x13")
    bm = load_benchmark(benchmark_file("medium"))
    n = 2048
    vec = VecEnv(params, n, bm)
    ora = oracle_from_table(params, bm.task_table(), vec._ids_host)
    root = key_from_seed(0)
    vec.reset(root)
    ora.reset(root)
    pk = policy_keys(key_from_seed(1), n, device=vec.device)
    acts_h = random_actions(pk, 0, 560).cpu().numpy()
    t = 0
    for kind, k in [("roll", 100), ("step", 3), ("roll", 1), ("step", 1), ("roll", 405), ("step", 50)]:
        if kind == "roll":
            tr = vec.rollout(k, policy_keys=pk, t0=t)
            recs = [(tr.observations[i], tr.rewards[i], tr.discounts[i], tr.step_types[i]) for i in range(k)]
        else:
            recs = []
            for i in range(k):
                ts = vec.step(torch.from_numpy(acts_h[t + i]).cuda())
                recs.append((ts.observations.clone(), ts.rewards.clone(), ts.discounts.clone(), ts.step_types.clone()))
        for i in range(k):
            o, r, d, s = ora.step(acts_h[t + i])
            np.testing.assert_array_equal(recs[i][0].cpu().numpy(), o, err_msg=f"obs t={t + i}")
            np.testing.assert_array_equal(recs[i][1].cpu().numpy(), r.astype(np.float32))
            np.testing.assert_array_equal(recs[i][2].cpu().numpy(), d.astype(np.float32))
            np.testing.assert_array_equal(recs[i][3].cpu().numpy(), s, err_msg=f"step type t={t + i}")
        t += k
        np.testing.assert_array_equal(vec.grids.cpu().numpy(), ora.grids, err_msg=f"grids t={t}")
        np.testing.assert_array_equal(vec.rng.cpu().numpy().view(np.uint64), ora.rng)
    vec.check()


@pytest.mark.parametrize("fused", [None, False])
def test_rollout_explicit_actions_and_partial_records(fused):
    """A (T, N) action tensor instead of the policy keys; records subset;
    stats-only mode; invalid actions rejected before any mutation (the fused
    kernel and the per-call rollout path)."""
    from paper_2312_12044_b200 import InvalidAction, key_from_seed
    params, bm, a, b = _pair("XLand-MiniGrid-R4-13x13", "medium", 777)
    root = key_from_seed(3)
    a.reset(root)
    b.reset(root)
    g = torch.Generator().manual_seed(5)
    acts = torch.randint(0, 6, (530, 777), generator=g, dtype=torch.int64)
    sa, sb = a.enable_stats(), b.enable_stats()
    tr = b.rollout(300, actions=acts[:300], record=("rewards", "step_types"), fused=fused)
    assert tr.observations is None and tr.discounts is None
    b.rollout(230, actions=acts[300:].cuda(), record=(), fused=fused)
    rews, sts = [], []
    for t in range(530):
        ts = a.step(acts[t].cuda())
        if t < 300:
            rews.append(ts.rewards.clone())
            sts.append(ts.step_types.clone())
    assert torch.equal(torch.stack(rews), tr.rewards)
    assert torch.equal(torch.stack(sts), tr.step_types)
    _same_state(a, b, "after explicit-action rollout")
    torch.testing.assert_close(sa.sum(0), sb.sum(0), rtol=1e-12, atol=1e-9)
    before = b.grids.clone()
    bad = acts[:10].clone()
    bad[4, 17] = 6
    with pytest.raises(InvalidAction):
        b.rollout(10, actions=bad, fused=fused)
    assert torch.equal(before, b.grids)


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("env_name,config,n,k", [
    ("XLand-MiniGrid-R4-13x13", "medium", 4096, 530),
    ("MiniGrid-Empty-8x8", None, 1024, 256),      # BASELINE configs[0] shape
    ("XLand-MiniGrid-R1-9x9", "trivial", 1 << 16, 260),
])
def test_steps_block_equals_single_steps(env_name, config, n, k, fused):
    """VecEnv.steps (K steps from one host call: the fused kernel, or
    xmg_steps) == K step() calls, interleaved with single steps and a rollout
    on the same state."""
    from paper_2312_12044_b200 import InvalidAction, key_from_seed, policy_keys, random_actions
    params, bm, a, b = _pair(env_name, config, n)
    root = key_from_seed(9)
    a.reset(root)
    b.reset(root)
    sa, sb = a.enable_stats(), b.enable_stats()
    pk = policy_keys(key_from_seed(1), n, device=a.device)
    acts = random_actions(pk, 0, k + 20)
    tr = b.steps(acts[:k], fused=fused)
    for t in range(k):
        ts = a.step(acts[t])
        assert torch.equal(ts.observations, tr.observations[t]), f"obs t={t}"
        assert torch.equal(ts.rewards, tr.rewards[t]) and torch.equal(ts.step_types, tr.step_types[t])
        assert torch.equal(ts.discounts, tr.discounts[t])
    _same_state(a, b, "after steps")
    for t in range(k, k + 10):  # single steps after a block, then a rollout
        a.step(acts[t])
        b.step(acts[t])
    a.rollout(10, policy_keys=pk, t0=k + 10, record=())
    b.steps(acts[k + 10:k + 20], compute_obs=False, fused=fused)
    _same_state(a, b, "after mixing")
    torch.testing.assert_close(sa.sum(0), sb.sum(0), rtol=1e-12, atol=1e-9)
    bad = acts[:4].clone()
    bad[2, 5] = 7
    before = b.grids.clone()
    with pytest.raises(InvalidAction):
        b.steps(bad, fused=fused)
    assert torch.equal(before, b.grids)


def test_resample_on_reset_uses_sample_ruleset():
    """Resample mode (an extension without a reference
    oracle) is pinned to the reference's sampling primitive: a trial that ends
    with episode key ek continues with task Benchmark.sample_ruleset(split(ek,
    2)) = row randint(split(ek, 2), M) (ref benchio.py:57-58), and its new
    trial equals a plain reset_with_keys(ek) of an env bound to that task."""
    from paper_2312_12044_b200 import Key, VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions
    from paper_2312_12044_b200.core import randint, split
    _, params = make("XLand-MiniGrid-R4-13x13")
    bm = load_benchmark(benchmark_file("medium"))
    n, budget = 512, params.step_budget
    vec = VecEnv(params, n, bm, resample_tasks=True)
    vec.reset(key_from_seed(3))
    acts = random_actions(policy_keys(key_from_seed(4), n, device=vec.device), 0, budget)
    for t in range(budget - 1):
        vec.step(acts[t])
    ek = vec.rng.cpu().numpy().view(np.uint64).copy()
    ts = vec.step(acts[budget - 1])
    last = ts.step_types.cpu().numpy() == 2
    assert last.sum() > n // 2  # the synchronized budget reset
    want = np.array([randint(split(Key(int(a), int(b)), 3)[2], bm.num_rulesets()) for a, b in ek], np.int64)
    got = vec.task.cpu().numpy()
    np.testing.assert_array_equal(got[last], want[last])
    ref = VecEnv(params, n, bm, task_ids=want)
    rts = ref.reset_with_keys(ek[:, 0], ek[:, 1])
    np.testing.assert_array_equal(vec.grids.cpu().numpy()[last], ref.grids.cpu().numpy()[last])
    np.testing.assert_array_equal(vec.state_words().cpu().numpy()[last], ref.state_words().cpu().numpy()[last])
    np.testing.assert_array_equal(vec.rng.cpu().numpy()[last], ref.rng.cpu().numpy()[last])
    np.testing.assert_array_equal(ts.observations.cpu().numpy()[last], rts.observations.cpu().numpy()[last])
