"""Graph mode (VecEnv(graph=True), csrc xmg_step_fused): each step() is ONE
fused kernel (the rollout kernel at T = 1 with in-kernel validation and a
device step counter) replayed from a CUDA graph — the small-batch path that
replaces the reference's per-step loop (ref harness.py:149-158) without the
per-step launch overhead.  Results must equal the two-kernel step bit for bit
and the reference's InvalidAction semantics must hold (ref vecenv.py:297-301:
an invalid batch changes nothing)."""
import numpy as np
import pytest
import torch

from .helpers import benchmark_file

pytestmark = pytest.mark.gpu


def _pair(env_name, config, n):
    from paper_2312_12044_b200 import VecEnv, load_benchmark, make
    _, params = make(env_name)
    bm = load_benchmark(benchmark_file(config)) if config else None
    return params, VecEnv(params, n, bm, graph=True), VecEnv(params, n, bm)


@pytest.mark.parametrize("env_name,config,n,budgets", [
    ("MiniGrid-Empty-8x8", None, 1024, 1.5),
    ("MiniGrid-DoorKey-8x8", None, 1000, 1.3),
    ("XLand-MiniGrid-R1-9x9", "trivial", 4096, 2.2),
    ("XLand-MiniGrid-R4-13x13", "medium", 2048, 1.1),
])
def test_graph_steps_equal_two_kernel_steps(env_name, config, n, budgets):
    from paper_2312_12044_b200 import key_from_seed, policy_keys, random_actions
    params, g, ref = _pair(env_name, config, n)
    g.reset(key_from_seed(7))
    ref.reset(key_from_seed(7))
    steps = int(budgets * params.step_budget)
    acts = random_actions(policy_keys(key_from_seed(8), n, device=g.device), 0, steps)
    for t in range(steps):
        a = acts[t]
        if t % 3 == 1:  # int64 device actions and host actions take the staging paths
            a = a.to(torch.int64)
        elif t % 3 == 2:
            a = a.cpu().numpy()
        tg, tr = g.step(a), ref.step(acts[t])
        assert torch.equal(tg.observations, tr.observations), f"obs t={t}"
        assert torch.equal(tg.rewards, tr.rewards) and torch.equal(tg.discounts, tr.discounts), f"t={t}"
        assert torch.equal(tg.step_types, tr.step_types), f"step_type t={t}"
    assert torch.equal(g.grids, ref.grids) and torch.equal(g.state_words(), ref.state_words())
    assert torch.equal(g.rng, ref.rng)
    g.check()
    assert g.launches <= steps + steps // 8 + 2  # one fused kernel per step (+ reset-ahead batches)


def test_graph_invalid_batch_changes_nothing():
    from paper_2312_12044_b200 import InvalidAction, key_from_seed, policy_keys, random_actions
    params, g, _ = _pair("XLand-MiniGrid-R1-9x9", "trivial", 2048)
    g.reset(key_from_seed(3))
    acts = random_actions(policy_keys(key_from_seed(4), 2048, device=g.device), 0, 8)
    for t in range(4):
        g.step(acts[t])
    g.check()
    before = (g.grids.clone(), g.agent.clone(), g.rng.clone())
    bad = acts[4].clone()
    bad[1234] = 7
    g.step(bad)  # device actions: rejected on the device, raised at check()
    with pytest.raises(InvalidAction):
        g.check()
    assert torch.equal(g.grids, before[0]) and torch.equal(g.agent, before[1]) and torch.equal(g.rng, before[2])
    wide = acts[4].to(torch.int64)
    wide[5] = 256  # would wrap to 0 in u8: must still be rejected
    g.step(wide)
    with pytest.raises(InvalidAction):
        g.check()
    assert torch.equal(g.grids, before[0]) and torch.equal(g.agent, before[1])
    with pytest.raises(InvalidAction):  # host actions: checked before anything is launched
        g.step(np.full(2048, 6))
    g.step(acts[4])
    g.check()
    assert not torch.equal(g.agent, before[1])
