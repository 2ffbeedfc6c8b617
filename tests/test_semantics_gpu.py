"""GPU: the reference's scripted semantics tests, run through VecEnv.

* ref tests/test_acceptance.py:345-418 — the put-near merge on a hand-built
  6x6 room (TILE_NEAR rule fires on PUT_DOWN, AGENT_HOLD goal, reward
  1 - 0.9 * (6 / 30), terminal discount 0) and budget exhaustion;
* ref tests/test_vecenv.py:149-160 — an empty ruleset ends trials on the
  budget only;
* ref tests/test_vecenv.py:188-208, tests/test_harness.py:125-133 — the
  constructor / reset errors.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

FLOOR, WALL = 57, 72


def _pack(r, c, d, pocket=0, sc=0):
    return r | (c << 8) | (d << 16) | (pocket << 24) | (sc << 32)


def _merge_env(max_steps):
    from paper_2312_12044_b200 import EnvParams, Ruleset, VecEnv
    a, b, out = 6 * 16 + 6, 6 * 16 + 7, 5 * 16 + 3  # purple square, yellow square, red ball
    rs = Ruleset(goal=(1, out, 0, 0), rules=((3, a, b, out),), init_objects=(a, b)).validate()
    params = EnvParams(height=6, width=6, max_steps=max_steps, ruleset=rs)
    vec = VecEnv(params, 1)
    cells = np.full(36, FLOOR, np.uint8)
    for i in range(6):
        for j in (0, 5):
            cells[i * 6 + j] = WALL
            cells[j * 6 + i] = WALL
    cells[3 * 6 + 1] = a  # purple square, west of the agent
    cells[1 * 6 + 3] = b  # yellow square, by the north wall
    goal = rs.goal[0] | (rs.goal[1] << 8) | (rs.goal[2] << 16) | (rs.goal[3] << 24)
    word = np.array([_pack(3, 2, 3), goal], np.uint64).view(np.int64)  # (3, 2) facing LEFT, task 0
    vec.agent[0] = torch.from_numpy(word).cuda()
    vec.set_grid(0, cells)
    return vec, a, b, out


def test_put_near_merge_and_terminal_discounts():
    vec, a, b, out = _merge_env(30)
    script = [3, 2, 0, 2, 4, 3]  # PICK_UP, TURN_RIGHT, MOVE, TURN_RIGHT, PUT_DOWN, PICK_UP
    grids = []
    for t, act in enumerate(script, start=1):
        ts = vec.step(np.array([act]))
        grids.append(vec.grids[0].cpu().numpy().copy())
        _, rew, disc, st = ts.numpy()
        if t < len(script):
            assert st[0] == 1 and rew[0] == 0.0 and disc[0] == 1.0, t
    assert st[0] == 2 and disc[0] == 0.0
    assert rew[0] == np.float32(1.0 - 0.9 * (6 / 30))
    g5 = grids[4]  # the merged state, one step before the pickup
    assert g5[2 * 6 + 3] == out and g5[1 * 6 + 3] == FLOOR
    assert (g5 == a).sum() == 0 and (g5 == b).sum() == 0 and (g5 == out).sum() == 1
    g6 = grids[5]  # the terminal step's grid is the NEXT trial's (auto-reset) ...
    assert g6.shape == (36,)
    # ... so check the pocket through a replay that stops before the reset:
    vec2, *_ = _merge_env(30)
    for act in script[:5]:
        vec2.step(np.array([act]))
    pocket_before = (int(vec2.agent[0, 0].item()) >> 24) & 0xFF
    assert pocket_before == 0  # the square was put down and merged away

    # budget exhaustion is also a discount-0 terminal with reward 0
    short, *_ = _merge_env(4)
    for t in range(1, 5):
        _, rew, disc, st = short.step(np.array([1])).numpy()
        if t < 4:
            assert st[0] == 1 and disc[0] == 1.0
    assert st[0] == 2 and disc[0] == 0.0 and rew[0] == 0.0


def test_empty_ruleset_trials_end_on_budget_only():
    from paper_2312_12044_b200 import EnvParams, VecEnv, key_from_seed
    vec = VecEnv(EnvParams(max_steps=30), 16)
    vec.reset(key_from_seed(20240601))
    rng = np.random.default_rng(0)
    for t in range(1, 61):
        _, rew, disc, st = vec.step(rng.integers(0, 6, 16)).numpy()
        last = t % 30 == 0
        assert (st == (2 if last else 1)).all() and (rew == 0.0).all() and (disc == (0.0 if last else 1.0)).all()


def test_constructor_and_reset_errors():
    from paper_2312_12044_b200 import EnvParams, GridFull, Ruleset, VecEnv, key_from_seed, load_benchmark
    from .helpers import benchmark_file
    task = Ruleset(goal=(3, 85, 0, 0), init_objects=(85,) * 60)  # 60 > 49 free cells
    with pytest.raises(GridFull):
        VecEnv(EnvParams(ruleset=task), 2)
    bm = load_benchmark(benchmark_file("trivial"))
    with pytest.raises(ValueError):
        VecEnv(EnvParams(), 2, rulesets=[bm.get_ruleset(i) for i in range(3)])
    with pytest.raises(ValueError):
        VecEnv(EnvParams(), 0)
    vec = VecEnv(EnvParams(), 4)
    with pytest.raises(ValueError):
        vec.reset_with_keys(np.zeros(3, np.uint64), np.zeros(3, np.uint64))
    vec.reset(key_from_seed(1))
    st = vec.env_state(2)
    assert st.step_count == 0 and not st.goal_reached and st.grid.height == 9


def test_compute_obs_false_skips_only_observations():
    """ref vecenv.py:295 step(actions, compute_obs=False): no observation
    record, identical rewards / discounts / step types and state."""
    from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions
    from .helpers import benchmark_file
    _, params = make("XLand-MiniGrid-R4-13x13")
    bm = load_benchmark(benchmark_file("medium"))
    a, b = VecEnv(params, 1024, bm), VecEnv(params, 1024, bm)
    assert a.reset(key_from_seed(2), compute_obs=False).observations is None
    b.reset(key_from_seed(2))
    acts = random_actions(policy_keys(key_from_seed(3), 1024, device="cuda"), 0, 520)
    for t in range(520):
        ta, tb = a.step(acts[t], compute_obs=False), b.step(acts[t])
        assert ta.observations is None
        assert torch.equal(ta.rewards, tb.rewards) and torch.equal(ta.step_types, tb.step_types)
        assert torch.equal(ta.discounts, tb.discounts)
    assert torch.equal(a.grids, b.grids) and torch.equal(a.state_words(), b.state_words()) and torch.equal(a.rng, b.rng)
