"""Reset-ahead (include/xmg.h next_*, csrc/xmg_main.cuh): each env's next
trial is pre-built while the current one runs (it depends only on the env's
rng key and task, ref vecenv.py:224-233 via :359-361), and an auto-reset at
stage 2 copies it instead of rebuilding in place.  These tests drive both
paths in one batch — trials whose pre-build is ready (copy) and trials that
end before it is (goal reached early, or a PUT_DOWN that ends the trial:
in-place rebuild) — and require every output and the final state to equal
the oracle and a twin batch with reset-ahead off, bit for bit."""
import numpy as np
import pytest
import torch

from .helpers import benchmark_file, oracle_from_table
from .test_parity_gpu import _assert_state

pytestmark = pytest.mark.gpu


def _pair(env_name, config, n, resample=False, table_rows=None, **param_changes):
    from paper_2312_12044_b200 import VecEnv, load_benchmark, make
    from paper_2312_12044_b200.ruleset import TaskTable
    _, params = make(env_name)
    if param_changes:
        params = params.replace(**param_changes)
    if config:
        bm = load_benchmark(benchmark_file(config, table_rows))
        on = VecEnv(params, n, bm, reset_ahead=True, resample_tasks=resample)
        off = VecEnv(params, n, bm, reset_ahead=False, resample_tasks=resample)
        ora = None if resample else oracle_from_table(params, bm.task_table(), on._ids_host)
    else:
        on = VecEnv(params, n, reset_ahead=True)
        off = VecEnv(params, n, reset_ahead=False)
        ora = oracle_from_table(params, TaskTable(np.zeros((1, 4), np.uint32), 0, 0, 0), np.zeros(n, np.int64))
    return params, on, off, ora


@pytest.mark.parametrize("env_name,config,n,budgets,resample,see", [
    ("MiniGrid-Empty-5x5", None, 4096, 3.2, False, True),          # goals reached early and often
    ("MiniGrid-DoorKey-5x5", None, 4096, 3.2, False, True),
    ("MiniGrid-Unlock", None, 2048, 2.2, False, True),             # the goal is rewritten per reset
    ("XLand-MiniGrid-R1-9x9", "trivial", 8192, 3.1, False, True),  # ~27% of trials end by goal
    ("XLand-MiniGrid-R4-13x13", "medium", 4096, 2.1, False, True),
    ("XLand-MiniGrid-R4-13x13", "medium", 2048, 2.1, True, True),  # resample: the next task comes with the record
    ("XLand-MiniGrid-R4-13x13", "medium", 2048, 2.1, False, False),  # occluded: the record's first observation
    ("XLand-MiniGrid-R9-25x25", "high", 1024, 1.1, False, True),
])
def test_reset_ahead_matches_rebuild_and_oracle(env_name, config, n, budgets, resample, see):
    from paper_2312_12044_b200 import key_from_seed, policy_keys, random_actions
    changes = {} if see else {"see_through_walls": False}
    params, on, off, ora = _pair(env_name, config, n, resample, **changes)
    root = key_from_seed(21)
    a0, b0 = on.reset(root), off.reset(root)
    assert torch.equal(a0.observations, b0.observations)
    if ora is not None:
        np.testing.assert_array_equal(a0.observations.cpu().numpy(), ora.reset(root))
    steps = int(budgets * params.step_budget) + 3
    acts = random_actions(policy_keys(key_from_seed(22), n, device=on.device), 0, steps)
    ah = acts.cpu().numpy()
    copied = rebuilt = put_taken = 0
    for t in range(steps):
        stage = on.reset_ahead_stage.cpu().numpy()
        holding = on.agent_fields()[:, 3].cpu().numpy() != 0
        ta, tb = on.step(acts[t]), off.step(acts[t])
        st = ta.step_types.cpu().numpy()
        last = st == 2
        copied += int((last & (stage == 2)).sum())
        rebuilt += int((last & (stage != 2)).sum())
        # PUT_DOWN while holding something, ending a trial with a record:
        # step_rare's take-over path (xmg_rare.cuh put_consume)
        put_taken += int((last & (stage == 2) & holding & (ah[t] == 4)).sum())
        assert torch.equal(ta.observations, tb.observations), f"obs t={t}"
        assert torch.equal(ta.rewards, tb.rewards) and torch.equal(ta.discounts, tb.discounts), f"t={t}"
        assert torch.equal(ta.step_types, tb.step_types), f"step_type t={t}"
        if ora is not None:
            o, r, d, s = ora.step(ah[t])
            np.testing.assert_array_equal(st, s, err_msg=f"step_type t={t}")
            np.testing.assert_array_equal(ta.observations.cpu().numpy(), o, err_msg=f"obs t={t}")
            np.testing.assert_array_equal(ta.rewards.cpu().numpy(), r.astype(np.float32), err_msg=f"reward t={t}")
    assert torch.equal(on.grids, off.grids)
    assert torch.equal(on.state_words(), off.state_words())
    assert torch.equal(on.rng, off.rng)
    if ora is not None:
        _assert_state(on, ora.grids, ora.agent(), ora.rng, ora.step_count, "final")
    on.check()
    # both auto-reset paths ran: copies of pre-built trials, and rebuilds of
    # trials that ended before their pre-build was ready
    assert copied > 0, "no auto-reset used a pre-built trial"
    assert rebuilt > 0 or env_name.startswith("XLand-MiniGrid-R9"), "no trial ended before its pre-build"
    # the budget burst is served from the records: nearly every budget end copies
    assert copied > rebuilt or env_name.startswith("MiniGrid-Empty")
    assert put_taken > 0 or not env_name.startswith("XLand"), "no PUT_DOWN ended a trial that had a record"


def test_reset_ahead_across_rollouts_and_blocks():
    """Steps, fused rollouts and steps() blocks interleaved on one batch: the
    rollout kernel keeps the stage of a running trial (its records stay
    valid) and clears it when it rebuilds in place; outputs equal a batch with
    reset-ahead off."""
    from paper_2312_12044_b200 import key_from_seed, policy_keys, random_actions
    params, on, off, _ = _pair("XLand-MiniGrid-R1-9x9", "trivial", 4096)
    root = key_from_seed(5)
    on.reset(root)
    off.reset(root)
    pk = policy_keys(key_from_seed(6), 4096, device=on.device)
    total = 3 * params.step_budget
    acts = random_actions(pk, 0, total)
    t = 0
    segment = 0
    while t < total:
        k = min([37, 61, 5][segment % 3], total - t)
        if segment % 3 == 1:  # fused rollout
            ra = on.rollout(k, actions=acts[t:t + k])
            rb = off.rollout(k, actions=acts[t:t + k])
            assert torch.equal(ra.observations, rb.observations) and torch.equal(ra.step_types, rb.step_types)
        elif segment % 3 == 2:  # per-call kernels in one host call
            ra = on.steps(acts[t:t + k], fused=False)
            rb = off.steps(acts[t:t + k], fused=False)
            assert torch.equal(ra.observations, rb.observations) and torch.equal(ra.rewards, rb.rewards)
        else:
            for j in range(k):
                ta, tb = on.step(acts[t + j]), off.step(acts[t + j])
                assert torch.equal(ta.observations, tb.observations), f"t={t + j}"
                assert torch.equal(ta.step_types, tb.step_types)
        t += k
        segment += 1
    assert torch.equal(on.grids, off.grids) and torch.equal(on.state_words(), off.state_words())
    assert torch.equal(on.rng, off.rng)


def test_reset_ahead_stage_lifecycle():
    """Every env's class (e mod classes) gets one batch in every cycle of
    every * classes <= budget - 2 steps (xmg_ahead_plan), so at the
    synchronized budget end every env whose trial ran the whole budget holds a
    pre-built trial (stage 2), and the new trials start at stage 0."""
    from paper_2312_12044_b200 import key_from_seed, policy_keys, random_actions
    params, on, _, _ = _pair("XLand-MiniGrid-R4-13x13", "medium", 2048)
    on.reset(key_from_seed(1))
    b = params.step_budget
    acts = random_actions(policy_keys(key_from_seed(2), 2048, device=on.device), 0, b)
    for t in range(b - 1):
        on.step(acts[t])
    sc = on.agent_fields()[:, 4].cpu().numpy()
    stage = on.reset_ahead_stage.cpu().numpy()
    full = sc == b - 1  # trials that started at the reset and reach the budget next step
    assert full.sum() > 1900
    assert (stage[full] == 2).all()
    ts = on.step(acts[b - 1])
    last = ts.step_types.cpu().numpy() == 2
    assert last[full].all()
    assert (on.reset_ahead_stage.cpu().numpy()[full] == 0).all()
    assert (on.agent_fields()[:, 4].cpu().numpy()[full] == 0).all()
    # the take-overs flipped those envs to the second grid buffer: the
    # accessors follow the buffer bit
    flipped = ((on.agent[:, 0] >> 20) & 1).cpu().numpy().astype(bool)
    assert flipped[full].all()
    i = int(np.flatnonzero(flipped)[0])
    g = on.grids
    assert on.env_state(i).grid.cells == g[i].cpu().numpy().tobytes()
    cells = g[i].clone()
    cells[0] = 0x77
    on.set_grid(i, cells)
    assert torch.equal(on.grids[i], cells) and on._next_grids[i * cells.numel()].item() == 0x77
