"""GPU parity: the sm_100a step (through the C ABI) against the reference's
golden fixtures and the CPU oracle.

Bars (BASELINE.json north_star): grid, agent pose/pocket, step count, rng
keys, observations, discounts and step types bit-exact; rewards equal to
float32(reference float64) bit for bit (i.e. well inside 1 ulp of f32).
"""
import numpy as np
import pytest
import torch

from .helpers import (benchmark_file, fixture_params, fixture_rulesets, golden_cases, load_golden,
                      oracle_from_table)

pytestmark = pytest.mark.gpu


def _unpack_agent(vec):
    a = vec.agent_fields().cpu().numpy()
    return a[:, :4].astype(np.int32), a[:, 4]


def _assert_state(vec, grids, agent, rng, sc, msg):
    np.testing.assert_array_equal(vec.grids.cpu().numpy(), grids, err_msg=f"grid {msg}")
    ag, stc = _unpack_agent(vec)
    np.testing.assert_array_equal(ag, agent, err_msg=f"agent {msg}")
    np.testing.assert_array_equal(vec.rng.cpu().numpy().view(np.uint64), rng, err_msg=f"rng {msg}")
    np.testing.assert_array_equal(stc, sc, err_msg=f"step_count {msg}")


@pytest.mark.parametrize("case", golden_cases())
def test_golden_lockstep(case):
    """Every step of every golden trace, via VecEnv -> libxmg.so."""
    from paper_2312_12044_b200 import Key, VecEnv
    fx = load_golden(case)
    params = fixture_params(fx)
    n = len(fx["goals"])
    rulesets = fixture_rulesets(fx) if params.scenario == "xland" else None
    vec = VecEnv(params, n, rulesets)
    ts = vec.reset(Key(int(fx["key"][0]), int(fx["key"][1])))
    np.testing.assert_array_equal(ts.observations.cpu().numpy(), fx["obs0"])
    assert (ts.step_types.cpu().numpy() == 0).all()
    _assert_state(vec, fx["grids0"], fx["agent0"], fx["rng0"], fx["step_count0"], "after reset")
    acts = torch.from_numpy(fx["actions"]).cuda()
    for t in range(len(fx["actions"])):
        ts = vec.step(acts[t])
        obs, rew, disc, st = ts.numpy()
        np.testing.assert_array_equal(obs, fx["obs"][t], err_msg=f"obs t={t}")
        np.testing.assert_array_equal(rew, fx["reward"][t].astype(np.float32), err_msg=f"reward t={t}")
        np.testing.assert_array_equal(disc, fx["discount"][t].astype(np.float32))
        np.testing.assert_array_equal(st, fx["step_type"][t])
        _assert_state(vec, fx["grids"][t], fx["agent"][t], fx["rng"][t], fx["step_count"][t], f"t={t}")
    vec.check()


@pytest.mark.parametrize("config,env_name,n,steps", [
    ("trivial", "XLand-MiniGrid-R1-9x9", 8192, 520),
    ("medium", "XLand-MiniGrid-R4-13x13", 8192, 1100),
    ("high", "XLand-MiniGrid-R9-25x25", 2048, 1900),
    (None, "MiniGrid-DoorKey-8x8", 4096, 400),
    (None, "MiniGrid-Empty-8x8", 4096, 256),
    (None, "MiniGrid-UnlockPickUp", 2048, 500),
    (None, "MiniGrid-FourRooms", 1024, 1100),
])
def test_random_policy_vs_oracle(config, env_name, n, steps):
    """Thousands of envs under the on-device random policy, compared with the
    oracle on identical keys, tasks and actions (state every 25 steps, all
    outputs every step)."""
    from paper_2312_12044_b200 import (VecEnv, key_from_seed, load_benchmark, make, policy_keys,
                                       random_actions)
    _, params = make(env_name)
    if config:
        bm = load_benchmark(benchmark_file(config))
        vec = VecEnv(params, n, bm)
        ora = oracle_from_table(params, bm.task_table(), vec._ids_host)
    else:
        vec = VecEnv(params, n)
        from oracle.oracle import OracleVecEnv
        ora = OracleVecEnv(params.height, params.width, params.view_size, params.step_budget, params.scenario,
                           int(params.layout), 1, np.zeros((n, 4), np.uint8), np.zeros((n, 1, 4), np.uint8),
                           np.zeros(n, np.int32), np.zeros((n, 1), np.uint8), np.zeros(n, np.int32), 0)
    root = key_from_seed(0)
    ts = vec.reset(root)
    obs0 = ora.reset(root)
    np.testing.assert_array_equal(ts.observations.cpu().numpy(), obs0)
    acts = random_actions(policy_keys(key_from_seed(1), n, device=vec.device), 0, steps)
    acts_h = acts.cpu().numpy()
    for t in range(steps):
        ts = vec.step(acts[t])
        o, r, d, s = ora.step(acts_h[t])
        obs, rew, disc, st = ts.numpy()
        np.testing.assert_array_equal(st, s, err_msg=f"step_type t={t}")
        np.testing.assert_array_equal(rew, r.astype(np.float32), err_msg=f"reward t={t}")
        np.testing.assert_array_equal(disc, d.astype(np.float32))
        np.testing.assert_array_equal(obs, o, err_msg=f"obs t={t}")
        if t % 25 == 0 or t == steps - 1:
            _assert_state(vec, ora.grids, ora.agent(), ora.rng, ora.step_count, f"t={t}")
    vec.check()


def test_philox_kat_and_keys():
    """Philox vs numpy.random.Philox (ref tests/test_rng.py:22-30), split_batch
    and the random policy stream vs the oracle."""
    from oracle import oracle as O
    from paper_2312_12044_b200 import key_from_seed, philox, random_actions, split_batch
    rng = np.random.default_rng(3)
    ctr = rng.integers(0, 2**63, size=(512, 4), dtype=np.uint64)
    key = rng.integers(0, 2**63, size=(512, 2), dtype=np.uint64)
    out = philox(torch.from_numpy(ctr.view(np.int64)).cuda(), torch.from_numpy(key.view(np.int64)).cuda())
    np.testing.assert_array_equal(out.cpu().numpy().view(np.uint64), O.philox(ctr, key))
    for i in range(0, 512, 37):
        c = ctr[i].copy()
        c[0] -= 1
        ref = np.random.Philox(counter=c, key=key[i]).random_raw(4)
        np.testing.assert_array_equal(out[i].cpu().numpy().view(np.uint64), ref)
    root = key_from_seed(20240601)
    ks = split_batch(root, 1000, offset=123).cpu().numpy().view(np.uint64)
    k0, k1 = O.split_batch((root.hi, root.lo), 1000, offset=123)
    np.testing.assert_array_equal(ks[:, 0], k0)
    np.testing.assert_array_equal(ks[:, 1], k1)
    acts = random_actions(torch.from_numpy(ks.view(np.int64)).cuda(), 5, 37).cpu().numpy()
    np.testing.assert_array_equal(acts, O.random_actions(k0, k1, 5, 37))


def test_invalid_device_actions_mutate_nothing():
    from paper_2312_12044_b200 import EnvParams, InvalidAction, VecEnv, key_from_seed
    vec = VecEnv(EnvParams(), 64)
    vec.reset(key_from_seed(0))
    g = vec.grids.clone()
    a = vec.agent.clone()
    bad = torch.zeros(64, dtype=torch.int64, device="cuda")
    bad[17] = 6
    vec.step(bad)
    with pytest.raises(InvalidAction):
        vec.check()
    assert torch.equal(vec.grids, g) and torch.equal(vec.agent, a)
    with pytest.raises(InvalidAction):
        vec.step(np.array([0, 1]))
    strict = VecEnv(EnvParams(), 64, strict=True)
    strict.reset(key_from_seed(0))
    with pytest.raises(InvalidAction):
        strict.step(bad)


@pytest.mark.parametrize("dtype", [torch.uint8, torch.int32, torch.int64])
def test_validation_catches_every_position(dtype):
    """Device-side validation (vectorised body, scalar head / tail) rejects a
    single bad action anywhere, for each dtype and a misaligned view."""
    from paper_2312_12044_b200 import EnvParams, InvalidAction, VecEnv, key_from_seed
    n = 1000
    vec = VecEnv(EnvParams(), n)
    vec.reset(key_from_seed(0))
    store = torch.zeros(n + 8, dtype=dtype, device="cuda")
    for shift in (0, 1, 3):
        acts = store[shift:shift + n]
        acts.fill_(5)
        vec.step(acts)
        vec.check()  # all valid
        for pos in (0, 1, 2, 15, 16, 17, 500, n - 17, n - 2, n - 1):
            for badv in ((6, 255) if dtype == torch.uint8 else (6, -1, 1 << 20)):
                acts.fill_(2)
                acts[pos] = badv
                g = vec.grids.clone()
                vec.step(acts)
                with pytest.raises(InvalidAction):
                    vec.check()
                assert torch.equal(vec.grids, g), (shift, pos, badv)


def test_shards_reproduce_the_global_batch():
    """Env-range shards with global key offsets == one big batch
    (ref tests/test_harness.py:105-122, tests/test_acceptance.py:494-517)."""
    from paper_2312_12044_b200 import (VecEnv, key_from_seed, load_benchmark, make, policy_keys,
                                       random_actions)
    _, params = make("XLand-MiniGrid-R4-13x13")
    bm = load_benchmark(benchmark_file("medium"))
    n, steps = 4096, 600
    root = key_from_seed(0)
    acts = random_actions(policy_keys(key_from_seed(1), n, device="cuda"), 0, steps)
    whole = VecEnv(params, n, bm)
    whole.reset(root)
    parts = [VecEnv(params, n // 4, bm, global_offset=g * (n // 4)) for g in range(4)]
    for p in parts:
        p.reset(root)
    for t in range(steps):
        w = whole.step(acts[t])
        for g, p in enumerate(parts):
            s = p.step(acts[t, g * (n // 4):(g + 1) * (n // 4)])
            if t % 50 == 0 or t == steps - 1:
                sl = slice(g * (n // 4), (g + 1) * (n // 4))
                assert torch.equal(s.observations, w.observations[sl])
                assert torch.equal(s.rewards, w.rewards[sl])
                assert torch.equal(p.grids, whole.grids[sl])


@pytest.mark.parametrize("knobs", [{"XMG_AHEAD": "0"}, {"XMG_AGENT_ROWS": "0"}, {"XMG_PDL": "0"}, {"XMG_RARE_PDL": "0"}, {"XMG_RARE_CTAS": "2"}])
def test_tuning_knobs_keep_parity(knobs):
    """The library's tuning switches (reset-ahead off, whole task rows instead of
    the compact agent-rule rows, no programmatic
    overlap at all or none for step_rare, a small step_rare grid) change scheduling only: a fresh process
    with each switch reproduces the oracle bit for bit (switches are read once
    per process)."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, sys
sys.path.insert(0, "tests")
from helpers import benchmark_file, oracle_from_table
from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions
for env_name, cfg, n, steps in (("XLand-MiniGrid-R4-13x13", "medium", 2048, 520), ("MiniGrid-DoorKey-8x8", None, 1024, 200)):
    _, params = make(env_name)
    if cfg:
        bm = load_benchmark(benchmark_file(cfg)); vec = VecEnv(params, n, bm)
        ora = oracle_from_table(params, bm.task_table(), vec._ids_host)
    else:
        from paper_2312_12044_b200.ruleset import TaskTable
        vec = VecEnv(params, n)
        ora = oracle_from_table(params, TaskTable(np.zeros((1, 4), np.uint32), 0, 0, 0), np.zeros(n, np.int64))
    root = key_from_seed(0)
    assert np.array_equal(vec.reset(root).observations.cpu().numpy(), ora.reset(root))
    acts = random_actions(policy_keys(key_from_seed(1), n, device="cuda"), 0, steps)
    ah = acts.cpu().numpy()
    for t in range(steps):
        ts = vec.step(acts[t]); o, r, d, s = ora.step(ah[t])
        assert np.array_equal(ts.observations.cpu().numpy(), o), t
        assert np.array_equal(ts.rewards.cpu().numpy(), r.astype(np.float32)), t
        assert np.array_equal(ts.step_types.cpu().numpy(), s), t
    assert np.array_equal(vec.grids.cpu().numpy(), ora.grids)
    vec.check()
print("ok")
'''
    from .conftest import ROOT
    env = dict(os.environ, **knobs)
    res = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-3000:]


@pytest.mark.parametrize("env_name,config", [("XLand-MiniGrid-R4-13x13", "medium"),
                                             ("XLand-MiniGrid-R9-25x25", "high"),
                                             ("MiniGrid-DoorKey-8x8", None)])
def test_checked_build_parity(env_name, config):
    """The XMG_CHECKS build (device asserts on every window / grid / queue
    index) runs the soak workload -- pipelined steps with a slice vs the
    oracle every step, then the fused rollout vs the stepped state -- without
    a trap (compute-sanitizer is not available on this pool)."""
    import os
    import subprocess
    import sys
    from .conftest import ROOT
    lib = os.path.join(ROOT, "paper_2312_12044_b200", "libxmg_checked.so")
    assert os.path.exists(lib), "build() makes libxmg_checked.so"
    env = dict(os.environ, XMG_LIB=lib)
    args = [sys.executable, os.path.join(ROOT, "tools", "soak.py"), "1100", "8192", env_name]
    if config:
        args.append(config)
    res = subprocess.run(args, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize.py"), "1000"], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]


@pytest.mark.parametrize("env_name,config,v,see", [
    ("XLand-MiniGrid-R9-25x25", "high", 9, True),
    ("XLand-MiniGrid-R6-19x19", "medium", 11, True),
    ("MiniGrid-DoorKey-16x16", None, 3, True),
    ("XLand-MiniGrid-R2-17x17", "small", 7, False),
    ("MiniGrid-EmptyRandom-16x16", None, 13, True),
])
def test_view_sizes_and_layouts_vs_oracle(env_name, config, v, see):
    """Non-default views (3..13 cells: other window chunk counts / generic
    observation path), R6 fixed doors, occlusion at v=7, 16x16 ports."""
    from dataclasses import replace
    from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions
    from paper_2312_12044_b200.ruleset import TaskTable
    _, params = make(env_name)
    params = replace(params, view_size=v, see_through_walls=see)
    n, steps = 1024, min(params.step_budget + 5, 800)
    if config:
        bm = load_benchmark(benchmark_file(config))
        vec = VecEnv(params, n, bm)
        ora = oracle_from_table(params, bm.task_table(), vec._ids_host)
    else:
        vec = VecEnv(params, n)
        ora = oracle_from_table(params, TaskTable(np.zeros((1, 4), np.uint32), 0, 0, 0), np.zeros(n, np.int64))
    root = key_from_seed(5)
    np.testing.assert_array_equal(vec.reset(root).observations.cpu().numpy(), ora.reset(root))
    acts = random_actions(policy_keys(key_from_seed(6), n, device=vec.device), 0, steps)
    ah = acts.cpu().numpy()
    for t in range(steps):
        ts = vec.step(acts[t])
        o, r, d, s = ora.step(ah[t])
        np.testing.assert_array_equal(ts.observations.cpu().numpy(), o, err_msg=f"obs t={t}")
        np.testing.assert_array_equal(ts.rewards.cpu().numpy(), r.astype(np.float32))
        np.testing.assert_array_equal(ts.step_types.cpu().numpy(), s)
    np.testing.assert_array_equal(vec.grids.cpu().numpy(), ora.grids)
    vec.check()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_vecenv_on_a_non_current_device():
    """A VecEnv on cuda:1 while cuda:0 is current launches on its own GPU
    (libxmg uses the current device; VecEnv makes its device current per call)
    and equals the same batch on cuda:0, including the >48 KB rollout kernel
    whose attributes are set per device."""
    from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions
    _, params = make("XLand-MiniGrid-R4-13x13")
    bm = load_benchmark(benchmark_file("medium"))
    torch.cuda.set_device(0)
    a = VecEnv(params, 1024, bm, device="cuda:0")
    b = VecEnv(params, 1024, bm, device="cuda:1")
    a.reset(key_from_seed(1))
    b.reset(key_from_seed(1))
    acts = random_actions(policy_keys(key_from_seed(2), 1024, device="cuda:0"), 0, 40)
    for t in range(20):
        ta, tb = a.step(acts[t]), b.step(acts[t].to("cuda:1"))
        assert torch.equal(ta.observations.cpu(), tb.observations.cpu())
    ra = a.rollout(20, actions=acts[20:40])
    rb = b.rollout(20, actions=acts[20:40].to("cuda:1"))
    assert torch.equal(ra.observations.cpu(), rb.observations.cpu())
    assert torch.equal(a.grids.cpu(), b.grids.cpu()) and torch.equal(a.state_words().cpu(), b.state_words().cpu())
    assert torch.cuda.current_device() == 0
