"""Generate golden lockstep fixtures from the REFERENCE implementation.

Run in the build container (the reference is not present on the GPU box):

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python /root/repo/tests/golden/make_golden.py

Each case drives the reference ``rulegrid.VecEnv`` (pinned to the scalar
engine by the reference's own tests/test_vecenv.py:45-66) with a fixed root
key and action matrix and records, per step, the VecTimeStep fields and the
mirrored per-env state (``env_state(i)``: grid, agent, rng, step_count).  The
resulting ``tests/golden/<case>.npz`` files pin the oracle (oracle/) and the
CUDA path (tests/test_parity_gpu.py) to the reference bit for bit.

A subset of cases is additionally replayed through the scalar
``Environment`` here, so the fixtures are checked against both reference
engines before they are written.
"""

from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np

from rulegrid.benchgen import CONFIGS, generate_benchmark
from rulegrid.env import Environment, EnvParams
from rulegrid.layouts import Layout
from rulegrid.registry import make
from rulegrid.rng import fold_in, key_from_seed, random_words, split
from rulegrid.ruleset import Ruleset
from rulegrid.vecenv import VecEnv

OUT = os.path.dirname(os.path.abspath(__file__))
ROOT = key_from_seed(20240601)  # same root as reference tests/test_vecenv.py:19
SCEN = {"xland": 0, "empty": 1, "empty_random": 2, "door_key": 3, "four_rooms": 4,
        "unlock": 5, "unlock_pickup": 6}


def pack_tasks(tasks, n):
    goals = np.zeros((n, 4), np.uint8)
    rules = np.zeros((n, 18, 4), np.uint8)
    objs = np.zeros((n, 18), np.uint8)
    rc = np.zeros(n, np.int32)
    oc = np.zeros(n, np.int32)
    for i in range(n):
        t = tasks[i] if tasks else Ruleset()
        goals[i] = t.goal
        for s, r in enumerate(t.active_rules):
            rules[i, s] = r
        rc[i] = len(t.active_rules)
        ob = t.active_objects
        objs[i, : len(ob)] = ob
        oc[i] = len(ob)
    return goals, rules, rc, objs, oc


def snapshot(vec, n):
    hw = vec.params.height * vec.params.width
    grids = np.zeros((n, hw), np.uint8)
    agent = np.zeros((n, 4), np.int32)
    rng = np.zeros((n, 2), np.uint64)
    sc = np.zeros(n, np.int64)
    for i in range(n):
        s = vec.env_state(i)
        grids[i] = np.frombuffer(s.grid.cells, np.uint8)
        agent[i] = (s.agent.position.row, s.agent.position.col, int(s.agent.direction), s.agent.pocket)
        rng[i] = (s.rng.hi, s.rng.lo)
        sc[i] = s.step_count
    return grids, agent, rng, sc


def scalar_check(params, tasks, key, actions, recs):
    """Replay through the scalar engine (ref tests/test_vecenv.py:23-42)."""
    env = Environment()
    n = actions.shape[1]
    keys = split(key, n)
    plist = [dataclasses.replace(params, ruleset=tasks[i]) if tasks else params for i in range(n)]
    steps = [env.reset(plist[i], keys[i]) for i in range(n)]
    for t, row in enumerate(actions):
        for i in range(n):
            ts = env.step(plist[i], steps[i], int(row[i]))
            assert ts.reward == recs["reward"][t, i]
            assert int(ts.step_type) == recs["step_type"][t, i]
            ts = env.auto_reset(plist[i], ts)
            steps[i] = ts
            assert (ts.observation == recs["obs"][t, i]).all()
            assert np.frombuffer(ts.state.grid.cells, np.uint8).tobytes() == recs["grids"][t, i].tobytes()


def run_case(name, params, tasks, n, steps, seed, *, action_p=None, scalar=False, key=ROOT):
    rng = np.random.default_rng(seed)
    actions = rng.choice(6, size=(steps, n), p=action_p).astype(np.int64)
    vec = VecEnv(params, n, rulesets=tasks)
    first = vec.reset(key)
    g0, a0, r0, s0 = snapshot(vec, n)
    hw = params.height * params.width
    v = params.view_size
    recs = {
        "obs": np.zeros((steps, n, v, v, 2), np.uint8),
        "reward": np.zeros((steps, n), np.float64),
        "discount": np.zeros((steps, n), np.float64),
        "step_type": np.zeros((steps, n), np.int8),
        "grids": np.zeros((steps, n, hw), np.uint8),
        "agent": np.zeros((steps, n, 4), np.int32),
        "rng": np.zeros((steps, n, 2), np.uint64),
        "step_count": np.zeros((steps, n), np.int64),
    }
    for t in range(steps):
        ts = vec.step(actions[t])
        recs["obs"][t] = ts.observations
        recs["reward"][t] = ts.rewards
        recs["discount"][t] = ts.discounts
        recs["step_type"][t] = ts.step_types
        g, a, r, s = snapshot(vec, n)
        recs["grids"][t], recs["agent"][t], recs["rng"][t], recs["step_count"][t] = g, a, r, s
    if scalar:
        scalar_check(params, tasks, key, actions, recs)
    goals, rules, rc, objs, oc = pack_tasks(tasks, n)
    meta = np.array([params.height, params.width, params.view_size, params.step_budget,
                     SCEN[params.scenario], int(params.layout), int(params.see_through_walls)], np.int64)
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"),
        meta=meta, key=np.array([key.hi, key.lo], np.uint64), actions=actions.astype(np.uint8),
        goals=goals, rules=rules, rule_count=rc, objs=objs, obj_count=oc,
        obs0=first.observations, grids0=g0, agent0=a0, rng0=r0, step_count0=s0,
        **recs,
    )
    fires = int((recs["reward"] > 0).sum())
    print(f"{name}: {n} envs x {steps} steps, goal hits {fires}, "
          f"LAST {int((recs['step_type'] == 2).sum())}", flush=True)


def stress_tasks(n, h, w, seed):
    """Random tasks on a small room exercising every rule and goal kind.

    Inputs are drawn from a tiny object alphabet that is placed several
    times, so AGENT_NEAR / TILE_NEAR conditions hold often and slots chain.
    """
    rng = np.random.default_rng(seed)
    alphabet = [5 * 16 + 3, 6 * 16 + 4, 7 * 16 + 5, 9 * 16 + 7, 13 * 16 + 8]  # ball, square, pyramid, key, hex
    outs = alphabet + [14 * 16 + 10, 57, 8 * 16 + 4]  # star, floor, goal
    tasks = []
    for _ in range(n):
        rules = []
        for _ in range(18):
            kind = int(rng.integers(1, 12))
            a = int(rng.choice(alphabet))
            b = int(rng.choice(alphabet)) if 3 <= kind <= 7 else 0
            rules.append((kind, a, b, int(rng.choice(outs))))
        gk = int(rng.integers(1, 15))
        if gk == 5:
            goal = (5, int(rng.integers(1, h - 1)), int(rng.integers(1, w - 1)), 0)
        elif gk == 6:
            goal = (6, int(rng.choice(outs[:-2])), int(rng.integers(0, h + 1)), int(rng.integers(0, w + 1)))
        elif gk in (4, 7, 8, 9, 10):
            goal = (gk, int(rng.choice(outs)), int(rng.choice(alphabet)), 0)
        else:
            goal = (gk, int(rng.choice(outs)), 0, 0)
        objs = tuple(int(rng.choice(alphabet)) for _ in range(int(rng.integers(4, 11))))
        tasks.append(Ruleset(goal=goal, rules=tuple(rules), init_objects=objs))
    return tasks


def main():
    only = set(sys.argv[1:])

    def want(name):
        return not only or name in only

    bench = {c: generate_benchmark(CONFIGS[c], 16) for c in ("trivial", "small", "medium", "high")}
    if want("trivial_r1"):
        run_case("trivial_r1", EnvParams(), bench["trivial"][:6], 6, 700, 1, scalar=True)
    if want("medium_r1"):
        run_case("medium_r1", EnvParams(), bench["medium"][:6], 6, 600, 2, scalar=True)
    if want("high_r4_13"):
        _, p = make("XLand-MiniGrid-R4-13x13")
        run_case("high_r4_13", p, bench["high"][:4], 4, 500, 3)
    if want("medium_r4_13"):
        _, p = make("XLand-MiniGrid-R4-13x13")
        run_case("medium_r4_13", p, bench["medium"][:8], 8, 1100, 11, key=key_from_seed(0))
    if want("high_r9_25"):
        _, p = make("XLand-MiniGrid-R9-25x25")
        run_case("high_r9_25", p, bench["high"][:4], 4, 1900, 12)
    if want("high_r6_19"):
        _, p = make("XLand-MiniGrid-R6-19x19")
        run_case("high_r6_19", p, bench["high"][4:8], 4, 1200, 13)
    if want("small_r2_13"):
        _, p = make("XLand-MiniGrid-R2-13x13")
        run_case("small_r2_13", p, bench["small"][:6], 6, 600, 14)
    ports = [("MiniGrid-Empty-8x8", 8, 400), ("MiniGrid-DoorKey-8x8", 8, 450),
             ("MiniGrid-DoorKey-5x5", 6, 300), ("MiniGrid-UnlockPickUp", 4, 700),
             ("MiniGrid-Unlock", 4, 700), ("MiniGrid-FourRooms", 3, 1100),
             ("MiniGrid-EmptyRandom-6x6", 4, 350), ("MiniGrid-Empty-5x5", 4, 200)]
    for env_name, n, steps in ports:
        name = "port_" + env_name.split("-", 1)[1].replace("-", "_").lower()
        if want(name):
            _, p = make(env_name)
            run_case(name, p, None, n, steps, 4, scalar=env_name.endswith("8x8"))
    if want("occluded_small"):
        run_case("occluded_small", EnvParams(see_through_walls=False, view_size=5), bench["small"][:3], 3, 300, 5,
                 scalar=True)
    if want("occluded_r4_13_v7"):
        p = EnvParams(layout=Layout.R4, height=13, width=13, see_through_walls=False, view_size=7)
        run_case("occluded_r4_13_v7", p, bench["medium"][8:12], 4, 600, 6)
    if want("stress_6x6"):
        p = EnvParams(height=6, width=6, max_steps=60)
        tasks = stress_tasks(48, 6, 6, 7)
        # bias towards pick/put/toggle so every rule kind fires often
        run_case("stress_6x6", p, tasks, 48, 500, 8, action_p=[0.3, 0.1, 0.1, 0.2, 0.2, 0.1], scalar=True)
    if want("stress_7x9_v3"):
        p = EnvParams(height=7, width=9, max_steps=80, view_size=3)
        tasks = stress_tasks(32, 7, 9, 9)
        run_case("stress_7x9_v3", p, tasks, 32, 500, 10, action_p=[0.3, 0.1, 0.1, 0.2, 0.2, 0.1])
    if want("policy_stream"):
        # batch-invariance stream: env i's actions are random_words(fold_in(ROOT, i)) % 6
        # (ref tests/test_vecenv.py:118-141); also pins the random-policy word stream.
        n, steps = 8, 300
        words = np.array([random_words(fold_in(ROOT, i), steps) for i in range(n)], dtype=np.uint64)
        np.savez_compressed(os.path.join(OUT, "policy_stream.npz"), key=np.array([ROOT.hi, ROOT.lo], np.uint64),
                            words=words)
        print("policy_stream written")


if __name__ == "__main__":
    main()
