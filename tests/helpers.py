"""Shared test helpers: build the product VecEnv and the oracle from the same
description (golden fixture or benchmark file)."""
from __future__ import annotations

import glob
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "data")
SCEN_NAMES = ("xland", "empty", "empty_random", "door_key", "four_rooms", "unlock", "unlock_pickup")


def golden_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if "policy_stream" not in p)


def load_golden(case):
    return np.load(os.path.join(GOLDEN, case + ".npz"))


def fixture_params(fx):
    from paper_2312_12044_b200 import EnvParams, Layout
    h, w, v, budget, sc, layout, see = (int(x) for x in fx["meta"])
    return EnvParams(layout=Layout(layout), height=h, width=w, view_size=v, max_steps=budget,
                     see_through_walls=bool(see), scenario=SCEN_NAMES[sc])


def fixture_rulesets(fx):
    from paper_2312_12044_b200 import Ruleset
    out = []
    for i in range(len(fx["goals"])):
        rules = tuple(tuple(int(b) for b in fx["rules"][i, s]) for s in range(int(fx["rule_count"][i])))
        objs = tuple(int(b) for b in fx["objs"][i, : int(fx["obj_count"][i])])
        out.append(Ruleset(tuple(int(b) for b in fx["goals"][i]), rules, objs))
    return out


def benchmark_file(config, rows=None):
    """data/<config>-<M>.xmgb: the smallest table by default (parity tests),
    or the one with exactly `rows` rows (e.g. 2**20 for the "1m-style" C3 /
    C4 tables of SURVEY.md §8(d))."""
    paths = glob.glob(os.path.join(DATA, f"{config}-*.xmgb"))
    sized = sorted((int(os.path.basename(p)[len(config) + 1:-5]), p) for p in paths)
    if rows is not None:
        sized = [(m, p) for m, p in sized if m == rows]
    if not sized:
        want = f"{config}-{rows}" if rows else f"{config}-*"
        raise FileNotFoundError(f"no data/{want}.xmgb; run data/make_benchmarks.py")
    return sized[0][1]


def oracle_from_table(params, table, ids, threads=0):
    """OracleVecEnv over the rows `ids` of a TaskTable (left-packed rows)."""
    from oracle.oracle import OracleVecEnv
    rows = table.rows[ids]
    n = len(ids)
    R, O = table.rule_width, table.obj_width
    goals = rows[:, 0].copy().view(np.uint8).reshape(n, 4)
    rc = (rows[:, 1] & 0xFF).astype(np.int32)
    oc = ((rows[:, 1] >> 8) & 0xFF).astype(np.int32)
    from paper_2312_12044_b200.ruleset import HEADER_WORDS as HW_
    rules = rows[:, HW_:HW_ + R].copy().view(np.uint8).reshape(n, max(R, 0), 4) if R else np.zeros((n, 1, 4), np.uint8)
    objs = rows[:, HW_ + R:].copy().view(np.uint8)[:, :O] if O else np.zeros((n, 1), np.uint8)
    return OracleVecEnv(params.height, params.width, params.view_size, params.step_budget, params.scenario,
                        int(params.layout), int(params.see_through_walls), goals, rules if R else np.zeros((n, 1, 4), np.uint8),
                        rc, objs if O else np.zeros((n, 1), np.uint8), oc, threads)
