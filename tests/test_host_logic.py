"""Host-side mirror of the reference API (no GPU): registry, parameters,
layout geometry, benchmark files and the device task-table packing.
Mirrors reference tests/test_env.py:248-262, tests/test_layouts.py:48-82 and
tests/test_benchio.py:48-233."""
import os
import struct
import zlib

import numpy as np
import pytest

from paper_2312_12044_b200 import (EnvParams, FormatError, InvalidProportion, Layout, LayoutTooSmall, Ruleset,
                                   UnknownBenchmark, UnknownEnvironment, key_from_seed, load_benchmark, load_named,
                                   make, plan_layout, randint, registered_environments, save_benchmark)
from paper_2312_12044_b200.ruleset import HEADER_WORDS, Benchmark, pack_raw_rows, pack_rulesets

from .helpers import GOLDEN, benchmark_file, load_golden


def test_registry_names_and_budgets():
    names = registered_environments()
    assert len(names) == 30
    assert sum(1 for n in names if n.startswith("XLand-MiniGrid-R")) == 15
    assert make("XLand-MiniGrid-R9-25x25")[1].step_budget == 1875
    assert make("XLand-MiniGrid-R4-13x13")[1].step_budget == 507
    assert make("XLand-MiniGrid-R1-9x9")[1].step_budget == 243
    for n in names:
        p = make(n)[1]
        if n.startswith("XLand"):
            assert p.step_budget == 3 * p.height * p.width
    with pytest.raises(UnknownEnvironment):
        make("MiniGrid-Foo")
    with pytest.raises(ValueError):
        EnvParams(view_size=4)
    with pytest.raises(ValueError):
        EnvParams(scenario="nope")


def test_layout_geometry():
    plan = plan_layout(Layout.R4, 13, 13)
    base = plan.base_cells().reshape(13, 13)
    assert plan.wall_rows == (6,) and plan.wall_cols == (6,)
    assert int((base == 72).sum()) == 4 * 12 + 2 * 11 - 1  # border + one cross
    assert len(plan.door_segments) == 4
    assert plan_layout(Layout.R6, 19, 19).fixed_doors
    assert len(plan_layout(Layout.R9, 25, 25).door_segments) == 12
    with pytest.raises(LayoutTooSmall):
        plan_layout(Layout.R9, 9, 9)


@pytest.mark.parametrize("case", ["medium_r4_13", "high_r9_25", "high_r6_19", "small_r2_13", "trivial_r1"])
def test_layout_matches_reference_reset_grids(case):
    """The static walls of every reference reset grid are exactly the plan's
    walls; every door sits on one of the plan's door segments."""
    fx = load_golden(case)
    h, w = int(fx["meta"][0]), int(fx["meta"][1])
    plan = plan_layout(Layout(int(fx["meta"][5])), h, w)
    base = plan.base_cells()
    seg_cells = {c for s in plan.door_segments for c in s}
    for g in fx["grids0"]:
        walls = g == 72
        doors = (g >> 4) == 11
        assert np.array_equal(walls | doors, base == 72)
        assert set(np.nonzero(doors)[0]) <= seg_cells
        assert doors.sum() == len(plan.door_segments)


def test_benchmark_roundtrip_and_format(tmp_path):
    bm = load_benchmark(benchmark_file("medium"))
    assert len(bm) == 65536 and bm.max_rules == 18 and bm.max_objects == 18
    p = tmp_path / "x.xmgb"
    save_benchmark(p, bm)
    again = load_benchmark(p)
    assert np.array_equal(again.raw, bm.raw) and again.config_name == "medium" and again.seed == 42
    # header layout of ref docs/format.md
    raw = p.read_bytes()
    magic, version, flags, count, mr, mo, seed, nlen = struct.unpack_from("<4sHHIHHQH", raw)
    assert (magic, version, flags, count, mr, mo, seed) == (b"XMGB", 1, 1, 65536, 18, 18, 42)
    assert len(zlib.decompress(raw[26 + nlen:])) == 65536 * 94
    # corruption is rejected
    bad = tmp_path / "bad.xmgb"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(FormatError):
        load_benchmark(bad)
    bad.write_bytes(raw[:-10])
    with pytest.raises(FormatError):
        load_benchmark(bad)
    with pytest.raises(InvalidProportion):
        bm.split(1.5)
    a, b = bm.split(0.25)
    assert len(a) == 16384 and len(b) == 65536 - 16384


def test_sample_ruleset_is_reference_randint():
    bm = load_benchmark(benchmark_file("small"))
    for s in range(20):
        k = key_from_seed(s)
        assert bm.sample_ruleset(k) == bm.get_ruleset(randint(k, len(bm)))


def test_named_benchmarks(monkeypatch, tmp_path):
    bm = load_benchmark(benchmark_file("small"))
    save_benchmark(tmp_path / "small.xmgb", bm)
    monkeypatch.setenv("XMINIGRID_DATA", str(tmp_path))
    from paper_2312_12044_b200 import ruleset as rs
    rs.clear_cache()
    a = load_named("small")
    assert load_named("small") is a
    with pytest.raises(UnknownBenchmark):
        load_named("huge")


def test_task_table_left_packs_like_the_reference():
    """Rows keep the active rules / objects in stored order (ref
    ruleset.py:28-35, vecenv.py:143-151) with the MOVE / PICK_UP masks."""
    rs = Ruleset(goal=(4, 85, 102, 0), rules=((0, 0, 0, 0), (3, 85, 102, 150), (0, 0, 0, 0), (2, 86, 0, 57),
                                             (1, 151, 0, 57)), init_objects=(0, 85, 0, 102, 86))
    t = pack_rulesets([rs])
    row = t.rows[0]
    assert row[0] == 4 | 85 << 8 | 102 << 16
    assert row[1] & 0xFF == 3 and (row[1] >> 8) & 0xFF == 3
    assert row[2] == 0b010 and row[3] == 0b110  # MOVE: AGENT_NEAR slot 1; PICK: + AGENT_HOLD slot 2
    rules = row[HEADER_WORDS:HEADER_WORDS + 3].view(np.uint8).reshape(3, 4)
    # AGENT_NEAR carries its neighbour-slot mask (all four) in the unused in_b byte
    assert rules.tolist() == [[3, 85, 102, 150], [2, 86, 15, 57], [1, 151, 0, 57]]
    objs = row[HEADER_WORDS + t.rule_width:].view(np.uint8)[:3]
    assert objs.tolist() == [85, 102, 86]
    assert t.row_words % 4 == 0


def test_agent_rows_are_the_move_pickup_rules_in_stored_order():
    """TaskTable.agent_rows (the compact rows step_main fetches for MOVE /
    PICK_UP): the AGENT_HOLD / AGENT_NEAR-family rule words of each row in
    stored order, with the row's MOVE / PICK_UP masks re-indexed onto them."""
    rs = Ruleset(goal=(4, 85, 102, 0), rules=((0, 0, 0, 0), (3, 85, 102, 150), (0, 0, 0, 0), (2, 86, 0, 57),
                                             (1, 151, 0, 57)), init_objects=(0, 85, 0, 102, 86))
    t = pack_rulesets([rs])
    a = t.agent_rows[0]
    assert t.agent_row_words == 4
    assert a[0] & 0xFF == 2 and (a[0] >> 8) & 0xFFF == 0b01 and (a[0] >> 20) & 0xFFF == 0b11
    assert a[1:3].tolist() == t.rows[0, HEADER_WORDS + 1:HEADER_WORDS + 3].tolist()
    for cfg in ("medium", "high"):
        tt = load_benchmark(benchmark_file(cfg)).task_table()
        rows, ar = tt.rows, tt.agent_rows
        assert ar is not None and tt.agent_row_words % 4 == 0
        rng = np.random.default_rng(0)
        for i in rng.choice(tt.num_tasks, 500, replace=False):
            nr = int(rows[i, 1] & 0xFF)
            words = rows[i, HEADER_WORDS:HEADER_WORDS + nr]
            fam = [j for j in range(nr) if int(words[j] & 0xFF) in (1, 2, 8, 9, 10, 11)]
            n = int(ar[i, 0] & 0xFF)
            assert n == len(fam) and ar[i, 1:1 + n].tolist() == words[fam].tolist()
            move, pick = int(ar[i, 0] >> 8) & 0xFFF, int(ar[i, 0] >> 20)
            assert [(int(rows[i, 2]) >> j) & 1 for j in fam] == [(move >> k) & 1 for k in range(n)]
            assert [(int(rows[i, 3]) >> j) & 1 for j in fam] == [(pick >> k) & 1 for k in range(n)]
            assert move >> n == 0 and pick >> n == 0


def test_golden_fixtures_present():
    assert len([f for f in os.listdir(GOLDEN) if f.endswith(".npz")]) >= 20
