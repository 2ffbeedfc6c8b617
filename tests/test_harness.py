"""The throughput / scaling harness (paper_2312_12044_b200.harness), the GPU
counterpart of ref harness.py:149-282; shapes follow ref tests/test_harness.py."""
import csv

import pytest


def test_scaling_ruleset_and_axis_check_cpu(tmp_path):
    from paper_2312_12044_b200.harness import bench_scaling, scaling_ruleset, write_csv
    rs = scaling_ruleset(3)  # ref harness.py:224-246: NEAR(red ball, green square -> blue pyramid) x3
    assert rs.goal == (1, 13 * 16 + 6, 0, 0)
    assert rs.rules == ((3, 5 * 16 + 3, 6 * 16 + 4, 7 * 16 + 5),) * 3
    assert rs.init_objects == (5 * 16 + 3, 5 * 16 + 7, 5 * 16 + 6, 5 * 16 + 11)
    rs.validate()
    with pytest.raises(ValueError):
        bench_scaling("colour_depth", [1])
    write_csv(tmp_path / "x.csv", ("n", "sps"), [(1, 2.0), (3, 4.5)])
    assert list(csv.reader(open(tmp_path / "x.csv"))) == [["n", "sps"], ["1", "2.0"], ["3", "4.5"]]


@pytest.mark.gpu
def test_bench_throughput_and_scaling_shapes():
    from paper_2312_12044_b200.harness import bench_scaling, bench_throughput
    rows = bench_throughput("XLand-MiniGrid-R1-9x9", [256, 4096], num_steps=128, repeats=2)
    assert [n for n, _ in rows] == [256, 4096] and all(sps > 0 for _, sps in rows)
    assert rows[1][1] > rows[0][1]  # grows with the batch below saturation (ref test_harness.py:86-91)
    for mode in ("steps", "rollout"):
        (n, sps), = bench_throughput("MiniGrid-DoorKey-8x8", [2048], num_steps=64, repeats=1, mode=mode)
        assert n == 2048 and sps > 0
    g = bench_scaling("grid_size", [9, 13], num_envs=512, num_steps=64, repeats=1)
    r = bench_scaling("num_rules", [1, 24], num_envs=512, num_steps=64, repeats=1)
    assert [v for v, _ in g] == [9, 13] and [v for v, _ in r] == [1, 24]
    assert all(s > 0 for _, s in g + r)
