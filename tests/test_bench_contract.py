"""bench.py's JSON line keeps the driver's contract (both arms).

The reference arm (CPU oracle port on the host threads) runs here without a
GPU; our arm runs on the B200 at a small workload (C2, 2^16 envs) with every
leg the default run has except the image and fused-rollout legs.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def _common(d, steps, warmup):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["unit"] == "env-steps/s" and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["steps"] == steps and d["warmup"] == warmup and d["n_gpus"] == 1
    assert d["value"] > 0 and d["ms_per_step"] > 0 and "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("port", "reference") and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] >= 0 and e["d2h_bytes_per_step"] >= 0


def test_reference_arm_line():
    d = _line("--impl", "reference", "--workload", "c1", "--steps", "3", "--warmup", "3")
    _common(d, 3, 3)
    assert d["impl"] == "reference"
    assert d["e2e"]["value"] == d["value"] == d["cpu_baseline"]["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_line():
    d = _line("--workload", "c2", "--steps", "16", "--warmup", "3", "--e2e-steps", "16", "--no-image", "--no-fused")
    _common(d, 16, 3)
    assert "impl" not in d or d["impl"] == "ours"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    if r["traffic"] is not None:
        assert abs(r["dram_frac"] - r["dram_achieved"] / r["peak"]) < 1e-9
    n = d["config"]["envs_per_gpu"]
    assert d["e2e"]["h2d_bytes_per_step"] == n and d["e2e"]["d2h_bytes_per_step"] == n * (2 * 5 * 5 + 9)
    assert d["gpu_launches"] >= 2 * d["steps"]
    assert d["clocks"]["sm_mhz"] > 0
