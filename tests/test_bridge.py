"""The JSON-lines bridge (paper_2312_12044_b200.bridge) against a transcript
of the reference's own bridge (tests/golden/bridge_golden.jsonl, made by
tests/golden/make_bridge_golden.py from rulegrid.bridge).

CPU: protocol framing, error names, registry and benchmark ops.  GPU: the
whole transcript replayed (scalar and batched steps on the device), replies
equal to the reference's; rewards / discounts compared as float32 (the
device computes float32 of the reference's float64, bit for bit)."""
import io
import json
import os

import numpy as np
import pytest

from .conftest import GOLDEN
from .helpers import benchmark_file


def _transcript():
    with open(os.path.join(GOLDEN, "bridge_golden.jsonl")) as fh:
        return [json.loads(line) for line in fh]


def _same(got, want, path="result"):
    if isinstance(want, dict):
        assert isinstance(got, dict) and set(got) == set(want), f"{path}: keys {sorted(got)} != {sorted(want)}"
        for k in want:
            _same(got[k], want[k], f"{path}.{k}")
    elif isinstance(want, list):
        assert isinstance(got, list) and len(got) == len(want), f"{path}: length"
        for i, (g, w) in enumerate(zip(got, want)):
            _same(g, w, f"{path}[{i}]")
    elif isinstance(want, float):
        assert np.float32(got) == np.float32(want), f"{path}: {got} != {want}"
    else:
        assert got == want, f"{path}: {got!r} != {want!r}"


def test_protocol_errors_and_registry_cpu():
    from paper_2312_12044_b200.bridge import Bridge, serve
    tr = _transcript()
    envs = next(r for r in tr if r["request"]["op"] == "environments")
    assert Bridge().dispatch("environments", {}) == envs["reply"]["result"]
    lines = [{"id": 1, "op": "make", "name": "NoSuchEnv"}, {"id": 2, "op": "step", "handle": "env:99", "action": 0},
             {"id": 3, "op": "frobnicate"}, {"id": 4, "op": "load_benchmark", "path": "/does/not/exist.bin"},
             {"id": 5, "op": "make", "name": "XLand-MiniGrid-R1-9x9",
              "ruleset": {"goal": [99, 0, 0, 0], "rules": [], "init_objects": []}},
             {"id": 6, "op": "make", "name": "XLand-MiniGrid-R1-9x9"}, {"id": 7, "op": "step", "handle": "env:1",
                                                                      "action": 0},
             {"id": 8, "op": "shutdown"}, {"id": 9, "op": "ping"}]
    stdin = io.StringIO("not json\n" + "\n".join(json.dumps(x) for x in lines) + "\n")
    stdout = io.StringIO()
    serve(stdin, stdout)
    rep = [json.loads(x) for x in stdout.getvalue().splitlines()]
    assert rep[0]["ok"] is False and rep[0]["id"] is None
    by = {r["id"]: r for r in rep[1:]}
    assert sorted(by) == [1, 2, 3, 4, 5, 6, 7, 8]  # nothing answered after shutdown
    assert [by[i]["error"] for i in (1, 2, 3, 4, 5, 7)] == ["UnknownEnvironment", "KeyError", "ValueError",
                                                             "FileNotFoundError", "InvalidEncoding", "RuntimeError"]
    assert by[6]["result"]["view_size"] == 5 and by[6]["result"]["step_budget"] == 243
    assert by[8] == {"id": 8, "ok": True, "result": {"bye": True}}


def test_benchmark_ops_cpu(tmp_path):
    from paper_2312_12044_b200.bridge import Bridge
    br = Bridge()
    meta = br.dispatch("load_benchmark", {"path": benchmark_file("small")})
    assert meta["num_rulesets"] == 4096
    a = br.dispatch("sample_ruleset", {"handle": meta["handle"], "seed": 5})
    assert a == br.dispatch("sample_ruleset", {"handle": meta["handle"], "seed": 5})
    assert br.dispatch("get_ruleset", {"handle": meta["handle"], "index": a["index"]})["ruleset"] == a["ruleset"]
    parts = br.dispatch("split", {"handle": meta["handle"], "prop": 0.8})
    assert (parts["left"]["num_rulesets"], parts["right"]["num_rulesets"]) == (3276, 820)
    sh = br.dispatch("shuffle", {"handle": meta["handle"], "seed": 1})
    assert sh["num_rulesets"] == 4096 and sh["handle"] != meta["handle"]
    out = str(tmp_path / "copy.xmgb")
    br.dispatch("save_benchmark", {"handle": sh["handle"], "path": out})
    again = br.dispatch("load_benchmark", {"path": out})
    assert br.dispatch("get_ruleset", {"handle": again["handle"], "index": 7}) == \
        br.dispatch("get_ruleset", {"handle": sh["handle"], "index": 7})


@pytest.mark.gpu
def test_transcript_replay_gpu():
    from paper_2312_12044_b200.bridge import Bridge
    br = Bridge()
    for i, rec in enumerate(_transcript()):
        req, want = rec["request"], rec["reply"]
        try:
            got = {"ok": True, "result": br.dispatch(req["op"], req)}
        except Exception as exc:
            got = {"ok": False, "error": type(exc).__name__}
        assert got["ok"] == want["ok"], f"request {i} {req}: {got}"
        if want["ok"]:
            _same(got["result"], want["result"], f"request {i} ({req['op']})")
        else:
            assert got["error"] == want["error"], f"request {i} {req}"
