"""Record a JSON-lines transcript of the REFERENCE bridge (rulegrid.bridge).

Run in the build container (the reference is not present on the GPU box):

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python /root/repo/tests/golden/make_bridge_golden.py

Writes tests/golden/bridge_golden.jsonl: one {"request", "reply"} per line,
covering scalar make/reset/step (300 steps of ref tests/test_bridge.py's
random actions, with auto-reset), overrides (max_steps, view_size,
see_through_walls, ruleset), batched make_batch/batch_reset/batch_step, a
DoorKey port and the error replies.  tests/test_bridge*.py replay the
requests through paper_2312_12044_b200.bridge and compare the replies.
"""
from __future__ import annotations

import json
import os

import numpy as np

from rulegrid.bridge import Bridge
from rulegrid.rng import key_from_seed, randint

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "bridge_golden.jsonl")


def main():
    br = Bridge()
    reqs = []

    def call(req):
        try:
            rep = {"ok": True, "result": br.dispatch(req["op"], req)}
        except Exception as exc:  # the error name is part of the protocol
            rep = {"ok": False, "error": type(exc).__name__}
        reqs.append({"request": req, "reply": rep})
        return rep

    h = call({"op": "make", "name": "XLand-MiniGrid-R1-9x9"})["result"]["handle"]
    call({"op": "reset", "handle": h, "seed": 11})
    key = key_from_seed(11)
    for t in range(300):
        call({"op": "step", "handle": h, "action": randint(key, 6, t)})
    h2 = call({"op": "make", "name": "XLand-MiniGrid-R1-9x9", "max_steps": 17, "view_size": 7})["result"]["handle"]
    call({"op": "reset", "handle": h2, "seed": 0})
    for t in range(40):
        call({"op": "step", "handle": h2, "action": (3 * t + 1) % 6})
    task = {"goal": [1, 53, 0, 0], "rules": [[1, 53, 0, 101], [2, 101, 0, 53]], "init_objects": [53, 101]}
    h3 = call({"op": "make", "name": "XLand-MiniGrid-R4-13x13", "ruleset": task,
               "see_through_walls": False})["result"]["handle"]
    call({"op": "reset", "handle": h3, "seed": 5})
    for t in range(120):
        call({"op": "step", "handle": h3, "action": randint(key_from_seed(5), 6, t)})
    h4 = call({"op": "make", "name": "MiniGrid-DoorKey-8x8"})["result"]["handle"]
    call({"op": "reset", "handle": h4, "seed": 2})
    for t in range(200):
        call({"op": "step", "handle": h4, "action": randint(key_from_seed(2), 6, t)})
    b = call({"op": "make_batch", "name": "XLand-MiniGrid-R4-13x13", "num_envs": 4})["result"]["handle"]
    call({"op": "batch_reset", "handle": b, "seed": 3})
    rng = np.random.default_rng(0)
    for _ in range(60):
        call({"op": "batch_step", "handle": b, "actions": rng.integers(0, 6, 4).tolist()})
    call({"op": "batch_step", "handle": b, "actions": [0, 1, 2]})
    call({"op": "batch_step", "handle": b, "actions": [0, 1, 2, 9]})
    call({"op": "make", "name": "NoSuchEnv"})
    call({"op": "step", "handle": "env:99", "action": 0})
    call({"op": "frobnicate"})
    h5 = call({"op": "make", "name": "XLand-MiniGrid-R1-9x9"})["result"]["handle"]
    call({"op": "step", "handle": h5, "action": 0})
    call({"op": "make", "name": "XLand-MiniGrid-R1-9x9", "ruleset": {"goal": [99, 0, 0, 0], "rules": [],
                                                                      "init_objects": []}})
    call({"op": "environments"})
    call({"op": "ping"})
    with open(OUT, "w") as fh:
        for r in reqs:
            fh.write(json.dumps(r) + "\n")
    print("wrote", OUT, len(reqs), "requests")


if __name__ == "__main__":
    main()
