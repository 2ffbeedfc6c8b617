"""Generate golden digests of the REFERENCE's sprites and observation images.

Run in the build container (the reference is not present on the GPU box):

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python /root/repo/tests/golden/make_render_golden.py

Writes tests/golden/render_golden.json:
  * "sprites": sha256 of rulegrid.render.sprite(tile, color, px) for every
    tile x color at the pixel sizes image observations use (224 // v for
    v = 3, 5, 7, 9, 11) and a few small ones;
  * "images": per golden fixture, sha256 of image_observation(obs) for each
    env of its first observation batch and of its steps 0, 5, 17 (the
    observations themselves are in the fixture);
  * "observations": the obs the digests were taken from, as nested lists
    (small: 8 envs of one fixture) for a direct byte comparison.
"""
from __future__ import annotations

import glob
import hashlib
import json
import os

import numpy as np

from rulegrid.core import Color, Tile
from rulegrid.render import image_observation, sprite

OUT = os.path.dirname(os.path.abspath(__file__))
PX = (4, 5, 8, 12, 20, 24, 32, 44, 74)


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint8).tobytes()).hexdigest()


def main():
    out = {"sprites": {}, "images": {}}
    for px in PX:
        out["sprites"][str(px)] = [[digest(sprite(t, c, px)) for c in Color] for t in Tile]
    for path in sorted(glob.glob(os.path.join(OUT, "*.npz"))):
        case = os.path.basename(path)[:-4]
        if case == "policy_stream":
            continue
        fx = np.load(path)
        batches = {"obs0": fx["obs0"]}
        for t in (0, 5, 17):
            if t < len(fx["obs"]):
                batches[f"obs{t + 1}"] = fx["obs"][t]
        out["images"][case] = {k: [digest(image_observation(o)) for o in b] for k, b in batches.items()}
    # an all-UNSEEN observation and a synthetic one with every (tile, color) pair
    allp = np.array([(t, c) for t in Tile for c in Color], np.uint8)
    pad = np.zeros((7 * 7 * 5 - len(allp), 2), np.uint8)
    synth = np.concatenate([allp, pad]).reshape(5, 7, 7, 2)
    out["synthetic"] = {"obs": synth.tolist(), "digests": [digest(image_observation(o)) for o in synth],
                        "unseen5": digest(image_observation(np.ones((5, 5, 2), np.uint8)))}
    with open(os.path.join(OUT, "render_golden.json"), "w") as fh:
        json.dump(out, fh)
    print("wrote", os.path.join(OUT, "render_golden.json"))


if __name__ == "__main__":
    main()
