"""CPU: the image-observation oracle (oracle/xmg_render_oracle.c) against the
reference's own sprites and images (digests in tests/golden/render_golden.json,
made by tests/golden/make_render_golden.py from rulegrid.render)."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

from .conftest import GOLDEN
from .helpers import golden_cases, load_golden


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint8).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLDEN, "render_golden.json")) as fh:
        return json.load(fh)


def test_sprites_match_reference(gold):
    for px, table in gold["sprites"].items():
        for t, row in enumerate(table):
            for c, want in enumerate(row):
                assert _digest(O.sprite(t, c, int(px))) == want, f"sprite tile {t} color {c} px {px}"


def test_images_match_reference(gold):
    for case in golden_cases():
        fx = load_golden(case)
        for key, digests in gold["images"][case].items():
            obs = fx["obs0"] if key == "obs0" else fx["obs"][int(key[3:]) - 1]
            imgs = O.image_observations(obs)
            assert [_digest(i) for i in imgs] == digests, f"{case} {key}"


def test_synthetic_every_pair_and_unseen(gold):
    syn = np.array(gold["synthetic"]["obs"], np.uint8)
    assert [_digest(i) for i in O.image_observations(syn)] == gold["synthetic"]["digests"]
    img = O.image_observations(np.ones((1, 5, 5, 2), np.uint8))[0]
    assert _digest(img) == gold["synthetic"]["unseen5"]
    assert len(np.unique(img.reshape(-1, 3), axis=0)) == 1 and img[0, 0].max() < 32  # ref test_render.py:125-129


def test_small_pixels_rejected():
    with pytest.raises(ValueError):
        O.sprite(5, 3, 3)
