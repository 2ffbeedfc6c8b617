"""GPU: the device sprite atlas and 224x224 observation images (xmg_sprites,
xmg_image_obs through the C ABI) against the reference's digests
(tests/golden/render_golden.json) and the CPU oracle; the decode round trip
of ref tests/test_render.py:132-153."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O

from .conftest import GOLDEN
from .helpers import golden_cases, load_golden

pytestmark = pytest.mark.gpu


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint8).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLDEN, "render_golden.json")) as fh:
        return json.load(fh)


def test_sprite_atlas_matches_reference(gold):
    from paper_2312_12044_b200.render import sprite_atlas
    for px, table in gold["sprites"].items():
        atlas = sprite_atlas(int(px), "cuda").cpu().numpy()
        for t, row in enumerate(table):
            for c, want in enumerate(row):
                assert _digest(atlas[t, c]) == want, f"sprite tile {t} color {c} px {px}"


def test_images_match_reference_and_oracle(gold):
    from paper_2312_12044_b200.render import image_observations
    for case in golden_cases():
        fx = load_golden(case)
        for key, digests in gold["images"][case].items():
            obs = fx["obs0"] if key == "obs0" else fx["obs"][int(key[3:]) - 1]
            imgs = image_observations(torch.from_numpy(obs).cuda()).cpu().numpy()
            assert [_digest(i) for i in imgs] == digests, f"{case} {key}"
    syn = np.array(gold["synthetic"]["obs"], np.uint8)
    imgs = image_observations(torch.from_numpy(syn).cuda()).cpu().numpy()
    assert [_digest(i) for i in imgs] == gold["synthetic"]["digests"]
    one = image_observations(torch.ones((1, 5, 5, 2), dtype=torch.uint8, device="cuda"))[0].cpu().numpy()
    assert _digest(one) == gold["synthetic"]["unseen5"]


@pytest.mark.parametrize("env_name,config,v", [("XLand-MiniGrid-R4-13x13", "medium", 5),
                                               ("MiniGrid-DoorKey-8x8", None, 3),
                                               ("XLand-MiniGrid-R9-25x25", "high", 7),
                                               ("XLand-MiniGrid-R4-13x13", "medium", 9)])
def test_batch_images_of_steps_vs_oracle(env_name, config, v):
    """Images of a whole batch of step observations (thousands of envs, mixed
    facings, objects, doors) equal the oracle's byte for byte."""
    from dataclasses import replace
    from paper_2312_12044_b200 import VecEnv, key_from_seed, load_benchmark, make, policy_keys, random_actions
    from paper_2312_12044_b200.render import image_observations
    from .helpers import benchmark_file
    _, params = make(env_name)
    params = replace(params, view_size=v)
    n = 2048
    vec = VecEnv(params, n, load_benchmark(benchmark_file(config)) if config else None)
    vec.reset(key_from_seed(11))
    acts = random_actions(policy_keys(key_from_seed(12), n, device=vec.device), 0, 60)
    for t in range(60):
        ts = vec.step(acts[t])
    imgs = image_observations(ts.observations)
    want = O.image_observations(ts.observations.cpu().numpy())
    assert torch.equal(imgs.cpu(), torch.from_numpy(want))


def test_decode_round_trip_and_errors():
    from dataclasses import replace
    from paper_2312_12044_b200 import VecEnv, key_from_seed, make
    from paper_2312_12044_b200.render import (decode_image_observations, image_observation, image_observations,
                                              sprite)
    for see in (True, False):
        _, params = make("XLand-MiniGrid-R4-13x13")
        params = replace(params, see_through_walls=see)
        vec = VecEnv(params, 64)
        ts = vec.reset(key_from_seed(4))
        for t in range(40):
            ts = vec.step(torch.full((64,), t * 7 % 6, dtype=torch.uint8, device="cuda"))
            if t % 13 == 0:
                dec = decode_image_observations(image_observations(ts.observations), params.view_size)
                assert torch.equal(dec, ts.observations)
    assert image_observation(ts.observations[0]).shape == (224, 224, 3)
    red_ball = sprite(5, 3, 8).cpu().numpy().astype(int).reshape(-1, 3).mean(0)  # ref test_render.py:88-91
    assert red_ball[0] > red_ball[1] and red_ball[0] > red_ball[2]
    with pytest.raises(ValueError):
        sprite(5, 3, 3)
    with pytest.raises(ValueError):
        image_observations(torch.zeros((1, 57, 57, 2), dtype=torch.uint8, device="cuda"))
    bad = torch.zeros((1, 5, 5, 2), dtype=torch.uint8, device="cuda")
    bad[0, 2, 2, 1] = 14
    with pytest.raises(ValueError):
        image_observations(bad)


def test_aligned_and_generic_image_paths_agree():
    """The aligned 16-byte path (views <= 37) and the word-gather path give the
    same bytes for every odd view both cover, and agree with the oracle."""
    from paper_2312_12044_b200 import _lib
    from paper_2312_12044_b200.render import aligned_atlas, sprite_atlas
    L = _lib.lib()
    g = torch.Generator(device="cuda").manual_seed(1)
    for v in (3, 5, 7, 9, 11, 13, 17, 21, 25, 31, 37):
        n = 64
        obs = torch.stack([torch.randint(0, 15, (n, v, v), device="cuda", generator=g),
                           torch.randint(0, 14, (n, v, v), device="cuda", generator=g)], -1).to(torch.uint8)
        a = torch.empty((n, 224, 224, 3), dtype=torch.uint8, device="cuda")
        b = torch.empty_like(a)
        al = aligned_atlas(v, "cuda")
        assert al is not None
        assert L.xmg_image_obs_aligned(obs.data_ptr(), n, v, al.data_ptr(), a.data_ptr(), None) == 0
        base = sprite_atlas(224 // v, "cuda")
        assert L.xmg_image_obs(obs.data_ptr(), n, v, base.data_ptr(), b.data_ptr(), None) == 0
        torch.cuda.synchronize()
        assert torch.equal(a, b), v
        if v in (3, 5, 13, 37):
            want = O.image_observations(obs[:8].cpu().numpy())
            assert np.array_equal(a[:8].cpu().numpy(), want), v
    assert aligned_atlas(39, "cuda") is None  # 5-px tiles: the word-gather path
