"""224x224 RGB observation images on the GPU.

Mirrors the image-observation part of ``rulegrid.render``
(/root/reference/pkg/src/rulegrid/render.py):

  IMAGE_SIDE                                    ref :21
  sprite(tile, color, px)                       ref :158-169 (cached atlas per px)
  image_observation(obs) / image_observations   ref :225-243
  decode_image_observation(image, view)         ref :246-272 (nearest sprite)

Sprites and images are produced by libxmg.so kernels (xmg_sprites,
xmg_image_obs) and are byte-identical to the reference's (pinned through the
oracle, tests/test_render_oracle.py, and on the GPU, tests/test_render_gpu.py).
The decoder is the reference's test oracle, evaluated with torch on the
images' device.  There is no CPU fallback.
"""

from __future__ import annotations

import threading

import torch

from . import _lib
from .vecenv import _device, _device_ctx, _stream

IMAGE_SIDE = 224

_atlas_lock = threading.Lock()
_ATLAS: dict[tuple[int, str], torch.Tensor] = {}


def sprite_atlas(px: int, device=None) -> torch.Tensor:
    """(15, 14, px, px, 3) uint8: every sprite at `px` pixels, built once per
    (px, device) on the device (ref render.py:93, the sprite cache)."""
    if px < 4:
        raise ValueError(f"tile_px must be >= 4, got {px}")
    dev = _device(device)
    key = (px, str(dev))
    with _atlas_lock:
        atlas = _ATLAS.get(key)
        if atlas is None:
            # 16 bytes either side: the image kernel reads aligned words around
            # unaligned offsets (up to 4 bytes before / 8 after a sprite row)
            flat = torch.zeros(210 * px * px * 3 + 32, dtype=torch.uint8, device=dev)
            atlas = flat[16: 16 + 210 * px * px * 3].view(15, 14, px, px, 3)
            with _device_ctx(dev):
                _lib.check(_lib.lib().xmg_sprites(px, atlas.data_ptr(), _stream(dev)), "xmg_sprites")
            _ATLAS[key] = atlas
    return atlas


_ALIGNED: dict[tuple[int, str], torch.Tensor] = {}


def aligned_atlas(view: int, device=None) -> torch.Tensor | None:
    """The phase-shifted atlas of the fast image path (xmg_image_atlas) for a
    view of at most 37 cells, built once per (view, device); None otherwise."""
    size = int(_lib.lib().xmg_image_atlas_bytes(view))
    if size < 0:
        return None
    dev = _device(device)
    key = (view, str(dev))
    with _atlas_lock:
        al = _ALIGNED.get(key)
    if al is None:
        base = sprite_atlas(IMAGE_SIDE // view, dev)
        al = torch.empty(size, dtype=torch.uint8, device=dev)
        with _device_ctx(dev):
            _lib.check(_lib.lib().xmg_image_atlas(view, base.data_ptr(), al.data_ptr(), _stream(dev)),
                       "xmg_image_atlas")
        with _atlas_lock:
            _ALIGNED[key] = al
    return al


def sprite(tile: int, color: int, px: int, device=None) -> torch.Tensor:
    """(px, px, 3) uint8 sprite of one entity code (ref render.py:158-169)."""
    if not (0 <= int(tile) <= 14 and 0 <= int(color) <= 13):
        raise ValueError(f"no entity ({tile}, {color})")
    return sprite_atlas(px, device)[int(tile), int(color)]


def image_observations(obs: torch.Tensor, out: torch.Tensor | None = None, check: bool = True) -> torch.Tensor:
    """(N, 224, 224, 3) uint8 images of (N, v, v, 2) observations on the GPU,
    each equal to ref render.py:225-243 image_observation(obs[i])."""
    if obs.is_cuda:
        with _device_ctx(obs.device):
            return _image_observations(obs, out, check)
    return _image_observations(obs, out, check)


def _image_observations(obs: torch.Tensor, out: torch.Tensor | None, check: bool) -> torch.Tensor:
    if obs.dim() != 4 or obs.shape[1] != obs.shape[2] or obs.shape[3] != 2:
        raise ValueError(f"expected square (N, v, v, 2) observations, got shape {tuple(obs.shape)}")
    if not obs.is_cuda:
        raise _lib.NativeLibraryError("image_observations needs CUDA tensors; there is no CPU fallback")
    n, v = obs.shape[0], obs.shape[1]
    px = IMAGE_SIDE // v
    if px < 4:
        raise ValueError(f"view size {v} leaves tiles under 4px")
    obs = obs.to(torch.uint8).contiguous()
    if check and bool(((obs[..., 0] > 14) | (obs[..., 1] > 13)).any()):
        raise ValueError("observation holds a code outside the tile / color enums")
    if out is None:
        out = torch.empty((n, IMAGE_SIDE, IMAGE_SIDE, 3), dtype=torch.uint8, device=obs.device)
    aligned = aligned_atlas(v, obs.device)
    if aligned is not None:  # views up to 37 cells: aligned 16-byte chunks
        _lib.check(_lib.lib().xmg_image_obs_aligned(obs.data_ptr(), n, v, aligned.data_ptr(), out.data_ptr(),
                                                    _stream(obs.device)), "xmg_image_obs_aligned")
        return out
    atlas = sprite_atlas(px, obs.device)
    _lib.check(_lib.lib().xmg_image_obs(obs.data_ptr(), n, v, atlas.data_ptr(), out.data_ptr(), _stream(obs.device)),
               "xmg_image_obs")
    return out


def image_observation(obs: torch.Tensor) -> torch.Tensor:
    """(224, 224, 3) image of one (v, v, 2) observation (ref render.py:225-243)."""
    if obs.dim() != 3 or obs.shape[0] != obs.shape[1] or obs.shape[2] != 2:
        raise ValueError(f"expected a square (N, N, 2) observation, got shape {tuple(obs.shape)}")
    return image_observations(obs.unsqueeze(0))[0]


def decode_image_observations(images: torch.Tensor, view: int) -> torch.Tensor:
    """Nearest-sprite decoding of (N, 224, 224, 3) images back to (N, v, v, 2)
    observations (ref render.py:246-272: L1 distance over every distinct
    sprite; sentinel tiles only with their own color id)."""
    px = IMAGE_SIDE // view
    off = (IMAGE_SIDE - view * px) // 2
    atlas = sprite_atlas(px, images.device).to(torch.int32)
    codes = [(t, c) for t in range(15) for c in range(14) if not (t in (0, 1, 2) and c != t)]
    tmpl = torch.stack([atlas[t, c] for t, c in codes]).reshape(len(codes), -1)  # (K, px*px*3)
    n = images.shape[0]
    cells = images[:, off:off + view * px, off:off + view * px].to(torch.int32)
    cells = cells.reshape(n, view, px, view, px, 3).permute(0, 1, 3, 2, 4, 5).reshape(n * view * view, -1)
    best = torch.empty(n * view * view, dtype=torch.int64, device=images.device)
    step = max(1, (1 << 28) // (4 * tmpl.numel()))  # cells per block: <= 256 MB of differences
    for s in range(0, cells.shape[0], step):
        blk = cells[s:s + step]
        best[s:s + step] = (blk[:, None, :] - tmpl[None]).abs().sum(-1).argmin(1)
    lut = torch.tensor(codes, dtype=torch.uint8, device=images.device)
    return lut[best].reshape(n, view, view, 2)


def decode_image_observation(image: torch.Tensor, view: int) -> torch.Tensor:
    return decode_image_observations(image.unsqueeze(0), view)[0]
