"""Entity codes, grid/agent value types, errors and keys (host side).

Mirrors the public vocabulary of the reference's primitives so code written
against ``rulegrid`` reads the same here:
  * tile / color ids and codes          ref core.py:17-70
  * Direction, Position, AgentState, Grid ref core.py:106-175
  * exception types                      ref errors.py:4-45
  * Key + key derivation                 ref rng.py:35-145
Key derivation calls the scalar host helpers of libxmg.so (xmg_key_from_seed,
xmg_fold_in); batched derivation runs on the GPU (vecenv.split_batch).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum
from typing import NamedTuple

import numpy as np

from . import _lib


# ------------------------------------------------------------------ errors
class InvalidCode(ValueError):
    """Entity code or its tile/color parts fall outside the legal ranges."""


class InvalidEncoding(ValueError):
    """Rule or goal encoding does not describe any known variant."""


class InvalidAction(ValueError):
    """Action id outside the discrete action space."""


class GridFull(RuntimeError):
    """Not enough free floor cells left to place the requested entities."""


class LayoutTooSmall(ValueError):
    """Grid dimensions cannot accommodate the requested room layout."""


class UnknownEnvironment(KeyError):
    """Environment name not present in the registry."""


class UnknownBenchmark(KeyError):
    """Benchmark name not present in the named-benchmark registry."""


class FormatError(ValueError):
    """Benchmark file is corrupt or has an unsupported version."""


class InvalidProportion(ValueError):
    """Split proportion outside the open interval (0, 1)."""


# ------------------------------------------------------------------ codes
# tile and color ids in code order (ref core.py:17-49); code = tile * 16 + color
Tile = IntEnum("Tile", [(name, i) for i, name in enumerate(
    "END_OF_MAP UNSEEN EMPTY FLOOR WALL BALL SQUARE PYRAMID GOAL KEY DOOR_LOCKED DOOR_CLOSED DOOR_OPEN HEX STAR"
    .split())])
Color = IntEnum("Color", [(name, i) for i, name in enumerate(
    "END_OF_MAP UNSEEN EMPTY RED GREEN BLUE PURPLE YELLOW GREY BLACK ORANGE WHITE BROWN PINK".split())])
Tile.__module__ = Color.__module__ = __name__


PICKABLE_TILES = frozenset({Tile.BALL, Tile.SQUARE, Tile.PYRAMID, Tile.KEY, Tile.HEX, Tile.STAR})
WALKABLE_TILES = frozenset({Tile.FLOOR, Tile.GOAL, Tile.DOOR_OPEN})
MAX_TILE = max(Tile)
MAX_COLOR = max(Color)
FLOOR_CODE = int(Tile.FLOOR) * 16 + int(Color.BLACK)  # 57
WALL_CODE = int(Tile.WALL) * 16 + int(Color.GREY)  # 72
EMPTY_POCKET = 0
GENERATION_COLORS = (Color.RED, Color.GREEN, Color.BLUE, Color.PURPLE, Color.YELLOW,
                     Color.GREY, Color.ORANGE, Color.WHITE, Color.BROWN, Color.PINK)


def _check_part(value: int, top: int, what: str) -> None:
    if not 0 <= value <= top:
        raise InvalidCode(f"{what} {value} outside [0, {top}]")


def pack_entity(tile: int, color: int) -> int:
    """tile * 16 + color, both parts range-checked (ref core.py:73-79)."""
    _check_part(tile, MAX_TILE, "tile id")
    _check_part(color, MAX_COLOR, "color id")
    return tile * 16 + color


@dataclass(frozen=True, slots=True)
class Entity:
    tile: Tile
    color: Color

    @property
    def code(self) -> int:
        return self.tile * 16 + self.color


def unpack_entity(code: int) -> Entity:
    """Inverse of pack_entity; rejects codes no (tile, color) maps to (ref core.py:82-89)."""
    tile, color = divmod(code, 16)
    _check_part(tile, MAX_TILE, f"code {code}: tile part")
    _check_part(color, MAX_COLOR, f"code {code}: color part")
    return Entity(Tile(tile), Color(color))


class Direction(IntEnum):
    UP = 0
    RIGHT = 1
    DOWN = 2
    LEFT = 3


@dataclass(frozen=True, slots=True)
class Position:
    row: int
    col: int


@dataclass(frozen=True, slots=True)
class AgentState:
    position: Position
    direction: Direction
    pocket: int = EMPTY_POCKET


@dataclass(frozen=True, slots=True)
class Grid:
    height: int
    width: int
    cells: bytes

    def code_at(self, row: int, col: int) -> int:
        return self.cells[row * self.width + col]

    def tile_at(self, row: int, col: int) -> int:
        return self.cells[row * self.width + col] >> 4


# ------------------------------------------------------------------- keys
class Key(NamedTuple):
    """128-bit generator key (ref rng.py:35-39)."""

    hi: int
    lo: int


DOMAIN_DRAW, DOMAIN_SPLIT, DOMAIN_FOLD, DOMAIN_SEED = 1, 2, 3, 4
_MASK64 = (1 << 64) - 1


def key_from_seed(seed: int) -> Key:
    out = (C.c_uint64 * 2)()
    _lib.lib().xmg_key_from_seed(seed & _MASK64, (seed >> 64) & _MASK64, out)
    return Key(int(out[0]), int(out[1]))


def fold_in(key: Key, data: int, _domain: int = DOMAIN_FOLD) -> Key:
    out = (C.c_uint64 * 2)()
    _lib.lib().xmg_fold_in(key[0], key[1], data & _MASK64, (data >> 64) & _MASK64, _domain, out)
    return Key(int(out[0]), int(out[1]))


def split(key: Key, num: int = 2) -> tuple[Key, ...]:
    return tuple(fold_in(key, i, DOMAIN_SPLIT) for i in range(num))


def philox_block(ctr, key: Key) -> tuple[int, int, int, int]:
    c = (C.c_uint64 * 4)(*(int(x) & _MASK64 for x in ctr))
    out = (C.c_uint64 * 4)()
    _lib.lib().xmg_philox_host(c, key[0], key[1], out)
    return tuple(int(x) for x in out)


def random_words(key: Key, count: int) -> list[int]:
    out: list[int] = []
    for block in range((count + 3) // 4):
        out.extend(philox_block((block, 0, DOMAIN_DRAW, 0), key))
    return out[:count]


def randint(key: Key, bound: int, index: int = 0) -> int:
    block, offset = divmod(index, 4)
    return philox_block((block, 0, DOMAIN_DRAW, 0), key)[offset] % bound


def keys_to_u64(keys) -> np.ndarray:
    """Sequence of Keys -> (n, 2) uint64 array of (hi, lo)."""
    return np.array([[k[0], k[1]] for k in keys], dtype=np.uint64).reshape(-1, 2)
