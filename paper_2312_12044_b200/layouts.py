"""Room layouts: static geometry resolved on the host, uploaded once.

Behaviour follows the reference (ref layouts.py:18-127): a bordered grid
split into 1/2/4/6/9 rooms by wall lines at ``i*(size-1)//rooms``, one door
segment per shared wall, enumerated vertical walls first (room row, then
wall column) and then horizontal walls (wall row, then room column); that
order fixes the Philox draw sequence of the doors.  Only the geometry lives
here; doors, objects and spawns are drawn on the GPU at every reset.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from .core import FLOOR_CODE, WALL_CODE, LayoutTooSmall


class Layout(IntEnum):
    R1 = 1
    R2 = 2
    R4 = 4
    R6 = 6
    R9 = 9


ROOM_GRID = {Layout.R1: (1, 1), Layout.R2: (1, 2), Layout.R4: (2, 2), Layout.R6: (2, 3), Layout.R9: (3, 3)}


@dataclass(frozen=True)
class LayoutPlan:
    height: int
    width: int
    wall_rows: tuple[int, ...]
    wall_cols: tuple[int, ...]
    door_segments: tuple[tuple[int, ...], ...]
    fixed_doors: bool

    def base_cells(self) -> np.ndarray:
        """(H*W,) uint8: border and dividing walls, floor elsewhere."""
        g = np.full((self.height, self.width), FLOOR_CODE, np.uint8)
        g[[0, -1], :] = WALL_CODE
        g[:, [0, -1]] = WALL_CODE
        for r in self.wall_rows:
            g[r, :] = WALL_CODE
        for c in self.wall_cols:
            g[:, c] = WALL_CODE
        return g.reshape(-1)

    def segment_arrays(self) -> tuple[np.ndarray, np.ndarray]:
        """CSR form (offsets int16 [S+1], cells int16) for the device."""
        off = np.zeros(len(self.door_segments) + 1, np.int16)
        off[1:] = np.cumsum([len(s) for s in self.door_segments])
        cells = np.array([c for s in self.door_segments for c in s] or [0], np.int16)
        return off, cells


def _lines(size: int, rooms: int) -> tuple[int, ...]:
    return tuple(k * (size - 1) // rooms for k in range(1, rooms))


def plan_layout(layout: Layout, height: int, width: int) -> LayoutPlan:
    rows, cols = ROOM_GRID[Layout(layout)]
    if height < 4 * rows + 1 or width < 4 * cols + 1:
        raise LayoutTooSmall(f"{height}x{width} cannot hold {rows}x{cols} rooms")
    wr, wc = _lines(height, rows), _lines(width, cols)
    redge, cedge = (0, *wr, height - 1), (0, *wc, width - 1)
    vertical = [tuple(r * width + x for r in range(redge[i] + 1, redge[i + 1])) for i in range(rows) for x in wc]
    horizontal = [tuple(y * width + c for c in range(cedge[j] + 1, cedge[j + 1])) for y in wr for j in range(cols)]
    return LayoutPlan(height, width, wr, wc, tuple(vertical + horizontal), Layout(layout) == Layout.R6)


def bordered(height: int, width: int, goal: bool) -> np.ndarray:
    """Single-room grid of the classic ports, optionally with the green goal
    square at (H-2, W-2) (ref scenarios.py:69-89)."""
    g = np.full((height, width), FLOOR_CODE, np.uint8)
    g[[0, -1], :] = WALL_CODE
    g[:, [0, -1]] = WALL_CODE
    if goal:
        g[height - 2, width - 2] = 8 * 16 + 4  # GOAL, GREEN
    return g.reshape(-1)
