"""Grid geometry: map types, lattices, neighbourhood kinds (host side).

Mirrors the reference grid.py (MapType 15-17, GridCoord 20-23, MOORE_OFFSETS
28-30, node_index 33-35, grid_distance 38-49, neighbors 52-73) and adds the
north-star extensions: a hexagonal offset-row lattice and the bubble
neighbourhood.  The device kernels implement the same definitions
(csrc/common.cuh grid_d2, csrc/hood.cu, csrc/umatrix.cu).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

import numpy as np


class MapType(Enum):
    PLANAR = "planar"
    TOROID = "toroid"


class GridType(Enum):
    """Extension. RECTANGULAR is the reference lattice."""
    RECTANGULAR = "rectangular"
    HEXAGONAL = "hexagonal"


class Neighborhood(Enum):
    """Extension. GAUSSIAN is the reference exp(-d/r) (train.py:138-144)."""
    GAUSSIAN = "gaussian"
    BUBBLE = "bubble"


@dataclass(frozen=True)
class GridCoord:
    col: int
    row: int


MOORE_OFFSETS = tuple(
    (dc, dr) for dr in (-1, 0, 1) for dc in (-1, 0, 1) if (dc, dr) != (0, 0)
)
# hexagonal offset-row adjacency (extension): odd rows sit half a column right
HEX_OFFSETS_EVEN = ((-1, -1), (0, -1), (-1, 0), (1, 0), (-1, 1), (0, 1))
HEX_OFFSETS_ODD = ((0, -1), (1, -1), (-1, 0), (1, 0), (0, 1), (1, 1))


def node_index(c: GridCoord, n_som_x: int) -> int:
    return c.row * n_som_x + c.col


def grid_distance(a: GridCoord, b: GridCoord, map_type: MapType, n_som_x: int,
                  n_som_y: int, grid: GridType = GridType.RECTANGULAR) -> float:
    """Euclidean lattice distance; toroids take the shorter way per axis.

    Hex: node (c, r) sits at (c + (r mod 2)/2, r sqrt(3)/2); the toroid is the
    rectangular period lattice (n_som_x, n_som_y sqrt(3)/2), n_som_y even.
    """
    if grid is GridType.HEXAGONAL:
        dx2 = abs((2 * a.col + (a.row & 1)) - (2 * b.col + (b.row & 1)))
        dr = abs(a.row - b.row)
        if map_type is MapType.TOROID:
            dx2 = min(dx2, 2 * n_som_x - dx2)
            dr = min(dr, n_som_y - dr)
        return math.sqrt(0.25 * dx2 * dx2 + 0.75 * dr * dr)
    dx = abs(a.col - b.col)
    dy = abs(a.row - b.row)
    if map_type is MapType.TOROID:
        dx = min(dx, n_som_x - dx)
        dy = min(dy, n_som_y - dy)
    return math.hypot(dx, dy)


def neighbors(c: GridCoord, map_type: MapType, n_som_x: int, n_som_y: int,
              grid: GridType = GridType.RECTANGULAR) -> list[GridCoord]:
    """U-matrix adjacency in scan order; planar drops out-of-range cells,
    toroids wrap and drop duplicates and the node itself (grid.py:52-73)."""
    if grid is GridType.HEXAGONAL:
        offs = HEX_OFFSETS_ODD if c.row & 1 else HEX_OFFSETS_EVEN
    else:
        offs = MOORE_OFFSETS
    out: list[GridCoord] = []
    seen: set[tuple[int, int]] = set()
    for dc, dr in offs:
        col, row = c.col + dc, c.row + dr
        if map_type is MapType.TOROID:
            col %= n_som_x
            row %= n_som_y
        elif not (0 <= col < n_som_x and 0 <= row < n_som_y):
            continue
        if (col, row) == (c.col, c.row) or (col, row) in seen:
            continue
        seen.add((col, row))
        out.append(GridCoord(col, row))
    return out


def distance_table(n_som_x: int, n_som_y: int, map_type: MapType) -> np.ndarray:
    """Rect lattice distance per wrapped offset [dy][dx], computed with numpy's
    hypot exactly as the reference builds its tables (kernels.py:107-112), so
    the device influence values see bit-identical distances."""
    dx = np.arange(n_som_x, dtype=np.float64)[None, :]
    dy = np.arange(n_som_y, dtype=np.float64)[:, None]
    return np.ascontiguousarray(np.hypot(np.broadcast_to(dx, (n_som_y, n_som_x)),
                                         np.broadcast_to(dy, (n_som_y, n_som_x))))
