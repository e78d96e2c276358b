"""U-matrix (umatrix.py of the reference) computed on the GPU."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .grid import GridType, MapType


@dataclass
class UMatrix:
    n_columns: int
    n_rows: int
    heights: np.ndarray  # (n_rows, n_columns) float32

    def __post_init__(self):
        self.heights = np.ascontiguousarray(self.heights, dtype=np.float32)


def compute_umatrix(cb, map_type: MapType, grid: GridType = GridType.RECTANGULAR,
                    device=None) -> UMatrix:
    """Mean fp64 distance to the grid neighbours, stored f32 (umatrix.py:26-45)."""
    from .engine import _ptr, _stream, pick_device
    dev = pick_device(device)
    w = torch.from_numpy(np.ascontiguousarray(cb.weights, dtype=np.float32)).to(dev)
    cmap = _lib.SombMap(cb.n_columns, cb.n_rows,
                        _lib.GRID_HEX if GridType(grid) is GridType.HEXAGONAL else _lib.GRID_RECT,
                        _lib.TOROID if MapType(map_type) is MapType.TOROID else _lib.PLANAR)
    u = torch.empty(cb.n_columns * cb.n_rows, dtype=torch.float32, device=dev)
    _lib.call("somb_umatrix", _ptr(w), cb.n_dimensions, C.byref(cmap), _ptr(u), _stream(dev))
    return UMatrix(cb.n_columns, cb.n_rows, u.view(cb.n_rows, cb.n_columns).cpu().numpy())
