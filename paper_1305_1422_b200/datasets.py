"""Dataset types, identical in layout to the reference (fileio.py:32-95)."""
from __future__ import annotations

from dataclasses import dataclass
from typing import Union

import numpy as np


@dataclass
class DenseDataset:
    """Row-major single-precision matrix of instances."""

    values: np.ndarray  # (n_vectors, n_dimensions) float32

    def __post_init__(self):
        if not _is_torch(self.values):
            self.values = np.ascontiguousarray(self.values, dtype=np.float32)
        if self.values.ndim != 2:
            raise ValueError("dense values must be 2-D")

    @property
    def n_vectors(self) -> int:
        return int(self.values.shape[0])

    @property
    def n_dimensions(self) -> int:
        return int(self.values.shape[1])

    def element_count(self) -> int:
        return int(self.values.shape[0] * self.values.shape[1])


@dataclass
class SparseDataset:
    """CSR rows: int64 offsets, int32 strictly increasing cols, f32 values."""

    n_dimensions: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.row_offsets = np.ascontiguousarray(self.row_offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(self.col_indices, dtype=np.int32)
        self.values = np.ascontiguousarray(self.values, dtype=np.float32)

    @property
    def n_vectors(self) -> int:
        return len(self.row_offsets) - 1

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    def row(self, i: int):
        s, e = self.row_offsets[i], self.row_offsets[i + 1]
        return self.col_indices[s:e], self.values[s:e]

    def densify(self) -> DenseDataset:
        out = np.zeros((self.n_vectors, self.n_dimensions), dtype=np.float32)
        rows = np.repeat(np.arange(self.n_vectors), np.diff(self.row_offsets))
        out[rows, self.col_indices] = self.values
        return DenseDataset(out)

    def element_count(self) -> int:
        return int(self.row_offsets.size + self.col_indices.size + self.values.size)


Dataset = Union[DenseDataset, SparseDataset]


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")
