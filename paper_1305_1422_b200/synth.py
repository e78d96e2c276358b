"""Synthetic inputs, identical streams to the reference generators
(bench.py:85-103), so the same seeds give the same data."""
from __future__ import annotations

import numpy as np

from . import errors
from .datasets import DenseDataset, SparseDataset


def gen_random_dense(n: int, d: int, seed: int) -> DenseDataset:
    """Uniform [0,1) dense data, deterministic per seed (bench.py:85-88)."""
    rng = np.random.default_rng(seed)
    return DenseDataset(rng.random((n, d), dtype=np.float32))


def gen_random_sparse(n: int, d: int, density: float, seed: int) -> SparseDataset:
    """round(density*d) distinct sorted random columns per row (bench.py:91-103)."""
    if not (0.0 < density <= 1.0):
        raise errors.InvalidConfig("density must be in (0, 1]")
    rng = np.random.default_rng(seed)
    k = max(int(round(density * d)), 0)
    offsets = np.arange(n + 1, dtype=np.int64) * k
    cols = np.empty(n * k, dtype=np.int32)
    for i in range(n):
        cols[i * k:(i + 1) * k] = np.sort(
            rng.choice(d, size=k, replace=False)).astype(np.int32)
    values = rng.random(n * k, dtype=np.float32)
    return SparseDataset(d, offsets, cols, values)
