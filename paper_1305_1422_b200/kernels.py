"""Reference-compatible kernel API (kernels.py of the reference), on the GPU.

`Kernel` keeps the reference values {0 DENSE_NAIVE, 1 DENSE_BLOCKED,
2 SPARSE} (kernels.py:51-54).  Both dense kernels run the same tcgen05
screen; they differ only in the fp64 formula of the exact re-rank (naive
sum of squared differences vs the norms identity), mirroring
kernels.py:182-205.  `search_accumulate` / `blend` / `epoch_kernel` /
`accumulate` return host numpy results with the reference shapes and dtypes
so callers (and the parity tests) can compare at the accumulator level.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum
from typing import Optional

import numpy as np
import torch

from . import _lib, errors
from .datasets import Dataset, DenseDataset, SparseDataset
from .grid import GridType, MapType, Neighborhood


class Kernel(IntEnum):
    DENSE_NAIVE = 0
    DENSE_BLOCKED = 1
    SPARSE = 2


DEFAULT_BLOCK_SIZE = 256
DEFAULT_CUTOFF = 1e-3


@dataclass
class Accumulators:
    """numerators N_j (K, D) and denominators D_j (K,), fp64 (kernels.py:69-84)."""

    numerators: np.ndarray
    denominators: np.ndarray

    @classmethod
    def zeros(cls, n_nodes: int, n_dimensions: int) -> "Accumulators":
        return cls(np.zeros((n_nodes, n_dimensions)), np.zeros(n_nodes))

    def merge(self, other: "Accumulators") -> None:
        self.numerators += other.numerators
        self.denominators += other.denominators


def _to_coords(bmu_idx: np.ndarray, n_som_x: int) -> np.ndarray:
    """Flat node indices -> (n, 2) int32 [row, col] (kernels.py:257-262)."""
    out = np.empty((len(bmu_idx), 2), dtype=np.int32)
    out[:, 0] = bmu_idx // n_som_x
    out[:, 1] = bmu_idx % n_som_x
    return out


def _check_dims(data: Dataset, cb) -> None:
    if data.n_dimensions != cb.n_dimensions:
        raise errors.DimensionMismatch(
            f"data has {data.n_dimensions} dimensions, codebook {cb.n_dimensions}")


def _check_pair(kernel, data) -> Kernel:
    kernel = Kernel(kernel)
    sparse = isinstance(data, SparseDataset)
    if (kernel is Kernel.SPARSE) != sparse:
        raise errors.KernelDataMismatch(
            f"kernel {kernel.name} cannot run on {'sparse' if sparse else 'dense'} data")
    return kernel


def make_engine(data: Dataset, n_columns, n_rows, map_type, grid=GridType.RECTANGULAR,
                device=None, group=None, options=None):
    if isinstance(data, SparseDataset):
        from .sparse import SparseEngine
        return SparseEngine(data, n_columns, n_rows, MapType(map_type), GridType(grid),
                            device=device, group=group, options=options)
    from .engine import SomEngine
    return SomEngine(data, n_columns, n_rows, MapType(map_type), GridType(grid), device=device,
                     group=group, options=options)


def make_engine_sharded(data: Dataset, cfg, device=None, group=None, options=None):
    """Engine over this rank's contiguous row slice (distributed.py:424-434)."""
    from .engine import dist_info
    from .parallel import partition, slice_rows
    rank, world = dist_info(group)
    first, count = partition(data.n_vectors, world)[rank]
    part = slice_rows(data, first, count) if world > 1 else data
    return make_engine(part, cfg.n_columns, cfg.n_rows, cfg.map_type, cfg.grid, device=device,
                       group=group, options=options)


def search_accumulate(data: Dataset, cb, radius: float, cutoff: float, map_type: MapType,
                      kernel: Kernel, workers: int = 1, with_accumulators: bool = True, *,
                      grid: GridType = GridType.RECTANGULAR,
                      neighborhood: Neighborhood = Neighborhood.GAUSSIAN, compact: bool = False,
                      options=None):
    """kernels.py:365-435 on the GPU: (bmu_flat int64[N], qe_sum, Accumulators | None)."""
    _check_dims(data, cb)
    kernel = _check_pair(kernel, data)
    eng = make_engine(data, cb.n_columns, cb.n_rows, map_type, grid, options=options)
    eng.set_codebook(cb.weights)
    mode = _lib.DIST_NAIVE if kernel is Kernel.DENSE_NAIVE else _lib.DIST_BLOCKED
    eng.search(mode)
    eng.qe_sum()
    acc = None
    if with_accumulators:
        eng.node_sums()
        num = torch.empty((eng.K, eng.d), dtype=torch.float64, device=eng.dev)
        den = torch.empty(eng.K, dtype=torch.float64, device=eng.dev)
        eng.update(radius, 0.0, cutoff, neighborhood, compact, num_out=num, den_out=den,
                   all_nodes=True)
        acc = Accumulators(num.cpu().numpy(), den.cpu().numpy())
    bmu = eng.bmu[: eng.n].to(torch.int64).cpu().numpy()
    qe = float(eng.qe.item())
    return bmu, qe, acc


def accumulate(data: Dataset, bmus: np.ndarray, radius: float, cutoff: float, map_type: MapType,
               n_som_x: int, n_som_y: int, workers: int = 1, *, grid=GridType.RECTANGULAR,
               neighborhood=Neighborhood.GAUSSIAN, compact=False, options=None) -> Accumulators:
    """Batch-update sums for given BMUs (kernels.py:326-360)."""
    if len(bmus) != data.n_vectors:
        raise errors.DimensionMismatch(f"BMU table has {len(bmus)} rows, data {data.n_vectors}")
    eng = make_engine(data, n_som_x, n_som_y, map_type, grid, options=options)
    flat = (np.asarray(bmus)[:, 0].astype(np.int64) * n_som_x + np.asarray(bmus)[:, 1])
    eng.bmu[: eng.n].copy_(torch.from_numpy(flat.astype(np.int32)).to(eng.dev))
    eng.node_sums()
    num = torch.empty((eng.K, eng.d), dtype=torch.float64, device=eng.dev)
    den = torch.empty(eng.K, dtype=torch.float64, device=eng.dev)
    eng.update(radius, 0.0, cutoff, neighborhood, compact, num_out=num, den_out=den, all_nodes=True)
    return Accumulators(num.cpu().numpy(), den.cpu().numpy())


def blend(weights: np.ndarray, acc: Accumulators, scale: float, device=None) -> np.ndarray:
    """w <- (1-scale) w + scale N/D where D > 0, fp64 then one f32 rounding
    (kernels.py:438-450); rows with D = 0 stay bit-identical."""
    from .engine import _ptr, _stream, pick_device
    dev = pick_device(device)
    w = torch.from_numpy(np.ascontiguousarray(weights, dtype=np.float32)).to(dev)
    num = torch.from_numpy(np.ascontiguousarray(acc.numerators, dtype=np.float64)).to(dev)
    den = torch.from_numpy(np.ascontiguousarray(acc.denominators, dtype=np.float64)).to(dev)
    out = torch.empty_like(w)
    k, d = w.shape
    _lib.call("somb_blend", _ptr(w), _ptr(num), _ptr(den), k, d, float(scale), _ptr(out),
              _stream(dev))
    return out.cpu().numpy()


def epoch_kernel(data: Dataset, cb, radius: float, scale: float, cutoff: float, map_type: MapType,
                 kernel: Kernel, workers: int = 1, *, grid=GridType.RECTANGULAR,
                 neighborhood=Neighborhood.GAUSSIAN, compact=False, options=None):
    """Search + accumulate + blend (kernels.py:453-466): (bmus (n,2) int32, CodeBook)."""
    from .train import CodeBook
    _check_dims(data, cb)
    kernel = _check_pair(kernel, data)
    eng = make_engine(data, cb.n_columns, cb.n_rows, map_type, grid, options=options)
    eng.set_codebook(cb.weights)
    eng.search(_lib.DIST_NAIVE if kernel is Kernel.DENSE_NAIVE else _lib.DIST_BLOCKED)
    eng.node_sums()
    eng.update(radius, scale, cutoff, neighborhood, compact, all_nodes=True)
    bmu = eng.bmu[: eng.n].to(torch.int64).cpu().numpy()
    new_cb = CodeBook(cb.n_columns, cb.n_rows, cb.n_dimensions, eng.codebook())
    return _to_coords(bmu, cb.n_columns), new_cb


def _bmu_only(data, cb, kernel, options=None):
    _check_dims(data, cb)
    kernel = _check_pair(kernel, data)
    eng = make_engine(data, cb.n_columns, cb.n_rows, MapType.PLANAR, options=options)
    eng.set_codebook(cb.weights)
    eng.search(_lib.DIST_NAIVE if kernel is Kernel.DENSE_NAIVE else _lib.DIST_BLOCKED)
    return _to_coords(eng.bmu[: eng.n].to(torch.int64).cpu().numpy(), cb.n_columns)


def bmu_search_naive(data: DenseDataset, cb, options=None) -> np.ndarray:
    """kernels.py:265-275."""
    if not isinstance(data, DenseDataset):
        _check_dims(data, cb)
        raise errors.KernelDataMismatch("dense kernel requires dense data")
    return _bmu_only(data, cb, Kernel.DENSE_NAIVE, options)


def bmu_search_blocked(data: DenseDataset, cb, block_size: int = DEFAULT_BLOCK_SIZE,
                       options=None) -> np.ndarray:
    """kernels.py:278-295 (block size is a pure scheduling choice)."""
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    if not isinstance(data, DenseDataset):
        _check_dims(data, cb)
        raise errors.KernelDataMismatch("dense kernel requires dense data")
    return _bmu_only(data, cb, Kernel.DENSE_BLOCKED, options)


def bmu_search_sparse(data: SparseDataset, cb, options=None) -> np.ndarray:
    """kernels.py:298-312."""
    if not isinstance(data, SparseDataset):
        _check_dims(data, cb)
        raise errors.KernelDataMismatch("sparse kernel requires sparse data")
    return _bmu_only(data, cb, Kernel.SPARSE, options)
