"""Sparse (CSR) epoch engine: the Kernel.SPARSE path (kernels.py:208-242).

Rows stay in CSR on the device (int64 offsets, int32 sorted cols, f32 vals);
per epoch the centred codebook is transposed to dT [d][kp] fp32 so each
nonzero gathers one contiguous node slice (csrc/sparse.cu).  Node sums are a
deterministic scatter into the dense fp64 K x d accumulator, after which the
update, the all-reduce and the blend are the dense engine's.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib, errors
from .datasets import SparseDataset
from .engine import SomEngine, _ptr, _round_up, _stream, to_device

# rigorous fp32 window for the gather screen: |r~ - r| <= 2 (nnz + 2) 2^-24
# |x| max|delta| (+ c rounding); the window is twice that bound.
_SPARSE_WINDOW = 4.0 * 2.0 ** -24


class SparseEngine(SomEngine):
    _sparse = True

    def _init_data(self, data):
        if not isinstance(data, SparseDataset):
            raise errors.KernelDataMismatch("SparseEngine needs a SparseDataset")
        dev = self.dev
        self.rowptr = to_device(np.ascontiguousarray(data.row_offsets, np.int64), dev)
        self.col = to_device(np.ascontiguousarray(data.col_indices, np.int32), dev)
        self.val = to_device(np.ascontiguousarray(data.values, np.float32), dev)
        if self.col.numel() == 0:
            self.col = torch.zeros(1, dtype=torch.int32, device=dev)
            self.val = torch.zeros(1, dtype=torch.float32, device=dev)
        self.n, self.d = int(data.n_vectors), int(data.n_dimensions)
        self.dp = _round_up(self.d, 8)
        self.passes = 1
        self.xexp = 0
        self.nu = torch.zeros(self.d, dtype=torch.float32, device=dev)   # no data centring
        self.X = None
        n = max(self.n, 1)
        self.x2 = torch.empty(n, dtype=torch.float64, device=dev)
        self.xnorm = torch.empty(n, dtype=torch.float32, device=dev)
        nnz_max = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("somb_sparse_row_stats", _ptr(self.rowptr), _ptr(self.val), self.n, _ptr(self.x2),
                  _ptr(self.xnorm), _ptr(nnz_max), _stream(dev))

    def _init_codebook_buffers(self):
        self.Wh = None
        self.Wl = None
        # the centred codebook transposed (the gather screen); after the screen
        # the repair of truncated rows reuses it for the ORIGINAL codebook
        # transposed (somb_bmu_sparse_repair), and the next prepare rebuilds it
        self.dT = torch.empty((self.d, self.kp), dtype=torch.float32, device=self.dev)

    def _window_coef(self) -> float:
        return _SPARSE_WINDOW

    def prepare(self):
        st = _stream(self.dev)
        _lib.call("somb_codebook_prepare", _ptr(self.W), self.K, self.d, _ptr(self.nu), 0, _ptr(None),
                  _ptr(None), self.dp, self.kp, _ptr(self.c), _ptr(self.w2), _ptr(self.scal),
                  _ptr(self.ws), st)
        # the codebook mean mu is the first d floats of the prepare workspace
        _lib.call("somb_sparse_codebook_T", _ptr(self.W), _ptr(self.ws), self.K, self.d, self.kp,
                  _ptr(self.dT), st)

    def search(self, dist_mode=_lib.DIST_BLOCKED):
        self._mark("prepare", True)
        self.prepare()
        self._mark("prepare", False)
        if self.n == 0:
            return
        self._mark("screen", True)
        _lib.call("somb_bmu_sparse", _ptr(self.rowptr), _ptr(self.col), _ptr(self.val), self.n, self.d,
                  _ptr(self.dT), _ptr(self.W), _ptr(self.c), _ptr(self.w2), self.K, self.kp,
                  _ptr(self.scal), _ptr(self.x2), _ptr(self.xnorm), C.c_float(self.window_coef),
                  1 if self.screen_impl == 2 else 2, _ptr(self.bmu), _ptr(self.d2min), _ptr(self.flags),
                  _ptr(self.ws), _stream(self.dev))
        if self.screen_impl != 2:   # rows whose candidate set was truncated: exact lockstep scan
            _lib.call("somb_bmu_sparse_repair", _ptr(self.rowptr), _ptr(self.col), _ptr(self.val), self.n,
                      self.d, _ptr(self.W), self.K, self.kp, _ptr(self.w2), _ptr(self.x2), _ptr(self.dT),
                      _ptr(self.bmu), _ptr(self.d2min), _ptr(self.ws), _stream(self.dev))
        self._mark("screen", False)
        self.has_prev = True

    def node_sums(self):
        _lib.call("somb_node_sums_sparse_cols", _ptr(self.rowptr), _ptr(self.col), _ptr(self.val), self.n,
                  self.d, _ptr(self.bmu), self.K, self.dc, _ptr(self.S), _ptr(self.cnt), None, _ptr(self.ws),
                  _stream(self.dev))

    def debug_screen_values(self):
        raise NotImplementedError("screen dump is a dense-path calibration tool")

    def candidate_counts(self) -> torch.Tensor:
        off = ((self.n * _lib.CAND_CAP * 4 + 255) // 256) * 256
        return self.ws[off: off + 4 * self.n].view(torch.int32)
