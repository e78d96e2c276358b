"""Sparse (CSR) engine -- placeholder until the CSR kernels land."""
from . import errors


class SparseEngine:
    def __init__(self, *a, **k):
        raise errors.DeviceError("the CSR (Kernel.SPARSE) device path is not built yet")
