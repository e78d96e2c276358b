"""ctypes binding of the native library libsomb200.so (include/somb200.h).

The product path has no CPU fallback: importing works anywhere, but the
first call that needs the library raises DeviceError if the shared object
is missing, cannot load, or the device is not an sm_100 B200.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsomb200.so")
# A/B measurement only (tools/ab.sh): load another build of the same library
if os.environ.get("SOMB_LIB_PATH"):
    LIB_PATH = os.environ["SOMB_LIB_PATH"]

SOMB_OK, SOMB_E_CONFIG, SOMB_E_INPUT, SOMB_E_CUDA, SOMB_E_ARCH = 0, 1, 2, 3, 4
GRID_RECT, GRID_HEX = 0, 1
PLANAR, TOROID = 0, 1
NBH_GAUSSIAN, NBH_BUBBLE = 0, 1
DIST_NAIVE, DIST_BLOCKED = 0, 1
CAND_CAP = 64


class SombMap(C.Structure):
    _fields_ = [("n_columns", C.c_int32), ("n_rows", C.c_int32),
                ("grid", C.c_int32), ("topology", C.c_int32)]


class SombHood(C.Structure):
    _fields_ = [("neighborhood", C.c_int32), ("compact", C.c_int32),
                ("radius", C.c_double), ("cutoff", C.c_double),
                ("method", C.c_int32), ("reserved", C.c_int32)]


CONV_AUTO, CONV_DIRECT, CONV_SPECTRAL = 0, 1, 2


P = C.c_void_p
I32, I64, F32, F64, SZ = C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_size_t

# name -> (restype, argtypes); the exported surface of include/somb200.h
SIGNATURES = {
    "somb_version": (C.c_char_p, []),
    "somb_last_error": (C.c_char_p, []),
    "somb_device_check": (C.c_int, [C.c_int]),
    "somb_data_stats_ws": (SZ, [I32]),
    "somb_data_stats": (C.c_int, [P, I64, I32, P, P, P, P]),
    "somb_data_pack": (C.c_int, [P, I64, I32, P, I32, P, P, I32, P, P, P, P]),
    "somb_codebook_ws": (SZ, [I32, I32]),
    "somb_codebook_prepare": (C.c_int, [P, I32, I32, P, I32, P, P, I32, I32, P, P, P, P, P]),
    "somb_bmu_ws": (SZ, [I64]),
    "somb_bmu_dense": (C.c_int, [P, P, P, P, I64, I32, I32, P, P, P, P, I32, I32, P, F32,
                                 I32, I32, P, P, P, P, P]),
    "somb_bmu_screen": (C.c_int, [P, P, P, I64, I32, P, P, P, I32, I32, P, F32, P, I32, P, P, P]),
    "somb_debug_screen_dump": (C.c_int, [P, P, P, I64, I32, P, P, P, I32, P, F32, I32, P, P, P]),
    "somb_data_pack_f8": (C.c_int, [P, I64, I32, P, I32, P, P, I32, P, P, P, P]),
    "somb_codebook_prepare_f8": (C.c_int, [P, I32, I32, P, I32, P, P, I32, I32, P, P, P, P, P]),
    "somb_bmu_rerank": (C.c_int, [P, P, I64, I32, P, P, I32, I32, I32, P, P, P, P, P, P]),
    "somb_l2_probe": (C.c_int, [P, I64, I32, P, P]),
    "somb_bmu_search": (C.c_int, [P, P, P, P, P, I64, I32, I32, P, P, P, P, P, I32, I32, P, F32, P, P, I32,
                                  I32, P, P, P, P, P]),
    "somb_qe_sum": (C.c_int, [P, I64, P, P, P]),
    "somb_bmu_repaired_rows": (I64, [P, I64, P]),
    "somb_launch_count": (C.c_ulonglong, []),
    "somb_format_f32_rows": (I64, [P, I64, I64, P, I64, I32]),
    "somb_format_bmus": (I64, [P, I64, P, I64, I32]),
    "somb_scan_dense_text": (I64, [P, I64, P, P, P]),
    "somb_parse_dense_text": (I64, [P, I64, I64, I64, P, I32]),
    "somb_uniform_f32": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, I64, P, P]),
    "somb_set_knob": (C.c_int, [C.c_char_p, I32]),
    "somb_node_sums_ws": (SZ, [I64, I32, I32]),
    "somb_node_sums_dense": (C.c_int, [P, I64, I32, P, I32, P, P, P, P, P]),
    "somb_node_sums_dense_cols": (C.c_int, [P, I64, I32, P, I32, I32, P, P, P, P, P]),
    "somb_hood_ws": (SZ, [C.POINTER(SombMap), I32, I32]),
    "somb_hood_update": (C.c_int, [P, P, I32, C.POINTER(SombMap), C.POINTER(SombHood), F64, P,
                                   P, I32, I32, P, P, P, P, P]),
    "somb_blend": (C.c_int, [P, P, P, I32, I32, F64, P, P]),
    "somb_sparse_row_stats": (C.c_int, [P, P, I64, P, P, P, P]),
    "somb_sparse_codebook_T": (C.c_int, [P, P, I32, I32, I32, P, P]),
    "somb_bmu_sparse": (C.c_int, [P, P, P, I64, I32, P, P, P, P, I32, I32, P, P, P, F32, I32,
                                  P, P, P, P, P]),
    "somb_bmu_sparse_ws": (SZ, [I64]),
    "somb_bmu_sparse_repair": (C.c_int, [P, P, P, I64, I32, P, I32, I32, P, P, P, P, P, P, P]),
    "somb_node_sums_sparse": (C.c_int, [P, P, P, I64, I32, P, I32, P, P, P, P, P]),
    "somb_node_sums_sparse_cols": (C.c_int, [P, P, P, I64, I32, P, I32, I32, P, P, P, P, P]),
    "somb_umatrix": (C.c_int, [P, I32, C.POINTER(SombMap), P, P]),
}

_lib = None
_lock = threading.Lock()
_checked_devices = set()


def load(path: str = LIB_PATH):
    """Load the shared library (no device needed).  Raises DeviceError."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise errors.DeviceError(
                f"native library {path} is missing; run `make` (or __graft_entry__.build())")
        try:
            lib = C.CDLL(path)
        except OSError as exc:
            raise errors.DeviceError(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    return load().somb_last_error().decode(errors="replace")


def check(status: int, what: str) -> None:
    if status == SOMB_OK:
        return
    msg = f"{what}: {last_error()}"
    if status == SOMB_E_CONFIG:
        raise errors.InvalidConfig(msg)
    if status == SOMB_E_INPUT:
        raise errors.InputError(msg)
    raise errors.DeviceError(msg)


def require_device(dev: int) -> None:
    """Fail loudly unless `dev` is a B200 the library can run on."""
    if dev in _checked_devices:
        return
    lib = load()
    check(lib.somb_device_check(dev), f"device cuda:{dev}")
    _checked_devices.add(dev)


def call(name: str, *args):
    """Invoke an int-returning entry point and raise on a non-zero status."""
    check(getattr(load(), name)(*args), name)
