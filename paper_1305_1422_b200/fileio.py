"""Artifact writers / codebook reader with the reference text formats
(fileio.py:322-401): floats as %.6g, LF endings, formatted by the library's
threaded host formatter (byte-identical, ~10x faster than the reference's
Python loop on the cfg2 codebook).  Text dataset parsing is out of scope for
the B200 hot path."""
from __future__ import annotations

from typing import NamedTuple, Optional

import numpy as np

from . import errors


class SnapshotPaths(NamedTuple):
    codebook: str
    bmus: str
    umatrix: str


def snapshot_paths(prefix: str, epoch: Optional[int] = None) -> SnapshotPaths:
    stem = prefix if epoch is None else f"{prefix}.{epoch}"
    return SnapshotPaths(stem + ".wts", stem + ".bm", stem + ".umx")


def _native_text(fn: str, arr: np.ndarray, *shape) -> memoryview:
    """Format through the library's threaded host formatter (somb_format_*,
    byte-identical to the reference's f"{float(v):.6g}" lines)."""
    import ctypes as C
    import os
    from . import _lib
    lib = _lib.load()
    arr = np.ascontiguousarray(arr)
    threads = min(16, os.cpu_count() or 1)
    cap = arr.size * 16 + (shape[0] if shape else len(arr)) + 64
    while True:
        buf = np.empty(cap, dtype=np.uint8)
        n = getattr(lib, fn)(arr.ctypes.data_as(C.c_void_p), *shape, buf.ctypes.data_as(C.c_void_p), cap, threads)
        if n >= 0:
            return memoryview(buf)[:n]
        cap = -n


def _rows_bytes(mat) -> memoryview:
    m = np.asarray(mat, dtype=np.float32)
    if m.ndim == 1:
        m = m[None, :]
    return _native_text("somb_format_f32_rows", m, m.shape[0], m.shape[1])


def _write(path: str, data) -> None:
    try:
        with open(path, "wb") as fh:
            for part in data:
                fh.write(part.encode("utf-8") if isinstance(part, str) else part)
    except OSError as exc:
        raise errors.IoFailure(f"cannot write {path}: {exc}") from exc


def write_codebook(cb, path: str) -> None:
    """fileio.py:335-342: grid header, dimension header, one node per line."""
    _write(path, [f"% {cb.n_rows} {cb.n_columns}\n% {cb.n_dimensions}\n", _rows_bytes(cb.weights)])


def write_bmus(bmus: np.ndarray, path: str) -> None:
    """fileio.py:345-351: one "index row col" line per instance."""
    b = np.ascontiguousarray(bmus, dtype=np.int32).reshape(-1, 2)
    _write(path, [f"% {len(b)}\n", _native_text("somb_format_bmus", b, len(b))])


def write_umatrix(u, path: str) -> None:
    """fileio.py:354-359: header-less number grid."""
    _write(path, [_rows_bytes(u.heights)])


def load_codebook(path_or_text):
    """Read a .wts codebook -> (n_columns, n_rows, weights f32) (fileio.py:362-401)."""
    if isinstance(path_or_text, str) and "\n" not in path_or_text:
        try:
            with open(path_or_text, "r", encoding="utf-8") as fh:
                text = fh.read()
        except OSError as exc:
            raise errors.IoFailure(f"cannot read {path_or_text}: {exc}") from exc
    else:
        text = path_or_text if isinstance(path_or_text, str) else path_or_text.read()
    headers, body = [], []
    for ln in text.splitlines():
        s = ln.strip()
        if not s or s.startswith("#"):
            continue
        if s.startswith("%") and len(headers) < 2:
            try:
                headers.append([int(t) for t in s[1:].split()])
            except ValueError as exc:
                raise errors.MalformedHeader(f"bad header {ln!r}") from exc
        else:
            body.append(s.split())
    if len(headers) < 2 or len(headers[0]) < 2 or not headers[1]:
        raise errors.MalformedHeader("codebook needs '% rows cols' and '% dims'")
    n_rows, n_columns, d = headers[0][0], headers[0][1], headers[1][0]
    if len(body) != n_rows * n_columns:
        raise errors.CodebookShapeMismatch(
            f"codebook declares {n_rows * n_columns} nodes, file has {len(body)}")
    w = np.empty((n_rows * n_columns, d), dtype=np.float32)
    for i, toks in enumerate(body):
        if len(toks) != d:
            raise errors.CodebookShapeMismatch(f"node {i}: expected {d} values, got {len(toks)}")
        w[i] = [float(t) for t in toks]
    return n_columns, n_rows, w
