"""Dataset text ingest with the reference formats (fileio.py:1-317): plain
dense, '%'-headered dense and zero-based sparse ``index:value`` rows,
content-detected; '#' comments, LF or CRLF.  Values become float32 exactly
as numpy converts the tokens (the reference's np.array(tokens, float32)).
Rows are converted in bulk (one numpy conversion per file, not per row);
the per-line error checks and messages follow the reference's."""
from __future__ import annotations

import os

import numpy as np

from . import errors
from .datasets import DenseDataset, SparseDataset


def _lines(src) -> list:
    if isinstance(src, bytes):
        src = src.decode("utf-8")
    if not isinstance(src, str):
        src = src.read()
    return src.splitlines()


def _comment(line: str) -> bool:
    return line.lstrip().startswith("#")


def _is_number(tok: str) -> bool:
    try:
        float(tok)
        return True
    except ValueError:
        return False


def _to_f32(tokens: list, lineno_of) -> np.ndarray:
    """Bulk conversion; on failure locate the first bad token for the
    reference's NonNumericToken message (line-accurate)."""
    try:
        vals = np.array(tokens, dtype=np.float32)
    except ValueError:
        for k, t in enumerate(tokens):
            if not _is_number(t):
                raise errors.NonNumericToken(f"line {lineno_of(k)}: token {t!r} is not a number") from None
        raise
    bad = np.flatnonzero(~np.isfinite(vals))
    if bad.size:
        raise errors.NonNumericToken(f"line {lineno_of(int(bad[0]))}: non-finite value")
    return vals


def _dense_body(rows: list, width: int, mismatch) -> DenseDataset:
    """rows: [(lineno, tokens)] that must all hold `width` tokens.  The
    reference checks and converts row by row (fileio.py:150-165, 215-220,
    _parse_row 130-139), so the error raised is the first in file order of
    a width mismatch, a non-numeric token or a non-finite value (within a
    row in that order).  Here the conversion is one bulk numpy call over the
    rows before the first width mismatch, and the failing row is located
    afterwards."""
    n_ok = next((i for i, (_, toks) in enumerate(rows) if len(toks) != width), len(rows))
    flat = [t for _, toks in rows[:n_ok] for t in toks]
    try:
        vals = np.array(flat, dtype=np.float32)
        n_num = n_ok
    except ValueError:   # rows before the first one holding a non-numeric token
        k = next(k for k, t in enumerate(flat) if not _is_number(t))
        n_num = k // max(width, 1)
        vals = np.array(flat[: n_num * width], dtype=np.float32)
    vals = vals.reshape(n_num, width)
    fin = np.isfinite(vals).all(axis=1)
    if not fin.all():
        raise errors.NonNumericToken(f"line {rows[int(np.argmin(fin))][0]}: non-finite value")
    if n_num < n_ok:
        lineno, toks = rows[n_num]
        bad = next((t for t in toks if not _is_number(t)), toks[0])
        raise errors.NonNumericToken(f"line {lineno}: token {bad!r} is not a number")
    if n_ok < len(rows):
        lineno, toks = rows[n_ok]
        raise mismatch(f"line {lineno}: expected {width} values, got {len(toks)}")
    return DenseDataset(vals)


def parse_dense(src) -> DenseDataset:
    """Plain dense text (fileio.py:150-165)."""
    rows = [(no, ln.split()) for no, ln in enumerate(_lines(src), 1) if ln.strip() and not _comment(ln)]
    if not rows:
        raise errors.EmptyInput("no data rows found")
    return _dense_body(rows, len(rows[0][1]), errors.RowWidthMismatch)


def _header_counts(line: str, lineno: int) -> list:
    counts = []
    for tok in line.lstrip()[1:].split():   # "%2" and "% 2" both; trailing words ignored
        try:
            counts.append(int(tok))
        except ValueError:
            break
    if not counts:
        raise errors.MalformedHeader(f"line {lineno}: no count in header {line!r}")
    if min(counts) < 0:
        raise errors.MalformedHeader(f"line {lineno}: negative count in header")
    return counts


def parse_dense_headered(src) -> DenseDataset:
    """Dense text after two '%' count headers: instances (a two-number header
    is a grid whose product is the count), then dimensions (fileio.py:186-229)."""
    headers, rows = [], []
    for no, ln in enumerate(_lines(src), 1):
        s = ln.strip()
        if not s or _comment(ln):
            continue
        if s.startswith("%"):
            if len(headers) == 2:
                raise errors.MalformedHeader(f"line {no}: unexpected extra header")
            headers.append(_header_counts(ln, no))
        elif len(headers) < 2:
            raise errors.MalformedHeader(f"line {no}: data before both header lines")
        else:
            rows.append((no, s.split()))
    if len(headers) < 2:
        raise errors.MalformedHeader("missing '%' header lines")
    n = headers[0][0] * headers[0][1] if len(headers[0]) >= 2 else headers[0][0]
    d = headers[1][0]
    if len(rows) != n:
        raise errors.HeaderBodyMismatch(f"header declares {n} rows, body has {len(rows)}")
    if n == 0:
        return DenseDataset(np.empty((0, d), dtype=np.float32))
    return _dense_body(rows, d, errors.HeaderBodyMismatch)


def parse_sparse(src, n_dimensions_hint=None) -> SparseDataset:
    """Zero-based ``index:value`` rows into CSR, indices sorted per row, a
    duplicate index an error, an empty line an all-zero instance, an empty
    file one all-zero instance (fileio.py:232-283)."""
    lines = _lines(src) or [""]
    offsets, cols, vals = [0], [], []
    top = -1
    for no, ln in enumerate(lines, 1):
        if _comment(ln):
            continue
        row = []
        for tok in ln.split():
            i_s, sep, v_s = tok.partition(":")
            if not sep:
                raise errors.MalformedToken(f"line {no}: token {tok!r} is not index:value")
            try:
                idx = int(i_s)
            except ValueError:
                raise errors.MalformedToken(f"line {no}: bad index in token {tok!r}") from None
            if idx < 0:
                raise errors.NegativeIndex(f"line {no}: index {idx} is negative")
            if not _is_number(v_s):
                raise errors.MalformedToken(f"line {no}: bad value in token {tok!r}")
            v = float(v_s)
            if not np.isfinite(np.float32(v)):
                raise errors.MalformedToken(f"line {no}: non-finite value")
            row.append((idx, v))
        row.sort(key=lambda e: e[0])
        for a, b in zip(row, row[1:]):
            if a[0] == b[0]:
                raise errors.DuplicateIndexInRow(f"line {no}: index {a[0]} appears twice")
        if row:
            top = max(top, row[-1][0])
        cols += [e[0] for e in row]
        vals += [e[1] for e in row]
        offsets.append(len(cols))
    d = top + 1
    if n_dimensions_hint is not None:
        if n_dimensions_hint < d:
            raise errors.HintTooSmall(f"dimension hint {n_dimensions_hint} < required {d}")
        d = n_dimensions_hint
    return SparseDataset(d, np.array(offsets, dtype=np.int64), np.array(cols, dtype=np.int32),
                         np.array(vals, dtype=np.float32))


def detect_format(lines) -> str:
    """'headered' if the first data line starts with '%', 'sparse' if its
    first token holds ':', else 'dense' (fileio.py:286-302)."""
    for ln in lines:
        s = ln.strip()
        if not s or _comment(ln):
            continue
        if s.startswith("%"):
            return "headered"
        return "sparse" if ":" in s.split()[0] else "dense"
    return "dense"


def _native_dense(raw: bytes, fmt: str):
    """Dense / headered body through the library's threaded parser
    (somb_scan_dense_text / somb_parse_dense_text); None when the input needs
    the reference-exact Python path (errors, unusual tokens, header layout)."""
    import ctypes as C
    from . import _lib
    try:
        lib = _lib.load()
    except errors.DeviceError:
        return None
    cols, nh, bad = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    rows = lib.somb_scan_dense_text(raw, len(raw), C.byref(cols), C.byref(nh), C.byref(bad))
    if bad.value or rows == 0:
        return None
    if fmt == "headered":
        if nh.value != 2:
            return None
        head, seen = [], 0
        for no, ln in enumerate(raw.decode("utf-8", errors="replace").splitlines(), 1):
            t = ln.strip()
            if not t or _comment(ln):
                continue
            if not t.startswith("%"):
                break                        # data before the second header: Python path raises
            head.append(_header_counts(ln, no))
            seen += 1
            if seen == 2:
                break
        if len(head) < 2:
            return None
        n = head[0][0] * head[0][1] if len(head[0]) >= 2 else head[0][0]
        if n != rows or head[1][0] != cols.value:
            return None
    elif nh.value:
        return None
    out = np.empty((rows, cols.value), dtype=np.float32)
    rc = lib.somb_parse_dense_text(raw, len(raw), rows, cols.value, out.ctypes.data_as(C.c_void_p),
                                   min(32, os.cpu_count() or 1))
    return DenseDataset(out) if rc == 0 else None


# ------------------------------------------------------------ binary cache
# INPUT.sombc next to a text input: a 64-byte header (magic, the source's
# size and mtime_ns, format, kind, n, d, nnz) and the raw arrays (dense f32
# n x d; CSR int64 offsets, int32 cols, f32 values), read back with one
# np.fromfile per array.  Stale (source changed) or malformed caches are
# ignored and rewritten; an unwritable directory just skips the cache.
_CACHE_MAGIC = b"SOMBC001"
_FMT_CODES = {"dense": 0, "headered": 1, "sparse": 2}


def cache_path(path: str) -> str:
    return path + ".sombc"


def _source_key(path: str):
    st = os.stat(path)
    return st.st_size, st.st_mtime_ns


def load_cached(path: str):
    """(dataset, format) from a fresh INPUT.sombc, else None."""
    cp = cache_path(path)
    try:
        size, mtime = _source_key(path)
        with open(cp, "rb") as fh:
            head = fh.read(64)
        if len(head) < 64 or head[:8] != _CACHE_MAGIC:
            return None
        src_size, src_mtime, code, kind, n, d, nnz = np.frombuffer(head[8:64], dtype="<i8", count=7)
        if (int(src_size), int(src_mtime)) != (size, mtime) or n < 0 or d < 0 or nnz < 0:
            return None
        fmt = {v: k for k, v in _FMT_CODES.items()}.get(int(code))
        total = os.path.getsize(cp)
        if kind == 0:
            if fmt is None or total != 64 + 4 * n * d:
                return None
            vals = np.fromfile(cp, dtype=np.float32, count=int(n * d), offset=64).reshape(int(n), int(d))
            return DenseDataset(vals), fmt
        if kind != 1 or fmt is None or total != 64 + 8 * (n + 1) + 8 * nnz:
            return None
        offs = np.fromfile(cp, dtype=np.int64, count=int(n + 1), offset=64)
        cols = np.fromfile(cp, dtype=np.int32, count=int(nnz), offset=64 + 8 * int(n + 1))
        vals = np.fromfile(cp, dtype=np.float32, count=int(nnz), offset=64 + 8 * int(n + 1) + 4 * int(nnz))
        return SparseDataset(int(d), offs, cols, vals), fmt
    except (OSError, ValueError):
        return None


def write_cache(path: str, ds, fmt: str) -> bool:
    """Write INPUT.sombc atomically (temporary file + rename); False when the
    directory is not writable."""
    cp = cache_path(path)
    tmp = f"{cp}.{os.getpid()}.tmp"
    try:
        size, mtime = _source_key(path)
        sparse = isinstance(ds, SparseDataset)
        n = ds.n_vectors
        d = ds.n_dimensions
        nnz = ds.nnz if sparse else 0
        head = _CACHE_MAGIC + np.array([size, mtime, _FMT_CODES[fmt], int(sparse), n, d, nnz],
                                       dtype="<i8").tobytes()
        with open(tmp, "wb") as fh:
            fh.write(head)
            if sparse:
                fh.write(np.ascontiguousarray(ds.row_offsets, dtype="<i8").tobytes())
                fh.write(np.ascontiguousarray(ds.col_indices, dtype="<i4").tobytes())
                fh.write(np.ascontiguousarray(ds.values, dtype="<f4").tobytes())
            else:
                np.ascontiguousarray(ds.values, dtype="<f4").tofile(fh)
        os.replace(tmp, cp)
        return True
    except OSError:
        try:
            os.unlink(tmp)
        except OSError:
            pass
        return False


def read_dataset(path: str, cache: bool = False):
    """(dataset, format) from a file, format auto-detected (fileio.py:305-317).
    Dense bodies go through the native parser; errors and edge cases through
    the reference-exact Python parsers.  cache=True reuses / refreshes the
    binary copy INPUT.sombc (valid while the input's size and mtime match)."""
    if cache:
        hit = load_cached(path)
        if hit is not None:
            return hit
    ds, fmt = _read_text(path)
    if cache:
        write_cache(path, ds, fmt)
    return ds, fmt


def _read_text(path: str):
    try:
        with open(path, "rb") as fh:
            raw = fh.read()
    except OSError as exc:
        raise errors.IoFailure(f"cannot read {path}: {exc}") from exc
    try:
        head = raw[:1 << 16].decode("utf-8", errors="ignore").splitlines()
        fmt = detect_format(head if len(raw) > (1 << 16) else raw.decode("utf-8").splitlines())
    except UnicodeDecodeError as exc:
        raise errors.IoFailure(f"cannot read {path}: {exc}") from exc
    if fmt in ("dense", "headered"):
        ds = _native_dense(raw, fmt)
        if ds is not None:
            return ds, fmt
    text = raw.decode("utf-8")
    parse = {"sparse": parse_sparse, "headered": parse_dense_headered, "dense": parse_dense}[fmt]
    return parse(text), fmt
