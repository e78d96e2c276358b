"""numpy restatement of the reference batch-SOM epoch (TEST INFRASTRUCTURE).

Every function names the reference file:line it restates; paths are relative
to /root/reference/pkg/src/somkit/.  Arithmetic follows the reference
operation-for-operation (fp64 from f32 storage, fixed 256-row chunks folded
in chunk order, first-minimum argmin), so on the same BLAS it reproduces the
reference bit for bit; `tests/test_oracle_golden.py` pins that against
fixtures produced by the reference itself.

Extensions (no reference counterpart, builder definitions -- see DESIGN.md):
hexagonal offset-row grid, bubble neighbourhood, compact support.
"""

from __future__ import annotations

import math
from collections import deque
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Optional

import numpy as np

try:  # the reference pins BLAS to one thread inside its pool (kernels.py:165)
    from threadpoolctl import threadpool_limits
except Exception:  # pragma: no cover - threadpoolctl is in the image
    threadpool_limits = None

__all__ = [
    "PLANAR", "TOROID", "RECT", "HEX", "GAUSSIAN", "BUBBLE",
    "DENSE_NAIVE", "DENSE_BLOCKED", "SPARSE", "CHUNK", "DEFAULT_CUTOFF",
    "CSR", "node_coords", "grid_distance", "distance_rows", "h_rows",
    "neighbors", "search_chunk_blocked", "search_chunk_naive",
    "search_chunk_sparse", "sparse_row_norms", "search_accumulate", "blend",
    "umatrix", "schedule", "resolve_defaults", "init_codebook",
    "epoch_schedules", "train", "partition", "gen_random_dense",
    "gen_random_sparse", "top2_gaps", "node_sums", "conv_update",
]

PLANAR, TOROID = "planar", "toroid"          # grid.py:15-17
RECT, HEX = "rectangular", "hexagonal"       # extension
GAUSSIAN, BUBBLE = "gaussian", "bubble"      # extension (reference: gaussian only)
DENSE_NAIVE, DENSE_BLOCKED, SPARSE = 0, 1, 2  # kernels.py:51-54
CHUNK = 256                                  # kernels.py:62
DEFAULT_CUTOFF = 1e-3                        # kernels.py:58
_SQRT3_2 = math.sqrt(3.0) / 2.0


@dataclass
class CSR:
    """CSR rows: int64 offsets, int32 sorted cols, f32 vals (fileio.py:56-95)."""
    n_dimensions: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def n_vectors(self) -> int:
        return len(self.row_offsets) - 1

    def row(self, i):
        s, e = self.row_offsets[i], self.row_offsets[i + 1]
        return self.col_indices[s:e], self.values[s:e]

    def densify(self) -> np.ndarray:
        out = np.zeros((self.n_vectors, self.n_dimensions), dtype=np.float32)
        for i in range(self.n_vectors):
            c, v = self.row(i)
            out[i, c] = v
        return out


# ------------------------------------------------------------------ geometry

def node_coords(nx: int, ny: int):
    """(cols, rows) int64 over flat row-major order (kernels.py:89-96)."""
    idx = np.arange(nx * ny, dtype=np.int64)
    rows, cols = np.divmod(idx, nx)
    return cols, rows


def _rect_dxdy(c1, r1, c2, r2, nx, ny, map_type):
    # kernels.py:107-111 / 122-126: |dc|, |dr| as f64, toroid min-wrap per axis
    dx = np.abs(c1 - c2).astype(np.float64)
    dy = np.abs(r1 - r2).astype(np.float64)
    if map_type == TOROID:
        np.minimum(dx, nx - dx, out=dx)
        np.minimum(dy, ny - dy, out=dy)
    return dx, dy


def _hex_d2(c1, r1, c2, r2, nx, ny, map_type):
    """Extension: offset-row hex lattice, node (c, r) at (c + (r&1)/2, r*sqrt3/2).

    Squared distance is exact in fp64: dx is a multiple of 1/2 and
    dy^2 = 0.75 * dr^2.  Toroid = min over the 9 images of the rectangular
    period lattice (nx, ny*sqrt3/2), i.e. per-axis min-wrap; ny must be even.
    """
    x1 = c1.astype(np.float64) + 0.5 * (r1 & 1)
    x2 = c2.astype(np.float64) + 0.5 * (r2 & 1)
    dx = np.abs(x1 - x2)
    dr = np.abs(r1 - r2).astype(np.float64)
    if map_type == TOROID:
        np.minimum(dx, nx - dx, out=dx)
        np.minimum(dr, ny - dr, out=dr)
    return dx * dx + 0.75 * (dr * dr)


def distance_rows(bmu_idx, nx, ny, map_type, grid=RECT):
    """Grid distance from each BMU in bmu_idx to every node (len(bmu) x K).

    Rect: np.hypot exactly as kernels.py:112 / 127.  Hex: sqrt of the exact d2.
    """
    cols, rows = node_coords(nx, ny)
    b = np.asarray(bmu_idx, dtype=np.int64)
    if grid == HEX:
        return np.sqrt(_hex_d2(cols[b][:, None], rows[b][:, None],
                               cols[None, :], rows[None, :], nx, ny, map_type))
    dx, dy = _rect_dxdy(cols[b][:, None], rows[b][:, None],
                        cols[None, :], rows[None, :], nx, ny, map_type)
    return np.hypot(dx, dy)


def grid_distance(c1, r1, c2, r2, nx, ny, map_type, grid=RECT) -> float:
    """Scalar grid distance (grid.py:38-49; hex = extension)."""
    d = distance_rows(np.array([r1 * nx + c1]), nx, ny, map_type, grid)
    return float(d[0, r2 * nx + c2])


def h_rows(bmu_idx, radius, cutoff, nx, ny, map_type, grid=RECT,
           neighborhood=GAUSSIAN, compact=False):
    """Influence rows for a batch of BMUs (kernels.py:117-150).

    gaussian: h = exp(d / -radius) (kernels.py:128-129, :139) -- unsquared d.
    bubble (ext.): h = 1 where d <= radius else 0.
    compact (ext.): additionally h = 0 where d > radius.
    cutoff: h[h < cutoff] = 0 (kernels.py:146-147).
    """
    d = distance_rows(bmu_idx, nx, ny, map_type, grid)
    if neighborhood == BUBBLE:
        h = (d <= radius).astype(np.float64)
    else:
        h = np.exp(d / -radius)
        if compact:
            h[d > radius] = 0.0
    if cutoff > 0.0:
        h[h < cutoff] = 0.0
    return h


def neighbors(col, row, nx, ny, map_type, grid=RECT):
    """U-matrix adjacency (grid.py:52-73: Moore-8, scan order, dedup, no self).

    Hex (ext.): the 6 unit-distance offset-row neighbours, same rules.
    """
    if grid == HEX:
        if row & 1:
            offs = ((0, -1), (1, -1), (-1, 0), (1, 0), (0, 1), (1, 1))
        else:
            offs = ((-1, -1), (0, -1), (-1, 0), (1, 0), (-1, 1), (0, 1))
    else:
        offs = tuple((dc, dr) for dr in (-1, 0, 1) for dc in (-1, 0, 1)
                     if (dc, dr) != (0, 0))
    out, seen = [], set()
    for dc, dr in offs:
        c, r = col + dc, row + dr
        if map_type == TOROID:
            c %= nx
            r %= ny
        elif not (0 <= c < nx and 0 <= r < ny):
            continue
        if (c, r) == (col, row) or (c, r) in seen:
            continue
        seen.add((c, r))
        out.append((c, r))
    return out


# ------------------------------------------------------------- chunk kernels

def search_chunk_naive(x64, w64):
    """kernels.py:182-192: per row sum((w - x)^2), first argmin."""
    m = x64.shape[0]
    idx = np.empty(m, dtype=np.int64)
    d2min = np.empty(m, dtype=np.float64)
    for i in range(m):
        diff = w64 - x64[i]
        d2 = np.einsum("jd,jd->j", diff, diff)
        k = int(np.argmin(d2))
        idx[i] = k
        d2min[i] = d2[k]
    return idx, d2min


def search_chunk_blocked(x64, w64, w2):
    """kernels.py:195-205: d2 = -2 x.w^T + |x|^2 + |w|^2, clamp >= 0, argmin."""
    d2 = x64 @ w64.T
    d2 *= -2.0
    d2 += np.einsum("id,id->i", x64, x64)[:, None]
    d2 += w2[None, :]
    np.maximum(d2, 0.0, out=d2)
    idx = np.argmin(d2, axis=1)
    d2min = np.take_along_axis(d2, idx[:, None], axis=1)[:, 0]
    return idx.astype(np.int64), d2min


def sparse_row_norms(data: CSR):
    """kernels.py:315-321 (np.add.at in nnz order)."""
    v64 = data.values.astype(np.float64)
    out = np.zeros(data.n_vectors, dtype=np.float64)
    np.add.at(out, np.repeat(np.arange(data.n_vectors),
                             np.diff(data.row_offsets)), v64 * v64)
    return out


def search_chunk_sparse(data: CSR, first, last, w64, w2, x2):
    """kernels.py:208-222: gathered dots, d2 = x2 - 2 dots + w2, clamp, argmin."""
    m = last - first
    dots = np.zeros((m, w64.shape[0]), dtype=np.float64)
    for i in range(m):
        cols, vals = data.row(first + i)
        if len(cols):
            dots[i] = vals.astype(np.float64) @ w64[:, cols].T
    d2 = x2[first:last, None] - 2.0 * dots
    d2 += w2[None, :]
    np.maximum(d2, 0.0, out=d2)
    idx = np.argmin(d2, axis=1)
    d2min = np.take_along_axis(d2, idx[:, None], axis=1)[:, 0]
    return idx.astype(np.int64), d2min


def _accumulate_chunk_sparse(data: CSR, first, last, h, d):
    """kernels.py:229-242: per-row outer-product scatter; empty rows add to den."""
    num = np.zeros((h.shape[1], d), dtype=np.float64)
    den = h.sum(axis=0)
    for i in range(last - first):
        cols, vals = data.row(first + i)
        if not len(cols):
            continue
        active = np.flatnonzero(h[i])
        if len(active):
            num[np.ix_(active, cols)] += np.outer(h[i, active],
                                                  vals.astype(np.float64))
    return num, den


def _run_chunks(jobs, workers, consume):
    """kernels.py:159-177: bounded pool, results consumed in job order."""
    ctx = threadpool_limits(limits=1) if threadpool_limits else None
    try:
        if ctx is not None:
            ctx.__enter__()
        if workers <= 1 or len(jobs) <= 1:
            for job in jobs:
                consume(job())
            return
        with ThreadPoolExecutor(max_workers=workers) as pool:
            inflight = deque()
            for job in jobs:
                inflight.append(pool.submit(job))
                if len(inflight) > workers + 2:
                    consume(inflight.popleft().result())
            while inflight:
                consume(inflight.popleft().result())
    finally:
        if ctx is not None:
            ctx.__exit__(None, None, None)


def search_accumulate(data, weights, nx, ny, radius, cutoff, map_type,
                      kernel=DENSE_BLOCKED, workers=1, with_accumulators=True,
                      grid=RECT, neighborhood=GAUSSIAN, compact=False):
    """kernels.py:365-435.  data: f32 (N, D) ndarray or CSR.

    Returns (bmu int64[N], qe_sum float, num f64[K,D] | None, den f64[K] | None).
    """
    sparse = isinstance(data, CSR)
    if (kernel == SPARSE) != sparse:
        raise ValueError("kernel/data mismatch")  # kernels.py:377-382
    n = data.n_vectors if sparse else data.shape[0]
    d = data.n_dimensions if sparse else data.shape[1]
    k = nx * ny
    w64 = weights.astype(np.float64)               # kernels.py:247-248, 386
    w2 = np.einsum("jd,jd->j", w64, w64)           # kernels.py:389-390
    x2 = sparse_row_norms(data) if sparse else None

    def job(a, b):
        x64 = None
        if sparse:
            idx, d2min = search_chunk_sparse(data, a, b, w64, w2, x2)
        else:
            x64 = data[a:b].astype(np.float64)     # kernels.py:402
            if kernel == DENSE_BLOCKED:
                idx, d2min = search_chunk_blocked(x64, w64, w2)
            else:
                idx, d2min = search_chunk_naive(x64, w64)
        qe = float(np.sqrt(d2min).sum())           # kernels.py:407
        if not with_accumulators:
            return a, idx, qe, None, None
        h = h_rows(idx, radius, cutoff, nx, ny, map_type, grid,
                   neighborhood, compact)          # kernels.py:410
        if sparse:
            num, den = _accumulate_chunk_sparse(data, a, b, h, d)
        else:
            num, den = h.T @ x64, h.sum(axis=0)    # kernels.py:225-226
        return a, idx, qe, num, den

    bmu = np.empty(n, dtype=np.int64)
    qe_sum = 0.0
    num_t = np.zeros((k, d), dtype=np.float64) if with_accumulators else None
    den_t = np.zeros(k, dtype=np.float64) if with_accumulators else None

    def consume(res):                               # kernels.py:423-430
        nonlocal qe_sum
        a, idx, qe, num, den = res
        bmu[a:a + len(idx)] = idx
        qe_sum += qe
        if num_t is not None:
            num_t[...] += num
            den_t[...] += den

    jobs = [(lambda a=a, b=min(a + CHUNK, n): job(a, b))
            for a in range(0, n, CHUNK)]
    _run_chunks(jobs, workers, consume)
    return bmu, qe_sum, num_t, den_t


def blend(weights, num, den, scale):
    """kernels.py:438-450: fp64 blend where den > 0, one rounding to f32."""
    out = weights.copy()
    mask = den > 0.0
    if mask.any():
        upd = num[mask] / den[mask][:, None]
        w64 = weights[mask].astype(np.float64)
        out[mask] = ((1.0 - scale) * w64 + scale * upd).astype(np.float32)
    return out


def node_sums(data, bmu, k):
    """S_b = sum_{i: bmu_i = b} x_i (fp64), c_b = |{i}| -- the regrouping the
    GPU path uses: num = H S, den = H c (mathematically kernels.py:225-226)."""
    sparse = isinstance(data, CSR)
    d = data.n_dimensions if sparse else data.shape[1]
    s = np.zeros((k, d), dtype=np.float64)
    c = np.bincount(bmu, minlength=k).astype(np.float64)
    if sparse:
        for i in range(data.n_vectors):
            cols, vals = data.row(i)
            s[bmu[i], cols] += vals.astype(np.float64)
    else:
        np.add.at(s, bmu, data.astype(np.float64))
    return s, c


def conv_update(s, c, nx, ny, radius, cutoff, map_type, grid=RECT,
                neighborhood=GAUSSIAN, compact=False, nodes=None):
    """num_j = sum_b h(b, j) S_b, den_j = sum_b h(b, j) c_b (fp64).

    h is symmetric in (b, j) for every grid/topology here, so the H rows of
    the output nodes serve as the influence matrix."""
    k = nx * ny
    nodes = np.arange(k) if nodes is None else np.asarray(nodes)
    h = h_rows(nodes, radius, cutoff, nx, ny, map_type, grid, neighborhood,
               compact)
    return h @ s, h @ c


def umatrix(weights, nx, ny, map_type, grid=RECT):
    """umatrix.py:26-45: fp64 mean distance to adjacency neighbours -> f32."""
    w64 = weights.astype(np.float64)
    heights = np.zeros((ny, nx), dtype=np.float64)
    for row in range(ny):
        for col in range(nx):
            nb = neighbors(col, row, nx, ny, map_type, grid)
            if not nb:
                continue
            idx = [r * nx + c for c, r in nb]
            diff = w64[idx] - w64[row * nx + col]
            heights[row, col] = np.sqrt(np.einsum("nd,nd->n", diff, diff)).mean()
    return heights.astype(np.float32)


# ------------------------------------------------------------- training loop

def schedule(start, end, cooling, epoch, n_epochs):
    """train.py:121-135 (endpoints exact)."""
    if epoch <= 0:
        return float(start)
    if epoch >= n_epochs - 1:
        return float(end)
    frac = epoch / (n_epochs - 1)
    if cooling == "linear":
        return start + (end - start) * frac
    return start * (end / start) ** frac


def resolve_defaults(n_columns, n_rows, radius0=0.0, radiusN=0.0, scale0=0.0,
                     scaleN=0.0):
    """train.py:101-118 sentinel rules (validation lives in the product)."""
    if radius0 == 0:
        radius0 = max(min(n_columns, n_rows) / 2.0, 1.0)
    if radiusN == 0:
        radiusN = 1.0
    if scale0 == 0:
        scale0 = 1.0
    if scaleN == 0:
        scaleN = 0.01
    return float(radius0), float(radiusN), float(scale0), float(scaleN)


def init_codebook(n_columns, n_rows, d, seed):
    """train.py:164-167: default_rng(seed).random((K, D), float32)."""
    rng = np.random.default_rng(seed)
    return rng.random((n_columns * n_rows, d), dtype=np.float32)


def epoch_schedules(epoch, n_epochs, radius0, radiusN, scale0, scaleN,
                    radius_cooling="linear", scale_cooling="linear"):
    """train.py:209-217."""
    return (schedule(radius0, radiusN, radius_cooling, epoch, n_epochs),
            schedule(scale0, scaleN, scale_cooling, epoch, n_epochs))


def train(data, nx, ny, n_epochs=10, map_type=PLANAR, kernel=DENSE_BLOCKED,
          radius0=0.0, radiusN=0.0, radius_cooling="linear", scale0=0.0,
          scaleN=0.0, scale_cooling="linear", seed=1, cutoff=DEFAULT_CUTOFF,
          initial_codebook=None, workers=1, grid=RECT, neighborhood=GAUSSIAN,
          compact=False, final_kernel=None, record=None):
    """train.py:252-296.  Returns (weights f32 (K,D), bmus int32 (N,2), U f32,
    per-epoch qe list).  The final BMU pass uses `final_kernel` (reference:
    DENSE_NAIVE, train.py:287-291; naive and blocked BMUs are bit-identical,
    SURVEY.md A.3, so the default here is the blocked kernel for speed).
    `record`, if a list, receives the codebook entering every epoch."""
    r0, rN, s0, sN = resolve_defaults(nx, ny, radius0, radiusN, scale0, scaleN)
    sparse = isinstance(data, CSR)
    d = data.n_dimensions if sparse else data.shape[1]
    n = data.n_vectors if sparse else data.shape[0]
    w = (initial_codebook.astype(np.float32).copy() if initial_codebook is not None
         else init_codebook(nx, ny, d, seed))
    qes = []
    for e in range(n_epochs):
        radius, scale = epoch_schedules(e, n_epochs, r0, rN, s0, sN,
                                        radius_cooling, scale_cooling)
        if record is not None:
            record.append(w.copy())
        _, qe_sum, num, den = search_accumulate(
            data, w, nx, ny, radius, cutoff, map_type, kernel, workers, True,
            grid, neighborhood, compact)
        w = blend(w, num, den, scale)
        qes.append(qe_sum / max(n, 1))
    fk = SPARSE if sparse else (DENSE_BLOCKED if final_kernel is None else final_kernel)
    bmu, _, _, _ = search_accumulate(data, w, nx, ny, 1.0, 0.0, map_type, fk,
                                     workers, False, grid)
    bm = np.empty((n, 2), dtype=np.int32)          # kernels.py:257-262
    bm[:, 0] = bmu // nx
    bm[:, 1] = bmu % nx
    return w, bm, umatrix(w, nx, ny, map_type, grid), qes


def partition(n_vectors, p):
    """distributed.py:424-434: contiguous slices, remainder to early ranks."""
    base, extra = divmod(n_vectors, p)
    out, first = [], 0
    for r in range(p):
        cnt = base + (1 if r < extra else 0)
        out.append((first, cnt))
        first += cnt
    return out


def gen_random_dense(n, d, seed):
    """bench.py:85-88."""
    return np.random.default_rng(seed).random((n, d), dtype=np.float32)


def gen_random_sparse(n, d, density, seed):
    """bench.py:91-103 (round(density*d) distinct sorted cols per row)."""
    rng = np.random.default_rng(seed)
    k = max(int(round(density * d)), 0)
    offsets = np.arange(n + 1, dtype=np.int64) * k
    cols = np.empty(n * k, dtype=np.int32)
    for i in range(n):
        cols[i * k:(i + 1) * k] = np.sort(
            rng.choice(d, size=k, replace=False)).astype(np.int32)
    values = rng.random(n * k, dtype=np.float32)
    return CSR(d, offsets, cols, values)


def top2_gaps(data, weights):
    """fp64 (best, second-best) relative gap per row, for tie-aware BMU
    comparison: gap_i = (d2_(2) - d2_(1)) / max(d2_(1), tiny)."""
    x64 = data.densify().astype(np.float64) if isinstance(data, CSR) \
        else data.astype(np.float64)
    w64 = weights.astype(np.float64)
    w2 = np.einsum("jd,jd->j", w64, w64)
    out = np.empty(x64.shape[0])
    for a in range(0, x64.shape[0], CHUNK):
        xb = x64[a:a + CHUNK]
        d2 = -2.0 * (xb @ w64.T) + np.einsum("id,id->i", xb, xb)[:, None] + w2
        np.maximum(d2, 0.0, out=d2)
        if d2.shape[1] < 2:
            out[a:a + CHUNK] = np.inf
            continue
        p = np.partition(d2, 1, axis=1)[:, :2]
        out[a:a + CHUNK] = (p[:, 1] - p[:, 0]) / np.maximum(p[:, 0], 1e-300)
    return out
