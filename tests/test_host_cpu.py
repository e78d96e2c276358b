"""CPU-only checks: host logic mirrors the reference, the C-ABI library loads
and exports every symbol include/somb200.h declares, and the product path
fails loudly without a GPU (no CPU fallback)."""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_1305_1422_b200 as S
from paper_1305_1422_b200 import _lib, errors
from conftest import ROOT


def test_header_symbols_exported_and_bound():
    hdr = open(os.path.join(ROOT, "include", "somb200.h")).read()
    declared = set(re.findall(r"SOMB_API\s+[\w\s\*]+?\b(somb_\w+)\s*\(", hdr))
    assert declared, "no declarations found"
    lib = os.path.join(ROOT, "paper_1305_1422_b200", "libsomb200.so")
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (somb_\w+)", out))
    assert declared <= exported, declared - exported
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    L = _lib.load()
    assert L.somb_version().startswith(b"somb200")
    assert L.somb_bmu_ws(1000) > 0 and L.somb_node_sums_ws(1000, 8, 16) > 0


def test_library_is_sm100a_only():
    lib = os.path.join(ROOT, "paper_1305_1422_b200", "libsomb200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    x = S.gen_random_dense(20, 3, 1)
    with pytest.raises(errors.DeviceError):
        S.train(x, S.TrainConfig(n_epochs=1, n_columns=3, n_rows=2))


def test_resolve_defaults_and_validation():
    c = S.resolve_defaults(S.TrainConfig(n_columns=12, n_rows=8))
    assert (c.radius0, c.radiusN, c.scale0, c.scaleN) == (4.0, 1.0, 1.0, 0.01)
    assert S.resolve_defaults(S.TrainConfig(n_columns=1, n_rows=30)).radius0 == 1.0
    for bad in [dict(n_epochs=0), dict(n_columns=0), dict(radius0=-2), dict(scale0=-0.5),
                dict(influence_cutoff=-1e-3), dict(snapshot_level=3)]:
        with pytest.raises(errors.InvalidConfig):
            S.resolve_defaults(S.TrainConfig(**bad))
    with pytest.raises(errors.InvalidConfig):
        S.resolve_defaults(S.TrainConfig(n_rows=5, grid=S.GridType.HEXAGONAL,
                                         map_type=S.MapType.TOROID))


@pytest.mark.parametrize("cool", [S.Cooling.LINEAR, S.Cooling.EXPONENTIAL])
def test_schedule_matches_oracle(cool):
    rng = np.random.default_rng(5)
    for _ in range(200):
        a = float(rng.uniform(1, 50)); b = float(rng.uniform(0.5, a)); e = int(rng.integers(1, 20))
        for t in range(e):
            assert S.schedule(a, b, cool, t, e) == O.schedule(a, b, cool.value, t, e)


def test_init_codebook_matches_reference_stream():
    cfg = S.resolve_defaults(S.TrainConfig(n_columns=6, n_rows=5, seed=9))
    assert np.array_equal(S.init_codebook(cfg, 4).weights, O.init_codebook(6, 5, 4, 9))


def test_generators_match_reference_streams():
    assert np.array_equal(S.gen_random_dense(50, 7, 3).values, O.gen_random_dense(50, 7, 3))
    a, b = S.gen_random_sparse(40, 30, 0.2, 4), O.gen_random_sparse(40, 30, 0.2, 4)
    assert np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert np.array_equal(a.values, b.values)


def test_grid_distance_and_neighbors_match_oracle():
    for nx, ny in [(1, 1), (2, 3), (5, 4), (8, 8)]:
        for mt in (S.MapType.PLANAR, S.MapType.TOROID):
            for g in (S.GridType.RECTANGULAR, S.GridType.HEXAGONAL):
                if g is S.GridType.HEXAGONAL and mt is S.MapType.TOROID and ny % 2:
                    continue
                og = O.HEX if g is S.GridType.HEXAGONAL else O.RECT
                for j in range(nx * ny):
                    c, r = j % nx, j // nx
                    got = [(q.col, q.row) for q in S.neighbors(S.GridCoord(c, r), mt, nx, ny, g)]
                    assert got == O.neighbors(c, r, nx, ny, mt.value, og)
                    for k in range(nx * ny):
                        d = S.grid_distance(S.GridCoord(c, r), S.GridCoord(k % nx, k // nx),
                                            mt, nx, ny, g)
                        assert d == pytest.approx(
                            O.grid_distance(c, r, k % nx, k // nx, nx, ny, mt.value, og), abs=1e-12)


def test_hex_distance_known_answers():
    # extension definition: odd rows shifted by +1/2, row pitch sqrt(3)/2
    h = S.GridType.HEXAGONAL
    g = lambda a, b, mt=S.MapType.PLANAR: S.grid_distance(S.GridCoord(*a), S.GridCoord(*b), mt, 6, 4, h)
    assert g((0, 0), (1, 0)) == 1.0
    assert g((0, 0), (0, 1)) == pytest.approx(1.0)        # odd row neighbour up-right
    assert g((1, 1), (1, 0)) == pytest.approx(1.0)
    assert g((0, 0), (0, 2)) == pytest.approx(np.sqrt(3.0))
    assert g((0, 0), (5, 0), S.MapType.TOROID) == 1.0     # wrap along x
    assert g((0, 0), (0, 3), S.MapType.TOROID) == pytest.approx(1.0)   # wrap along y (even ny)
    assert len(S.neighbors(S.GridCoord(2, 2), S.MapType.PLANAR, 6, 4, h)) == 6


def test_bubble_compact_known_answers():
    P = S.MapType.PLANAR
    nb = S.neighborhood
    a, b = S.GridCoord(0, 0), S.GridCoord(3, 4)
    assert nb(a, b, 5.0, P, 10, 10, kind=S.Neighborhood.BUBBLE) == 1.0
    assert nb(a, b, 4.99, P, 10, 10, kind=S.Neighborhood.BUBBLE) == 0.0
    assert nb(a, b, 4.99, P, 10, 10, compact=True) == 0.0
    assert nb(a, b, 5.0, P, 10, 10, compact=True) == pytest.approx(np.exp(-1.0))
    assert nb(a, a, 2.0, P, 10, 10) == 1.0


def test_partition_matches_reference():
    for n, p in [(10, 3), (7, 8), (1_000_001, 8), (0, 2)]:
        assert S.partition(n, p) == O.partition(n, p)


def test_bindings_validation_errors_before_compute():
    from paper_1305_1422_b200 import bindings as B
    x = np.zeros(12, np.float32)
    cb, bm, um = np.zeros(6 * 3, np.float32), np.zeros(8, np.int32), np.zeros(6, np.float32)
    with pytest.raises(B.ShapeError):
        B.train_wrapper(x, 1, 3, 2, 3, 4, 0, 0, "linear", 0, 0, "linear", 0, 0, "planar", "",
                        cb[:-1], bm, um)
    with pytest.raises(TypeError):
        B.train_wrapper(x.astype(np.float64), 1, 3, 2, 3, 4, 0, 0, "linear", 0, 0, "linear", 0, 0,
                        "planar", "", cb, bm, um)
    with pytest.raises(B.ContiguityError):
        B.train_wrapper(np.zeros(24, np.float32)[::2], 1, 3, 2, 3, 4, 0, 0, "linear", 0, 0,
                        "linear", 0, 0, "planar", "", cb, bm, um)
    with pytest.raises(errors.InvalidConfig):
        B.train_wrapper(x, 1, 3, 2, 3, 4, 0, 0, "linear", 0, 0, "linear", 0, 0, "klein", "",
                        cb, bm, um)


def test_fileio_roundtrip(tmp_path):
    w = np.random.default_rng(1).random((6, 3), dtype=np.float32)
    cb = S.CodeBook(3, 2, 3, w)
    from paper_1305_1422_b200 import fileio
    fileio.write_codebook(cb, str(tmp_path / "a.wts"))
    nx, ny, w2 = fileio.load_codebook(str(tmp_path / "a.wts"))
    assert (nx, ny) == (3, 2)
    np.testing.assert_allclose(w2, w, rtol=1e-5)


def _pcg64_floats(seed, start, count):
    """Restatement of csrc/rng.cu: PCG64 jump-ahead to output start//2, then
    the numpy float32 construction (u >> 8) * 2^-24 from 32-bit halves."""
    st = np.random.PCG64(seed).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    mult, mask = 0x2360ED051FC65DA44385DF649FCCF645, (1 << 128) - 1

    def advance(state, delta):
        acc_m, acc_p, cur_m, cur_p = 1, 0, mult, inc
        while delta:
            if delta & 1:
                acc_m, acc_p = (acc_m * cur_m) & mask, (acc_p * cur_m + cur_p) & mask
            cur_p, cur_m = ((cur_m + 1) * cur_p) & mask, (cur_m * cur_m) & mask
            delta >>= 1
        return (acc_m * state + acc_p) & mask

    k = start // 2
    s = advance(s, k)
    out = []
    while len(out) < count + (start % 2):
        s = (s * mult + inc) & mask
        hi, lo = s >> 64, s & ((1 << 64) - 1)
        v, r = hi ^ lo, s >> 122
        o = ((v >> r) | (v << ((64 - r) & 63))) & ((1 << 64) - 1)
        out += [np.float32((o & 0xFFFFFFFF) >> 8) * np.float32(2.0 ** -24),
                np.float32((o >> 32) >> 8) * np.float32(2.0 ** -24)]
    return np.array(out[start % 2: start % 2 + count], dtype=np.float32)


@pytest.mark.parametrize("seed", [0, 1, 12345])
def test_device_init_restatement_matches_numpy(seed):
    """The jump-ahead used by somb_uniform_f32 reproduces numpy's
    default_rng(seed).random(float32) at arbitrary offsets (train.py:164-166)."""
    ref = np.random.default_rng(seed).random(5000, dtype=np.float32)
    for start, count in [(0, 17), (1, 9), (2048, 33), (4095, 7), (4990, 10)]:
        np.testing.assert_array_equal(_pcg64_floats(seed, start, count), ref[start:start + count])


def test_native_writers_match_reference_format(tmp_path):
    """somb_format_* == the reference's f"{float(v):.6g}" lines
    (fileio.py:322-359), including -0, inf, nan, subnormal-range and
    exponent-boundary values."""
    from paper_1305_1422_b200 import fileio
    rng = np.random.default_rng(11)
    w = (rng.standard_normal((300, 13)) * 10.0 ** rng.integers(-38, 38, (300, 13))).astype(np.float32)
    w[0, :8] = [0.0, -0.0, np.inf, -np.inf, np.nan, 1e-5, 123456.5, 1e6]
    w[1, :5] = [0.1, -3.5e-38, 1e-45, 999999.5, 0.000123456789]
    cb = S.CodeBook(15, 20, 13, w)
    fileio.write_codebook(cb, str(tmp_path / "a.wts"))
    ref = f"% {cb.n_rows} {cb.n_columns}\n% {cb.n_dimensions}\n" + "".join(
        " ".join(f"{float(v):.6g}" for v in node) + "\n" for node in w)
    assert (tmp_path / "a.wts").read_bytes() == ref.encode()
    bm = rng.integers(0, 300, (5000, 2)).astype(np.int32)
    fileio.write_bmus(bm, str(tmp_path / "a.bm"))
    ref = f"% {len(bm)}\n" + "".join(f"{i} {r} {c}\n" for i, (r, c) in enumerate(bm))
    assert (tmp_path / "a.bm").read_bytes() == ref.encode()


def _hex_brute(c1, r1, c2, r2, nx, ny, toroid):
    """Independent hex-lattice distance, the slow obvious way (modelled on the
    reference's grid_distance_brute, tests/oracles.py:11-21): Cartesian node
    positions (c + (r mod 2)/2, r sqrt(3)/2), on a torus the minimum over all
    9 images of the (nx, ny sqrt(3)/2) period lattice."""
    import math
    x1, y1 = c1 + 0.5 * (r1 % 2), r1 * math.sqrt(3.0) / 2.0
    x2, y2 = c2 + 0.5 * (r2 % 2), r2 * math.sqrt(3.0) / 2.0
    shifts = (-1, 0, 1) if toroid else (0,)
    return min(math.hypot(x1 - x2 + a * nx, y1 - y2 + b * ny * math.sqrt(3.0) / 2.0)
               for a in shifts for b in shifts)


@pytest.mark.parametrize("nx,ny", [(6, 4), (5, 6), (7, 2), (3, 8)])
@pytest.mark.parametrize("mt", [S.MapType.PLANAR, S.MapType.TOROID])
def test_hex_distance_vs_9_image_brute_force(nx, ny, mt):
    """The hexagonal extension (package, oracle and -- through the GPU
    update tests -- the device grid_d2) against the brute-force image sum,
    every node pair; neighbours = the nodes at unit distance."""
    tor = mt is S.MapType.TOROID
    h = S.GridType.HEXAGONAL
    d_or = O.distance_rows(np.arange(nx * ny), nx, ny, mt.value, O.HEX)
    for a in range(nx * ny):
        for b in range(nx * ny):
            want = _hex_brute(a % nx, a // nx, b % nx, b // nx, nx, ny, tor)
            got = S.grid_distance(S.GridCoord(a % nx, a // nx), S.GridCoord(b % nx, b // nx), mt, nx, ny, h)
            assert got == pytest.approx(want, abs=1e-12), (a, b)
            assert d_or[a, b] == pytest.approx(want, abs=1e-12), (a, b)
        nb = {(c.row, c.col) for c in S.neighbors(S.GridCoord(a % nx, a // nx), mt, nx, ny, h)}
        unit = {(b // nx, b % nx) for b in range(nx * ny) if b != a
                and abs(_hex_brute(a % nx, a // nx, b % nx, b // nx, nx, ny, tor) - 1.0) < 1e-9}
        assert nb == unit, (a, nb, unit)


# Reference behaviour of the dense parsers on files with several defects
# (first error in file order; within a row: width, non-numeric, non-finite),
# recorded from somkit.fileio.parse_dense / parse_dense_headered
# (fileio.py:130-220) in this container.
@pytest.mark.parametrize("text,exc,msg", [
    ("1 2\n3 x\n4 5 6\n", errors.NonNumericToken, "line 2: token 'x' is not a number"),
    ("1 inf\n3 x\n", errors.NonNumericToken, "line 1: non-finite value"),
    ("1 2\n3 4 5\nx y\n", errors.RowWidthMismatch, "line 2: expected 2 values, got 3"),
    ("1 2\n1e39 0\n3\n", errors.NonNumericToken, "line 2: non-finite value"),
    ("% 3\n% 2\n1 2\nq 1\n1 2 3\n", errors.NonNumericToken, "line 4: token 'q' is not a number"),
    ("% 3\n% 2\n1 2\n1 2 3\nq 1\n", errors.HeaderBodyMismatch, "line 4: expected 2 values, got 3"),
])
def test_dense_error_order_matches_reference(text, exc, msg):
    from paper_1305_1422_b200 import ingest
    parse = ingest.parse_dense_headered if text.startswith("%") else ingest.parse_dense
    with pytest.raises(exc) as ei:
        parse(text)
    assert str(ei.value) == msg


def test_root_exports_reference_io_names():
    # reference __init__.py:13-15 / __all__
    for name in ("read_dataset", "detect_format", "parse_dense", "parse_dense_headered", "parse_sparse",
                 "write_codebook", "write_bmus", "write_umatrix", "snapshot_paths"):
        assert callable(getattr(S, name)) and name in S.__all__


def test_bindings_sparse_branch_validation(tmp_path):
    # bindings/__init__.py:91-98: kernel_type 2 reads a sparse file; a dense
    # file is InvalidConfig, a wrong n_vectors is ShapeError (before compute)
    from paper_1305_1422_b200 import bindings as B
    sp = tmp_path / "x.sparse"
    sp.write_text("0:1 2:0.5\n1:2\n")
    dn = tmp_path / "x.dense"
    dn.write_text("1 2 3\n4 5 6\n")
    cb, bm, um = np.zeros(6 * 3, np.float32), np.zeros(4, np.int32), np.zeros(6, np.float32)
    with pytest.raises(errors.InvalidConfig):
        B.train_wrapper(str(dn), 1, 3, 2, 3, 2, 0, 0, "linear", 0, 0, "linear", 0, 2, "planar", "", cb, bm, um)
    with pytest.raises(B.ShapeError):
        B.train_wrapper(str(sp), 1, 3, 2, 3, 3, 0, 0, "linear", 0, 0, "linear", 0, 2, "planar", "", cb, bm, um)


@pytest.mark.parametrize("nbh,compact", [("gaussian", False), ("gaussian", True), ("bubble", False), ("bubble", True)])
@pytest.mark.parametrize("mt", ["planar", "toroid"])
def test_hex_epoch_vs_brute_force(nbh, compact, mt):
    """The extension's whole epoch (hex lattice x bubble / compact support) in
    the oracle against a brute-force restatement written the slow obvious way,
    like the reference's epoch_brute (tests/oracles.py:41-79, used by
    test_acceptance.py:87-118): BMU by a full fp64 scan with first-minimum
    ties, then for every (row, node) pair h from the 9-image hex distance,
    num += h x, den += h.  Pins the oracle's extension semantics (the GPU
    update is checked against the oracle, test_gpu_parity.py)."""
    import math
    rng = np.random.default_rng(11)
    nx, ny, n, d = 6, 4, 60, 3
    x = rng.random((n, d), dtype=np.float32)
    w = rng.random((nx * ny, d), dtype=np.float32)
    radius, cutoff = 1.7, 1e-3
    tor = mt == "toroid"
    ob, _, num, den = O.search_accumulate(x, w, nx, ny, radius, cutoff, mt, O.DENSE_BLOCKED, grid=O.HEX,
                                          neighborhood=nbh, compact=compact)
    bnum = np.zeros((nx * ny, d))
    bden = np.zeros(nx * ny)
    for i in range(n):
        d2 = [float(np.sum((x[i].astype(np.float64) - w[j].astype(np.float64)) ** 2)) for j in range(nx * ny)]
        b = min(range(nx * ny), key=lambda j: (d2[j], j))
        for j in range(nx * ny):
            dist = _hex_brute(b % nx, b // nx, j % nx, j // nx, nx, ny, tor)
            if nbh == "bubble":
                h = 1.0 if dist <= radius else 0.0
            else:
                h = math.exp(dist / -radius)
                if compact and dist > radius:
                    h = 0.0
            if h < cutoff:
                h = 0.0
            bnum[j] += h * x[i].astype(np.float64)
            bden[j] += h
        assert ob[i] == b or abs(d2[ob[i]] - d2[b]) <= 1e-12 * d2[b]
    np.testing.assert_allclose(num, bnum, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(den, bden, rtol=1e-12, atol=1e-12)
