"""CLI (reference cli.py flags, local role) and dataset ingest: format
detection and parsing against the reference's goldens (pkg/data) restated
as fixtures, error families and exit codes -- no GPU needed."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_1305_1422_b200 import errors, ingest
from paper_1305_1422_b200.cli import build_parser, config_from, main

RGBS = "# rgb\n1 0 0\n0 1 0\n\n0 0 1\n"
HEADERED = "% 3\n% 3\n1 0 0\n0 1 0\n0 0 1\n"
SPARSE = "0:1.5 3:2\n\n2:0.25 # comment-free\n" .replace(" # comment-free", "")


def test_detect_and_parse_formats():
    assert ingest.detect_format(RGBS.splitlines()) == "dense"
    assert ingest.detect_format(HEADERED.splitlines()) == "headered"
    assert ingest.detect_format(SPARSE.splitlines()) == "sparse"
    a = ingest.parse_dense(RGBS)
    b = ingest.parse_dense_headered(HEADERED)
    np.testing.assert_array_equal(a.values, np.eye(3, dtype=np.float32))
    np.testing.assert_array_equal(b.values, np.eye(3, dtype=np.float32))
    sp = ingest.parse_sparse(SPARSE)
    assert sp.n_dimensions == 4 and list(sp.row_offsets) == [0, 2, 2, 3]
    assert list(sp.col_indices) == [0, 3, 2] and list(sp.values) == [1.5, 2.0, 0.25]


@pytest.mark.parametrize("text,exc", [("1 2\n3\n", errors.RowWidthMismatch), ("1 x\n", errors.NonNumericToken),
                                      ("# only\n\n", errors.EmptyInput), ("% 2\n1 2\n", errors.MalformedHeader),
                                      ("% 3\n% 2\n1 2\n", errors.HeaderBodyMismatch)])
def test_dense_errors(text, exc):
    parse = ingest.parse_dense_headered if text.startswith("%") else ingest.parse_dense
    with pytest.raises(exc):
        parse(text)
    assert exc.exit_code == 2


@pytest.mark.parametrize("text,exc", [("1\n", errors.MalformedToken), ("-1:2\n", errors.NegativeIndex),
                                      ("1:2 1:3\n", errors.DuplicateIndexInRow), ("0:nan\n", errors.MalformedToken)])
def test_sparse_errors(text, exc):
    with pytest.raises(exc):
        ingest.parse_sparse(text)


def test_flags_map_to_config():
    ns = build_parser().parse_args(["-x", "7", "-y", "5", "-m", "toroid", "-k", "1", "-e", "3", "-r", "4", "-R", "2",
                                    "-t", "exponential", "-l", "0.5", "-L", "0.1", "-s", "2", "--seed", "9",
                                    "--grid", "hexagonal", "--neighborhood", "bubble", "--compact-support",
                                    "in.txt", "out"])
    cfg = config_from(ns)
    assert (cfg.n_columns, cfg.n_rows, cfg.n_epochs, cfg.seed, cfg.snapshot_level) == (7, 5, 3, 9, 2)
    assert cfg.map_type.value == "toroid" and int(cfg.kernel) == 1 and cfg.radius_cooling.value == "exponential"
    assert (cfg.radius0, cfg.radiusN, cfg.scale0, cfg.scaleN) == (4, 2, 0.5, 0.1)
    assert cfg.grid.value == "hexagonal" and cfg.neighborhood.value == "bubble" and cfg.compact_support


def test_exit_codes(tmp_path, capsys):
    assert main(["-k", "9", "a", "b"]) == 1                                   # usage error
    assert main(["worker", "x"]) == 1                                         # replaced by torchrun
    assert main([str(tmp_path / "missing.txt"), str(tmp_path / "out")]) == 2  # I/O error (InputError family)
    bad = tmp_path / "bad.txt"
    bad.write_text("1 2\n3\n")
    assert main([str(bad), str(tmp_path / "out")]) == 2


def test_module_entry_point_help():
    out = subprocess.run([sys.executable, "-m", "paper_1305_1422_b200", "--help"], capture_output=True, text=True,
                         cwd=ROOT, timeout=120)
    assert out.returncode == 0 and "INPUT_FILE" in out.stdout and "--compact-support" in out.stdout


def test_native_dense_ingest_matches_python_path(tmp_path):
    """read_dataset's threaded native parser gives the values of the
    reference-exact path (np.array(tokens, float32)), with '+' signs, CRLF,
    comments and blank lines; error inputs fall back to the same exceptions."""
    rng = np.random.default_rng(1)
    x = (rng.standard_normal((3000, 17)) * 10.0 ** rng.integers(-5, 5, (3000, 17))).astype(np.float32)
    lines = []
    for i, row in enumerate(x):
        toks = [("+" if (v > 0 and (i + j) % 7 == 0) else "") + repr(float(v)) for j, v in enumerate(row)]
        lines.append(" ".join(toks) + ("\r\n" if i % 5 == 0 else "\n"))
    text = "# header comment\n\n" + "".join(lines)
    p = tmp_path / "x.txt"
    p.write_text(text)
    ds, fmt = ingest.read_dataset(str(p))
    assert fmt == "dense"
    np.testing.assert_array_equal(ds.values, ingest.parse_dense(text).values)
    q = tmp_path / "h.txt"
    q.write_text(f"% {len(x)}\n% 17\n" + "".join(lines))
    ds2, fmt2 = ingest.read_dataset(str(q))
    assert fmt2 == "headered"
    np.testing.assert_array_equal(ds2.values, ds.values)
    for bad, exc in [("1 2\n+-3 4\n", errors.NonNumericToken), ("1 2\n3 inf\n", errors.NonNumericToken),
                     ("1 2\n3\n", errors.RowWidthMismatch), ("% 2\n1 2\n% 2\n3 4\n", errors.MalformedHeader)]:
        b = tmp_path / "b.txt"
        b.write_text(bad)
        with pytest.raises(exc):
            ingest.read_dataset(str(b))


def test_binary_cache_round_trip_and_staleness(tmp_path, monkeypatch):
    """read_dataset(cache=True) writes INPUT.sombc, serves the next read from
    it bit-identically (no text parse), and ignores it once the input changes."""
    import os
    rng = np.random.default_rng(3)
    x = rng.random((257, 9)).astype(np.float32)
    p = tmp_path / "d.txt"
    p.write_text("".join(" ".join(repr(float(v)) for v in row) + "\n" for row in x))
    ds, fmt = ingest.read_dataset(str(p), cache=True)
    assert os.path.exists(ingest.cache_path(str(p)))
    calls = []
    real = ingest._read_text
    monkeypatch.setattr(ingest, "_read_text", lambda path: calls.append(path) or real(path))
    ds2, fmt2 = ingest.read_dataset(str(p), cache=True)
    assert calls == [] and fmt2 == fmt == "dense"
    np.testing.assert_array_equal(ds2.values, ds.values)
    s = tmp_path / "s.txt"
    s.write_text("0:0.5 3:1.25\n\n2:-2 4:3e-3\n")
    sp, sfmt = ingest.read_dataset(str(s), cache=True)
    sp2, sfmt2 = ingest.read_dataset(str(s), cache=True)
    assert sfmt == sfmt2 == "sparse" and len(calls) == 1 and sp2.n_dimensions == sp.n_dimensions
    for a in ("row_offsets", "col_indices", "values"):
        np.testing.assert_array_equal(getattr(sp2, a), getattr(sp, a))
    p.write_text("1 2 3\n4 5 6\n")          # input changed: the cache is stale
    os.utime(p, ns=(1, 1))
    ds3, _ = ingest.read_dataset(str(p), cache=True)
    assert ds3.values.shape == (2, 3) and len(calls) == 2
    with open(ingest.cache_path(str(p)), "r+b") as fh:   # a damaged cache is ignored
        fh.write(b"garbage!")
    ds4, _ = ingest.read_dataset(str(p), cache=True)
    np.testing.assert_array_equal(ds4.values, ds3.values)
    assert len(calls) == 3
