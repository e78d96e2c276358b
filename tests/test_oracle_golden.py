"""Pin the CPU oracle against outputs of the reference implementation itself
(fixtures made by tests/golden/make_golden.py) and against the reference
test-suite's hand-computed known answers."""
import math

import numpy as np
import pytest

import oracle as O
from conftest import cfg1_data, golden


def test_kernel_cases_match_reference():
    g = golden("kernels.npz")
    for ci in range(int(g["ncases"])):
        n, d, nx, ny, tor, radius, cutoff, kern, scale = g[f"c{ci}_params"]
        n, d, nx, ny, kern = int(n), int(d), int(nx), int(ny), int(kern)
        mt = O.TOROID if tor else O.PLANAR
        if kern == 2:
            data = O.CSR(d, g[f"c{ci}_offsets"], g[f"c{ci}_cols"], g[f"c{ci}_vals"])
        else:
            data = g[f"c{ci}_x"]
        w = g[f"c{ci}_w"]
        bmu, qe, num, den = O.search_accumulate(data, w, nx, ny, radius, cutoff, mt,
                                                kern, workers=3)
        assert np.array_equal(bmu, g[f"c{ci}_bmu"]), ci
        assert qe == pytest.approx(float(g[f"c{ci}_qe"]), rel=1e-13)
        np.testing.assert_allclose(num, g[f"c{ci}_num"], rtol=1e-12, atol=1e-300)
        np.testing.assert_allclose(den, g[f"c{ci}_den"], rtol=1e-12, atol=1e-300)
        out = O.blend(w, num, den, scale)
        np.testing.assert_array_max_ulp(out, g[f"c{ci}_blend"], maxulp=1)


def test_node_sum_regrouping_equals_reference_accumulators():
    """num = H S, den = H c (the GPU regrouping) equals the reference's
    per-chunk h^T x accumulation to fp64 rounding."""
    g = golden("kernels.npz")
    for ci in range(int(g["ncases"])):
        n, d, nx, ny, tor, radius, cutoff, kern, scale = g[f"c{ci}_params"]
        if int(kern) == 2:
            data = O.CSR(int(d), g[f"c{ci}_offsets"], g[f"c{ci}_cols"], g[f"c{ci}_vals"])
        else:
            data = g[f"c{ci}_x"]
        nx, ny = int(nx), int(ny)
        s, c = O.node_sums(data, g[f"c{ci}_bmu"], nx * ny)
        num, den = O.conv_update(s, c, nx, ny, radius, cutoff,
                                 O.TOROID if tor else O.PLANAR)
        np.testing.assert_allclose(num, g[f"c{ci}_num"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(den, g[f"c{ci}_den"], rtol=1e-12, atol=1e-12)
        assert np.array_equal(den > 0, g[f"c{ci}_den"] > 0)


def test_umatrix_cases_match_reference():
    g = golden("umatrix.npz")
    for i in range(int(g["ncases"])):
        nx, ny, d, tor = (int(v) for v in g[f"u{i}_shape"])
        u = O.umatrix(g[f"u{i}_w"], nx, ny, O.TOROID if tor else O.PLANAR)
        np.testing.assert_array_max_ulp(u, g[f"u{i}_u"], maxulp=1)


def _cfg(g, name):
    c = g[f"{name}_cfg"]
    return dict(n_epochs=int(c[0]), nx=int(c[1]), ny=int(c[2]),
                map_type=O.TOROID if c[3] else O.PLANAR, radius0=c[4], radiusN=c[5],
                radius_cooling="exponential" if c[6] else "linear", scale0=c[7],
                scaleN=c[8], scale_cooling="exponential" if c[9] else "linear",
                seed=int(c[10]), cutoff=c[11])


@pytest.mark.parametrize("name", ["t0", "t1", "t2", "blobs", "cfg1"])
def test_train_matches_reference(name):
    g = golden("train.npz")
    x = cfg1_data() if name == "cfg1" else g[f"{name}_x"]
    kw = _cfg(g, name)
    w, bm, u, qes = O.train(x, workers=8, **kw)
    assert np.array_equal(bm, g[f"{name}_bmus"])
    np.testing.assert_array_max_ulp(w, g[f"{name}_w"], maxulp=1)
    np.testing.assert_allclose(u, g[f"{name}_u"], rtol=1e-6)
    np.testing.assert_allclose(qes, g[f"{name}_qe"], rtol=1e-12)


def test_sparse_train_matches_reference():
    g = golden("sparse_train.npz")
    for s in ("s0", "s1"):
        e, nx, ny, tor = (int(v) for v in g[f"{s}_cfg"])
        d = 40 if s == "s0" else 500
        data = O.CSR(d, g[f"{s}_offsets"], g[f"{s}_cols"], g[f"{s}_vals"])
        init = g["s0_w0"] if s == "s0" else None
        w, bm, u, qes = O.train(data, nx, ny, n_epochs=e, kernel=O.SPARSE,
                                map_type=O.TOROID if tor else O.PLANAR,
                                initial_codebook=init)
        assert np.array_equal(bm, g[f"{s}_bmus"])
        np.testing.assert_array_max_ulp(w, g[f"{s}_w"], maxulp=1)
        np.testing.assert_allclose(u, g[f"{s}_u"], rtol=1e-6, atol=1e-12)


# --- known answers from the reference test-suite ---------------------------

def test_bmu_hand_case_and_tie_break():
    # reference tests/test_kernels.py:41-62
    w = np.array([[0, 0], [1, 1]], dtype=np.float32)
    x = np.array([[0.4, 0.4], [0.6, 0.6], [0.1, 0.0]], dtype=np.float32)
    bmu, _, _, _ = O.search_accumulate(x, w, 2, 1, 1.0, 0.0, O.PLANAR, O.DENSE_BLOCKED,
                                       with_accumulators=False)
    assert bmu.tolist() == [0, 1, 0]
    w = np.array([[9, 9], [0.5, 0.5], [8, 8], [0.5, 0.5]], dtype=np.float32)
    bmu, _, _, _ = O.search_accumulate(np.array([[0.5, 0.5]], np.float32), w, 2, 2, 1.0,
                                       0.0, O.PLANAR, O.DENSE_NAIVE, with_accumulators=False)
    assert bmu.tolist() == [1]


def test_neighborhood_and_schedule_known_answers():
    # reference tests/test_train.py:68-72, 98-110
    h = O.h_rows(np.array([0]), 2.0, 0.0, 10, 10, O.PLANAR)
    assert h[0, 4 * 10 + 3] == pytest.approx(math.exp(-5.0 / 2.0))
    ht = O.h_rows(np.array([0]), 2.0, 0.0, 10, 10, O.TOROID)
    assert ht[0, 9] == pytest.approx(math.exp(-0.5))
    assert h[0, 0] == 1.0
    vals = [O.schedule(16.0, 1.0, "exponential", e, 5) for e in range(5)]
    assert vals == pytest.approx([16, 8, 4, 2, 1])
    assert O.schedule(8.0, 1.0, "linear", 9, 10) == 1.0


def test_quantization_error_definition():
    # reference tests/test_train.py:241-247: one node at the origin -> qe 2.5
    _, qe, _, _ = O.search_accumulate(np.array([[3, 4], [0, 0]], np.float32),
                                      np.zeros((1, 2), np.float32), 1, 1, 1.0, 0.0,
                                      O.PLANAR, O.DENSE_BLOCKED, with_accumulators=False)
    assert qe / 2 == pytest.approx(2.5)


def test_tiny_radius_cutoff_keeps_only_bmu():
    # reference tests/test_kernels.py:118-129
    rng = np.random.default_rng(2)
    x = rng.random((30, 3), dtype=np.float32)
    w = np.random.default_rng(1).random((25, 3), dtype=np.float32)
    bmu, _, num, den = O.search_accumulate(x, w, 5, 5, 0.1, 1e-3, O.PLANAR)
    for j in range(25):
        m = bmu == j
        assert den[j] == m.sum()
        if m.any():
            np.testing.assert_allclose(num[j], x[m].astype(np.float64).sum(0))


def test_partition_matches_reference_rule():
    # reference distributed.py:424-434
    assert O.partition(10, 3) == [(0, 4), (4, 3), (7, 3)]
    assert sum(c for _, c in O.partition(1_000_001, 8)) == 1_000_001
