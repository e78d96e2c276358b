"""Oracle parity at the shape of every BASELINE config (cfg2-cfg5), on row
slices, teacher-forced over all 10 epochs of the reference schedule: each
epoch the device epoch (tcgen05 screen, fp64 re-rank, node sums, spectral
update) starts from the ORACLE's codebook of the previous epoch, and its
BMUs / codebook are compared with the oracle epoch (oracle/somoracle.py ->
kernels.py:365-450, train.py:269-296).

Data families: uniform [0,1) (the bench data) and structured inputs on which
a round-to-nearest fp16 screen mis-ranks nodes -- near-constant rows,
duplicated columns, Gaussian blobs (reference test_acceptance.py:304-327),
one-hot rows.  Bars: BMUs identical wherever the oracle's
top-2 relative gap is >= 1e-5 (north star), and the codebook within 1e-6
relative of the oracle blend computed from the device's own BMUs (so a
legitimate near-tie flip does not mask an update error)."""
import numpy as np
import pytest

import oracle as O
import paper_1305_1422_b200 as S
from test_gpu_parity import assert_bmus_tie_aware, rel_err

pytestmark = pytest.mark.gpu
WORKERS = 16


def family(name, n, d, seed=1001):
    rng = np.random.default_rng(seed)
    if name == "uniform":
        return rng.random((n, d), dtype=np.float32)
    if name == "nearconst":
        return (rng.random((n, 1)) + 1e-3 * rng.standard_normal((n, d))).astype(np.float32)
    if name == "dupcols":
        return np.repeat(rng.random((n, -(-d // 8)), dtype=np.float32), 8, axis=1)[:, :d].copy()
    if name == "blobs":
        cen = rng.random((20, d))
        return (cen[rng.integers(0, 20, n)] + 0.05 * rng.standard_normal((n, d))).astype(np.float32)
    if name == "onehot":
        x = np.zeros((n, d), np.float32)
        x[np.arange(n)[:, None], np.argsort(rng.random((n, d)), axis=1)[:, :10]] = 1.0
        return x
    raise ValueError(name)


def _oracle_acc_from_bmus(data, bmu, nx, ny, radius, cutoff, mt, grid, nbh, compact, cols=None):
    """num / den of the oracle's update for GIVEN BMUs (the node-sum
    regrouping num = sum_b h(b, .) S_b over occupied b), optionally on a
    column subset (the update is column-separable)."""
    k = nx * ny
    s, c = O.node_sums(data, bmu, k)
    if cols is not None:
        s = s[:, cols]
    occ = np.flatnonzero(c)
    h = O.h_rows(occ, radius, cutoff, nx, ny, mt, grid, nbh, compact)
    return h.T @ s[occ], h.T @ c[occ]


def _oracle_epoch(data, w, nx, ny, radius, cutoff, mt, grid, nbh, compact, sparse, regroup):
    """The oracle's BMUs and update accumulators for one epoch: its own
    search_accumulate, or (regroup, used for the 50,000-feature sparse
    shape, where the reference's per-chunk K x d accumulators would need
    ~4 GB each) its search plus the node-sum regrouping of the update."""
    kern = O.SPARSE if sparse else O.DENSE_BLOCKED
    if not regroup:
        ob, _, num, den = O.search_accumulate(data, w, nx, ny, radius, cutoff, mt, kern, workers=WORKERS,
                                              grid=grid, neighborhood=nbh, compact=compact)
        return ob, num, den
    ob, _, _, _ = O.search_accumulate(data, w, nx, ny, radius, cutoff, mt, kern, workers=WORKERS,
                                      with_accumulators=False)
    num, den = _oracle_acc_from_bmus(data, ob, nx, ny, radius, cutoff, mt, grid, nbh, compact)
    return ob, num, den


def _teacher_forced(data, x_dense, nx, ny, mt, grid, nbh, compact, w0, cfg, check_epochs, sparse=False,
                    cols=None):
    mtS = S.MapType(mt)
    if sparse:
        from paper_1305_1422_b200.sparse import SparseEngine
        eng = SparseEngine(S.SparseDataset(data.n_dimensions, data.row_offsets, data.col_indices, data.values),
                           nx, ny, mtS, S.GridType(grid))
    else:
        eng = S.SomEngine(S.DenseDataset(data), nx, ny, mtS, S.GridType(grid))
    regroup = cols is not None
    w = w0
    for e in range(cfg.n_epochs):
        st = S.epoch_schedules(cfg, e)
        args = (nx, ny, st.radius, cfg.influence_cutoff, mt, grid, nbh, compact)
        ob, num, den = _oracle_epoch(data, w, *args, sparse, regroup)
        if e in check_epochs:
            eng.set_codebook(w)
            eng.epoch(st.radius, st.scale, cfg.influence_cutoff, S.Neighborhood(nbh), compact)
            got = eng.codebook()
            bmu = eng.bmu[: eng.n].cpu().numpy().astype(np.int64)
            assert_bmus_tie_aware(bmu, ob, x_dense if x_dense is not None else data, w)
            # the update of the device's own BMUs (== the oracle's unless a
            # sub-1e-5 near tie flipped)
            mnum, mden = (num, den) if np.array_equal(bmu, ob) else _oracle_acc_from_bmus(data, bmu, *args)
            sel = slice(None) if cols is None else cols
            want = O.blend(w[:, sel], mnum[:, sel], mden, st.scale)
            assert rel_err(got[:, sel], want) <= 1e-6, (e, rel_err(got[:, sel], want))
        w = O.blend(w, num, den, st.scale)
    return w


def _cfg(nx, ny, mt, grid="rectangular", nbh="gaussian", compact=False, kernel=S.Kernel.DENSE_BLOCKED):
    return S.resolve_defaults(S.TrainConfig(n_epochs=10, n_columns=nx, n_rows=ny, map_type=S.MapType(mt),
                                            grid=S.GridType(grid), neighborhood=S.Neighborhood(nbh),
                                            compact_support=compact, kernel=kernel))


@pytest.mark.parametrize("fam", ["uniform", "nearconst", "dupcols", "blobs"])
def test_cfg2_shape_all_epochs(fam):
    """cfg2: 200x200 toroid, d = 1000 (1-pass fp16 screen), 2048 rows."""
    x = family(fam, 2048, 1000)
    cfg = _cfg(200, 200, "toroid")
    w0 = S.init_codebook(cfg, 1000).weights
    epochs = range(10) if fam == "uniform" else (0, 1, 3, 6, 9)
    _teacher_forced(x, x, 200, 200, O.TOROID, O.RECT, O.GAUSSIAN, False, w0, cfg, epochs)


@pytest.mark.parametrize("fam", ["uniform", "nearconst", "onehot"])
def test_cfg5_shape_all_epochs(fam):
    """cfg5: 500x500 planar, d = 128 (2-pass fp16 + fp8 split screen), 2048 rows."""
    x = family(fam, 2048, 128)
    cfg = _cfg(500, 500, "planar")
    w0 = S.init_codebook(cfg, 128).weights
    _teacher_forced(x, x, 500, 500, O.PLANAR, O.RECT, O.GAUSSIAN, False, w0, cfg, (0, 1, 2, 5, 9))


@pytest.mark.parametrize("fam", ["uniform", "blobs"])
def test_cfg4_shape_all_epochs(fam):
    """cfg4: 300x300 hexagonal toroid, bubble, compact support, d = 256 (1-pass by default), 2048 rows."""
    x = family(fam, 2048, 256)
    cfg = _cfg(300, 300, "toroid", "hexagonal", "bubble", True)
    w0 = S.init_codebook(cfg, 256).weights
    _teacher_forced(x, x, 300, 300, O.TOROID, O.HEX, O.BUBBLE, True, w0, cfg, (0, 1, 4, 9))


@pytest.mark.parametrize("init", ["default", "sampled"])
def test_cfg3_shape_sparse(init):
    """cfg3: 100x100 planar, d = 50,000 CSR at 0.5% density (250 nnz / row),
    512 rows; the reference default init and a data-sampled codebook (the
    default one collapses all rows onto few nodes).  BMUs over
    all 50,000 features; the update compared on 2,048 random columns."""
    sp = O.gen_random_sparse(512, 50_000, 0.005, 1001)
    cfg = _cfg(100, 100, "planar", kernel=S.Kernel.SPARSE)
    if init == "default":
        w0 = S.init_codebook(cfg, 50_000).weights
    else:
        rng = np.random.default_rng(3)
        dense = np.zeros((10_000, 50_000), np.float32)
        rows = rng.integers(0, 512, 10_000)
        for j, r in enumerate(rows):
            c, v = sp.row(int(r))
            dense[j, c] = v
        w0 = dense
    cols = np.sort(np.random.default_rng(4).choice(50_000, 2048, replace=False))
    _teacher_forced(sp, None, 100, 100, O.PLANAR, O.RECT, O.GAUSSIAN, False, w0, cfg, (0, 1, 5, 9),
                    sparse=True, cols=cols)


def test_auto_screen_switches_to_split_on_structured_data():
    """Auto screen for 128 < d <= 256 starts 1-pass; near-constant rows keep
    hundreds of nodes in its window, rows truncate and are repaired by full
    scans, and the engine switches to the fp16 + fp8 split screen
    (engine.SomEngine._switch_to_split).  Every epoch's BMUs equal the exact
    fp64 argmin (first-minimum ties), before and after the switch."""
    import torch
    x = family("nearconst", 4096, 256)
    eng = S.SomEngine(S.DenseDataset(x), 300, 300, S.MapType.TOROID, S.GridType.HEXAGONAL)
    assert eng.passes == 1 and eng._adaptive
    eng.init_codebook_device(1)
    X = torch.from_numpy(x).cuda().double()
    for e in range(4):
        eng.search()
        W = eng.W[: eng.K].double()
        d2 = torch.clamp((-2.0 * (X @ W.T) + eng.x2[: eng.n, None]) + eng.w2[None, : eng.K], min=0.0)
        want = torch.argmin(d2, dim=1)
        got = eng.bmu[: eng.n].long()
        bad = torch.nonzero(got != want).flatten()
        if len(bad):   # only fp64 summation-order ties
            gap = (d2[bad, got[bad]] - d2[bad, want[bad]]).abs() / (eng.x2[bad] + eng.w2.max())
            assert float(gap.max()) <= 1e-12, (e, len(bad))
        eng.qe_sum()
        eng.node_sums()
        eng.update(150.0 * (1 - e / 4) + 1, 1.0 - 0.2 * e, 1e-3, S.Neighborhood.BUBBLE, True)
    assert eng.passes == 2 and getattr(eng, "switched_to_split", False)
