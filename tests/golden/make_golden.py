"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (needs /root/reference, which does not exist on
the GPU box):  python tests/golden/make_golden.py
Outputs small .npz fixtures next to this script; the parity tests read only
those files.  Inputs are stored alongside outputs so nothing is regenerated.
"""
import hashlib
import os
import sys
from dataclasses import replace

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from somkit import (CodeBook, Cooling, DenseDataset, Kernel, MapType,  # noqa: E402
                    SparseDataset, TrainConfig, blend, compute_umatrix,
                    gen_random_dense, gen_random_sparse, search_accumulate,
                    train)

HERE = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def kernel_cases():
    """search_accumulate + blend on random inputs (kernels.py:365-450)."""
    rng = np.random.default_rng(20240901)
    out = {}
    cases = [  # n, d, nx, ny, toroid, radius, cutoff, kernel, scale
        (300, 7, 6, 5, False, 2.5, 1e-3, 1, 0.7),
        (300, 7, 6, 5, True, 2.5, 1e-3, 1, 0.7),
        (513, 16, 9, 7, True, 4.0, 0.0, 1, 1.0),
        (257, 5, 12, 3, False, 0.4, 1e-3, 1, 0.3),
        (200, 9, 8, 8, True, 1.7, 1e-3, 0, 0.5),
        (180, 12, 7, 6, False, 3.0, 1e-3, 2, 0.9),
        (180, 12, 7, 6, True, 3.0, 0.0, 2, 0.9),
        (1000, 6, 70, 50, True, 20.0, 1e-3, 1, 1.0),   # K=3500 > 3000: direct h rows
        (700, 20, 40, 40, False, 6.0, 1e-3, 1, 0.25),
    ]
    for ci, (n, d, nx, ny, tor, radius, cutoff, kern, scale) in enumerate(cases):
        mt = MapType.TOROID if tor else MapType.PLANAR
        w = rng.random((nx * ny, d), dtype=np.float32)
        cb = CodeBook(nx, ny, d, w)
        if kern == 2:
            sp = gen_random_sparse(n, d, 0.35, seed=100 + ci)
            data = sp
            out[f"c{ci}_offsets"] = sp.row_offsets
            out[f"c{ci}_cols"] = sp.col_indices
            out[f"c{ci}_vals"] = sp.values
        else:
            x = rng.random((n, d), dtype=np.float32)
            data = DenseDataset(x)
            out[f"c{ci}_x"] = x
        bmu, qe, acc = search_accumulate(data, cb, radius, cutoff, mt,
                                         Kernel(kern), workers=4)
        out[f"c{ci}_params"] = np.array([n, d, nx, ny, int(tor), radius, cutoff,
                                         kern, scale], dtype=np.float64)
        out[f"c{ci}_w"] = w
        out[f"c{ci}_bmu"] = bmu
        out[f"c{ci}_qe"] = np.array(qe)
        out[f"c{ci}_num"] = acc.numerators
        out[f"c{ci}_den"] = acc.denominators
        out[f"c{ci}_blend"] = blend(w, acc, scale)
    out["ncases"] = np.array(len(cases))
    save("kernels.npz", **out)


def umatrix_cases():
    rng = np.random.default_rng(31)
    out = {}
    shapes = [(1, 1, 3), (2, 1, 2), (3, 3, 2), (5, 4, 7), (10, 10, 3), (1, 6, 4),
              (7, 2, 1), (2, 2, 5), (13, 9, 17)]
    i = 0
    for nx, ny, d in shapes:
        for mt in (MapType.PLANAR, MapType.TOROID):
            w = rng.random((nx * ny, d), dtype=np.float32)
            u = compute_umatrix(CodeBook(nx, ny, d, w), mt).heights
            out[f"u{i}_shape"] = np.array([nx, ny, d, int(mt is MapType.TOROID)])
            out[f"u{i}_w"] = w
            out[f"u{i}_u"] = u
            i += 1
    out["ncases"] = np.array(i)
    save("umatrix.npz", **out)


def train_cases():
    """Full train() runs: codebook, BMU table, U-matrix, per-epoch qe."""
    out = {}
    runs = []
    # small configs spanning map types / coolings / explicit schedules
    runs.append(("t0", gen_random_dense(60, 4, seed=0).values,
                 TrainConfig(n_epochs=3, n_columns=6, n_rows=5, kernel=Kernel.DENSE_BLOCKED)))
    runs.append(("t1", gen_random_dense(400, 9, seed=5).values,
                 TrainConfig(n_epochs=5, n_columns=8, n_rows=7, map_type=MapType.TOROID,
                             kernel=Kernel.DENSE_BLOCKED, radius0=4.0, radiusN=1.0,
                             radius_cooling=Cooling.EXPONENTIAL, scale0=0.8,
                             scaleN=0.05, scale_cooling=Cooling.EXPONENTIAL, seed=7)))
    # clustered, well-conditioned data (test_acceptance.py:304-327 style)
    rng = np.random.default_rng(17)
    centers = np.full((4, 10), 8.0)
    for i in range(4):
        centers[i, i] += 3.0
    pts = np.concatenate([c + 0.15 * rng.standard_normal((100, 10))
                          for c in centers]).astype(np.float32)
    runs.append(("t2", pts, TrainConfig(n_epochs=10, n_columns=10, n_rows=10, seed=1,
                                        kernel=Kernel.DENSE_BLOCKED)))
    # cfg1 of BASELINE.json: 50x40 planar, 10k x 100 uniform, 10 epochs,
    # distinct data (1001) and codebook (1) seeds
    runs.append(("cfg1", gen_random_dense(10000, 100, seed=1001).values,
                 TrainConfig(n_epochs=10, n_columns=50, n_rows=40, seed=1,
                             kernel=Kernel.DENSE_BLOCKED)))
    # cfg1-shaped toroid on clustered data (16 gaussian blobs)
    rng = np.random.default_rng(23)
    cen = rng.random((16, 32))
    blobs = np.concatenate([c + 0.03 * rng.standard_normal((250, 32)) for c in cen])
    runs.append(("blobs", blobs.astype(np.float32),
                 TrainConfig(n_epochs=8, n_columns=30, n_rows=20, seed=3,
                             map_type=MapType.TOROID, kernel=Kernel.DENSE_BLOCKED)))
    for name, x, cfg in runs:
        qes = []
        cb, bmus, u = train(DenseDataset(x), cfg, workers=8,
                            progress=lambda s, q: qes.append(q))
        if x.size > 200000:  # regenerated from its seed by the tests; keep a digest
            out[f"{name}_xsha"] = np.array(hashlib.sha256(x.tobytes()).hexdigest())
        else:
            out[f"{name}_x"] = x
        out[f"{name}_cfg"] = np.array([cfg.n_epochs, cfg.n_columns, cfg.n_rows,
                                       int(cfg.map_type is MapType.TOROID),
                                       cfg.radius0, cfg.radiusN,
                                       int(cfg.radius_cooling is Cooling.EXPONENTIAL),
                                       cfg.scale0, cfg.scaleN,
                                       int(cfg.scale_cooling is Cooling.EXPONENTIAL),
                                       cfg.seed, cfg.influence_cutoff], dtype=np.float64)
        out[f"{name}_w"] = cb.weights
        out[f"{name}_bmus"] = bmus
        out[f"{name}_u"] = u.heights
        out[f"{name}_qe"] = np.array(qes)
    out["names"] = np.array([r[0] for r in runs])
    save("train.npz", **out)


def sparse_train_cases():
    out = {}
    sp = gen_random_sparse(300, 40, 0.3, seed=11)
    # data-sampled initial codebook keeps the sparse map non-degenerate
    dense = sp.densify().values
    w0 = dense[np.random.default_rng(2).choice(300, 36, replace=False)].copy()
    cfg = TrainConfig(n_epochs=4, n_columns=6, n_rows=6, kernel=Kernel.SPARSE,
                      map_type=MapType.TOROID)
    qes = []
    cb, bmus, u = train(sp, cfg, initial_codebook=CodeBook(6, 6, 40, w0),
                        progress=lambda s, q: qes.append(q))
    out.update(s0_offsets=sp.row_offsets, s0_cols=sp.col_indices, s0_vals=sp.values,
               s0_w0=w0, s0_w=cb.weights, s0_bmus=bmus, s0_u=u.heights,
               s0_qe=np.array(qes), s0_cfg=np.array([4, 6, 6, 1]))
    # reference defaults (uniform init): degenerate map -- exact ties
    sp2 = gen_random_sparse(200, 500, 0.01, seed=12)
    cfg2 = TrainConfig(n_epochs=3, n_columns=5, n_rows=4, kernel=Kernel.SPARSE)
    qes = []
    cb, bmus, u = train(sp2, cfg2, progress=lambda s, q: qes.append(q))
    out.update(s1_offsets=sp2.row_offsets, s1_cols=sp2.col_indices, s1_vals=sp2.values,
               s1_w=cb.weights, s1_bmus=bmus, s1_u=u.heights, s1_qe=np.array(qes),
               s1_cfg=np.array([3, 5, 4, 0]))
    save("sparse_train.npz", **out)


if __name__ == "__main__":
    kernel_cases()
    umatrix_cases()
    sparse_train_cases()
    train_cases()
