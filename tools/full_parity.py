"""Full-scale parity of the screened search: 10 epochs of a bench config with
the tcgen05 screen vs the exact fp64 scan (screen='exact'), same data, same
initial codebook.  Reports codebook / U-matrix max relative error and the
final BMU mismatches with their fp64 top-2 gaps.
   python tools/full_parity.py [cfg] [rows] [epochs] [family]
family (dense configs): uniform (default) or a tools/calib_window.py family."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200.engine import EngineOptions  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n0, d, nx, ny, mt, grid, nbh, compact, desc = bench.CONFIGS[cfg_name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else n0
E = int(sys.argv[3]) if len(sys.argv) > 3 else 10
sparse = cfg_name == "cfg3"
if sparse:   # CSR rows of the bench generator; the screened search is the sparse fp16 screen
    rp, cl, vl = bench.sparse_rows_device(n, d, bench.SPARSE_NNZ, 1001, torch.device("cuda", 0))
    data = S.SparseDataset(d, rp.cpu().numpy(), cl.cpu().numpy(), vl.cpu().numpy())
    X = None
else:
    from calib_window import family_data
    fam = sys.argv[4] if len(sys.argv) > 4 else "uniform"
    X = family_data(fam, n, d, torch.device("cuda", 0))
    data = S.DenseDataset(X)
cfg = S.TrainConfig(n_epochs=E, n_columns=nx, n_rows=ny, map_type=S.MapType(mt), grid=S.GridType(grid),
                    neighborhood=S.Neighborhood(nbh), compact_support=compact,
                    kernel=S.Kernel.SPARSE if sparse else S.Kernel.DENSE_BLOCKED, seed=1)
out = {}
for screen in ("tensor", "exact"):
    t0 = time.time()
    cb, bm, u = S.train(data, cfg, options=EngineOptions(screen=screen))
    out[screen] = (cb.weights, bm, u.heights, time.time() - t0)
    print(screen, f"{out[screen][3]:.1f} s", flush=True)
wt, bt, ut, _ = out["tensor"]
we, be, ue, _ = out["exact"]
rel = lambda a, b: float(np.max(np.abs(a.astype(np.float64) - b) / np.maximum(np.abs(b), 1e-12)))
fb = bt[:, 0].astype(np.int64) * nx + bt[:, 1]
eb = be[:, 0].astype(np.int64) * nx + be[:, 1]
bad = np.flatnonzero(fb != eb)
gap = None
if len(bad) and not sparse:
    W = torch.from_numpy(we).cuda().double()
    xs = X[torch.from_numpy(bad[:20000]).cuda()].double()
    d2 = (xs * xs).sum(1, keepdim=True) + (W * W).sum(1)[None] - 2 * xs @ W.T
    t2 = torch.topk(d2, 2, dim=1, largest=False).values
    gap = float(((t2[:, 1] - t2[:, 0]) / t2[:, 0]).max())
res = {"config": desc, "family": "sparse" if sparse else fam, "rows": n, "epochs": E,
       "seconds_tensor": out["tensor"][3], "seconds_exact": out["exact"][3], "codebook_max_rel": rel(wt, we),
       "codebook_bit_identical_frac": float(np.mean(wt == we)), "umatrix_max_rel": rel(ut, ue),
       "bmu_mismatch": int(len(bad)), "bmu_mismatch_max_gap": gap}
print(json.dumps(res))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open(f"gpurun_out/full_parity_{cfg_name}_{res['family']}_{n}.json", "w"))
