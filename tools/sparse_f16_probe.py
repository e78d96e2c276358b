"""Round-2 sizing probe: candidate counts a sparse screen on an fp16 copy of
the transposed codebook would produce with a rigorous per-pair bound
b_ij = 2^-11 sum_k |x_k| |delta_jk| (+ the fp32 accumulation term), against
the current fp32 screen's window, at trained cfg3 states (exact distances,
512 sample rows).   python tools/sparse_f16_probe.py [rows] [warm]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200.sparse import SparseEngine  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 6
n, d, nx, ny, mt, grid, nbh, compact, _ = bench.CONFIGS["cfg3"]
dev = torch.device("cuda", 0)
rp, cl, vl = bench.sparse_rows_device(rows, d, bench.SPARSE_NNZ, 1001, dev)
data = S.SparseDataset(d, rp.cpu().numpy(), cl.cpu().numpy(), vl.cpu().numpy())
eng = SparseEngine(data, nx, ny, S.MapType(mt), S.GridType(grid), device=dev)
eng.set_codebook(S.init_codebook(S.TrainConfig(n_columns=nx, n_rows=ny, seed=1), d).weights)
m = 512
Xs = torch.zeros((m, d), dtype=torch.float64, device=dev)
for i in range(m):
    a, b = int(rp[i]), int(rp[i + 1])
    Xs[i, cl[a:b].long()] = vl[a:b].double()
for e in range(warm + 1):
    if e >= 2:
        W = eng.W[: eng.K].double()
        mu = W.mean(0)
        D = W - mu
        r = (D * D).sum(1)[None] + 2 * (mu[None] * D).sum(1) - 2 * Xs @ D.T - 0  # r_ij up to a row constant
        rmin = r.min(1, keepdim=True).values
        xn = Xs.norm(dim=1, keepdim=True)
        dmax = D.norm(dim=1).max()
        nnz = (Xs != 0).sum(1, keepdim=True).double()
        w32 = 2 * (nnz + 2) * 2.0 ** -24 * xn * dmax             # current rigorous fp32 window
        c32 = (r <= rmin + w32).sum(1).double()
        b16 = 2 * 2.0 ** -11 * (Xs.abs() @ D.abs().T) + w32      # per-pair fp16 bound (+ fp32 term)
        c16 = (r - b16 <= (r + b16).min(1, keepdim=True).values).sum(1).double()
        print(f"epoch {e}: fp32 window cand mean {c32.mean():.2f} max {int(c32.max())}; "
              f"fp16 per-pair bound cand mean {c16.mean():.2f} p99 {c16.quantile(0.99):.0f} max {int(c16.max())}",
              flush=True)
    r0, sc = bench.schedule_for("cfg3", e)
    eng.epoch(r0, sc, 1e-3, S.Neighborhood(nbh), compact)
