"""Per-node |delta_j| (codebook row minus codebook mean) vs its maximum, over
all nodes and over the screen's candidate nodes (cfg2, epochs 2-5)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200 import _lib  # noqa: E402
from paper_1305_1422_b200.engine import SomEngine  # noqa: E402

n, d, nx, ny = 1_000_000, 1000, 200, 200
g = torch.Generator(device="cuda")
g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device="cuda")
eng = SomEngine(X, nx, ny, S.MapType.TOROID)
eng.set_codebook(S.init_codebook(S.TrainConfig(n_columns=nx, n_rows=ny, seed=1), d).weights)
for e in range(6):
    r, sc = bench.schedule_for("cfg2", e)
    eng.search()
    W = eng.W[: eng.K].double()
    dn = (W - W.mean(0)).norm(dim=1)
    mx = float(dn.max())
    cand = eng.ws[: n * _lib.CAND_CAP * 4].view(torch.int32).view(n, _lib.CAND_CAP)[:50000]
    cnt = eng.ws[((n * _lib.CAND_CAP * 4 + 255) // 256) * 256:][: 4 * n].view(torch.int32)[:50000]
    c0 = (cnt & 255).long()
    m = torch.arange(_lib.CAND_CAP, device="cuda")[None, :] < c0[:, None]
    cn = dn[cand.long().clamp(0, eng.K - 1)][m]
    q = torch.tensor([0.1, 0.5, 0.9], dtype=torch.float64, device="cuda")
    print(f"epoch {e}: max|delta| {mx:.4g}; all nodes |d|/max quantiles {torch.quantile(dn / mx, q).tolist()}; "
          f"candidates {torch.quantile(cn / mx, q).tolist() if cn.numel() else []}", flush=True)
    eng.qe_sum(); eng.node_sums(); eng.update(r, sc, 1e-3)
