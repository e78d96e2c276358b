"""How much do the candidate lists of consecutive BMU-sorted rows overlap?
(sum of list sizes / union size per group of G rows; local lists only)."""
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
    if e >= 2:
        cc = eng.candidate_counts()[:n].cpu().numpy()
        cand = eng.ws[: n * _lib.CAND_CAP * 4].view(torch.int32).view(n, _lib.CAND_CAP).cpu().numpy()
        cnt = eng.ws[((n * _lib.CAND_CAP * 4 + 255) // 256) * 256:][: 4 * n].view(torch.int32).cpu().numpy()
        c0, c1 = cnt & 255, (cnt >> 8) & 255
        order = eng.row_order[:n].cpu().numpy()
        for G in (8, 16, 32, 64):
            tot, uni = 0, 0
            for gi in range(0, 200000, G):
                rows = order[gi:gi + G]
                s = set()
                for rr in rows:
                    l = list(cand[rr, :c0[rr]]) + list(cand[rr, 32:32 + c1[rr]])
                    tot += len(l)
                    s.update(l)
                uni += len(s)
            print(f"epoch {e} G={G}: mean list {tot / 200000:.1f}, sharing factor {tot / max(uni, 1):.2f}", flush=True)
    eng.qe_sum(); eng.node_sums(); eng.update(r, sc, 1e-3)
