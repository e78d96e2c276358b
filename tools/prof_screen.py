"""Profile helper: cfg-shaped BMU searches (screen + re-rank) on cuda:0 after
`warm` training epochs of the reference schedule (epochs 2-7 of cfg2 are the
candidate-heavy regime).
   python tools/prof_screen.py [rows] [d] [nx] [ny] [reps] [warm_epochs]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200.engine import SomEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 148 * 128 * 4
d = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
nx = int(sys.argv[3]) if len(sys.argv) > 3 else 200
ny = int(sys.argv[4]) if len(sys.argv) > 4 else 200
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
warm = int(sys.argv[6]) if len(sys.argv) > 6 else 1
g = torch.Generator(device="cuda")
g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device="cuda")
eng = SomEngine(X, nx, ny, S.MapType.TOROID)
eng.set_codebook(S.init_codebook(S.TrainConfig(n_columns=nx, n_rows=ny), d).weights)
r0 = max(min(nx, ny) / 2, 1.0)
for e in range(warm):     # reference linear schedule, 10 epochs
    f = e / 9
    eng.epoch(r0 + (1 - r0) * f, 1 + (0.01 - 1) * f, 1e-3)
for _ in range(reps):
    eng.search()
torch.cuda.synchronize()
tot = eng.candidate_counts()[:n].float()
print(f"candidates/row mean {tot.mean():.2f} p50 {tot.median():.0f} max {tot.max():.0f}; "
      f"truncated rows {((eng.flags[:n] & 0xFFFF) != 0).float().mean():.3f}")
