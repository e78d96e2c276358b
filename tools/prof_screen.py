"""Profile helper: one cfg-shaped BMU search (screen + re-rank) on cuda:0.
   python tools/prof_screen.py [rows] [d] [nx] [ny] [reps]"""
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
g = torch.Generator(device="cuda")
g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device="cuda")
eng = SomEngine(X, nx, ny, S.MapType.TOROID)
eng.set_codebook(S.init_codebook(S.TrainConfig(n_columns=nx, n_rows=ny), d).weights)
eng.epoch(nx / 2, 1.0, 1e-3)          # collapse the codebook like a real run
for _ in range(reps):
    eng.search()
torch.cuda.synchronize()
cc = eng.ws[: 0].new_empty(0)
off = ((n * 32 * 4 + 255) // 256) * 256
cnt = eng.ws[off: off + 4 * n].view(torch.int32).cpu()
c0, c1 = cnt & 255, (cnt >> 8) & 255
tot = (c0 + c1).float()
print(f"candidates/row mean {tot.mean():.2f} p50 {tot.median():.0f} max {tot.max():.0f}; "
      f"truncated rows {((eng.flags[:n].cpu() & 0xFFFF) != 0).float().mean():.3f}")
