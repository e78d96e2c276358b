"""Time the screen kernel alone at a cfg shape (CUDA events, after warm-up).
   python tools/screen_time.py rows d nx ny [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200.engine import SomEngine  # noqa: E402

n, d, nx, ny = (int(v) for v in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
g = torch.Generator(device="cuda")
g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device="cuda")
eng = SomEngine(X, nx, ny, S.MapType.TOROID)
eng.set_codebook(S.init_codebook(S.TrainConfig(n_columns=nx, n_rows=ny), d).weights)
eng.epoch(max(min(nx, ny) / 2, 1), 1.0, 1e-3)
eng.search()
eng.timing = {}
for _ in range(reps):
    eng.search()
torch.cuda.synchronize()
ms = [a.elapsed_time(b) for a, b in eng.timing["screen"]]
cc = eng.candidate_counts().cpu()
print("candidates/row mean", cc.float().mean().item(), "zero-candidate rows", (cc == 0).sum().item(),
      "rerank ms", [round(a.elapsed_time(b), 2) for a, b in eng.timing["rerank"]])
fl = 2.0 * n * nx * ny * d
print(f"screen {min(ms):.2f} ms  ({fl / (min(ms) / 1e3) / 1e12:.0f} TFLOP/s algorithmic)  "
      f"rerank {min(a.elapsed_time(b) for a, b in eng.timing['rerank']):.2f} ms")
