"""Candidate counts of the screen with and without the previous-BMU threshold
seed (engine option seed_prev), on a 20k-row cfg2-shaped run."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_1422_b200 as S
from paper_1305_1422_b200.engine import SomEngine
n, d, nx, ny = 20000, 1000, 200, 200
g = torch.Generator(device="cuda"); g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device="cuda")
eng = SomEngine(X, nx, ny, S.MapType.TOROID)
eng.set_codebook(S.init_codebook(S.TrainConfig(n_columns=nx, n_rows=ny), d).weights)
def stats(tag):
    cc = eng.candidate_counts().cpu()
    print(tag, "cand mean", cc.float().mean().item(), "zero rows", (cc == 0).sum().item(),
          "bmu", eng.bmu[:5].tolist())
eng.search(); stats("first")
eng.search(); stats("second(seeded)")
eng.opt.seed_prev = False
eng.search(); stats("third(unseeded)")
eng.opt.seed_prev = True
eng.epoch(100, 1.0, 1e-3); stats("epoch")
eng.search(); stats("after-epoch seeded")
eng.search(); stats("again seeded")
ws = eng.ws
off = ((n * 32 * 4 + 255) // 256) * 256 + ((n * 4 + 255) // 256) * 256
thr0 = ws[off: off + 4 * n].view(torch.float32)
print("thr0[:5]", thr0[:5].tolist())
r = eng.debug_screen_values()
b = eng.bmu[:5].long()
print("screened at bmu", [r[i, b[i]].item() for i in range(5)], "row min", r[:5].min(1).values.tolist())
