"""Calibrate the screening window on hardware: tcgen05 screened values vs
exact fp64 distances on real (collapsing) codebooks.
   python tools/calib_screen.py [rows] [d] [nx] [ny] [epochs] [toroid]"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200.engine import SomEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
nx = int(sys.argv[3]) if len(sys.argv) > 3 else 200
ny = int(sys.argv[4]) if len(sys.argv) > 4 else 200
E = int(sys.argv[5]) if len(sys.argv) > 5 else 6
tor = (sys.argv[6] != "0") if len(sys.argv) > 6 else True
passes = int(sys.argv[7]) if len(sys.argv) > 7 else 0
g = torch.Generator(device="cuda")
g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device="cuda")
mt = S.MapType.TOROID if tor else S.MapType.PLANAR
from paper_1305_1422_b200.engine import EngineOptions  # noqa: E402
eng = SomEngine(X, nx, ny, mt, options=EngineOptions(screen_passes=passes))
print("passes", eng.passes, "window kappa", eng.window_coef * math.sqrt(d) / 2.0 ** -11)
cfg = S.resolve_defaults(S.TrainConfig(n_epochs=10, n_columns=nx, n_rows=ny, map_type=mt))
eng.set_codebook(S.init_codebook(cfg, d).weights)
x64 = X[:128].double()
unit = 2.0 ** -11
for e in range(E):
    st = S.epoch_schedules(cfg, e)
    r = eng.debug_screen_values().double()                       # 128 x K
    W = eng.W[: eng.K].double()
    d2 = (x64 * x64).sum(1, keepdim=True) + (W * W).sum(1)[None] - 2 * x64 @ W.T
    diff = r - d2
    diff -= diff.median(dim=1, keepdim=True).values
    xn = (x64 - eng.nu.double()).norm(dim=1)
    mu = W.mean(0)
    nmax = (W - mu).norm(dim=1).max()
    scale = unit * xn[:, None] * nmax / math.sqrt(d)
    ratio = (diff.abs() / scale).max().item()
    ex = d2.argmin(1)
    order = r.argsort(dim=1, stable=True)
    rank = (order == ex[:, None]).float().argmax(1)
    rmin = r.min(1, keepdim=True).values
    out = [f"ep{e} r={st.radius:.1f}: max|err|/(u16 |x'| nmax/sqrt(D)) = {ratio:.2f}; "
           f"exact-argmin screen rank max {int(rank.max())}"]
    for kappa in ((0.05, 0.1, 0.25, 0.5, 1.0) if eng.passes in (2, 3) else (4, 8, 12, 16, 24)):
        w = kappa * scale[:, :1]
        cnt = (r <= rmin + w).sum(1).float()
        out.append(f"k{kappa}: mean {cnt.mean():.1f} max {int(cnt.max())}")
    print("; ".join(out), flush=True)
    eng.search()
    cc = eng.candidate_counts()[:n].float()
    print(f"   full-N candidates/row mean {cc.mean():.2f} max {int(cc.max())}, "
          f"truncated {((eng.flags[:n] & 0xFFFF) != 0).float().mean():.3f}", flush=True)
    eng.epoch(st.radius, st.scale, 1e-3)
