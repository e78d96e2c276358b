"""At a bench-like cfg2 state (1M rows, epochs 0..E-1 trained), compare the
tcgen05-screened BMUs with an exact fp64 scan on a row sample."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200.engine import EngineOptions, SomEngine  # noqa: E402

n, d, nx, ny, E, m = 1_000_000, 1000, 200, 200, int(sys.argv[1]) if len(sys.argv) > 1 else 6, 50_000
kappa = float(sys.argv[2]) if len(sys.argv) > 2 else 16.0
g = torch.Generator(device="cuda")
g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device="cuda")
cfg = S.resolve_defaults(S.TrainConfig(n_epochs=10, n_columns=nx, n_rows=ny, map_type=S.MapType.TOROID))
eng = SomEngine(X, nx, ny, S.MapType.TOROID, options=EngineOptions(window_kappa=kappa))
eng.set_codebook(S.init_codebook(cfg, d).weights)
ref = SomEngine(X[:m], nx, ny, S.MapType.TOROID, options=EngineOptions(screen="exact"))
for e in range(E):
    st = S.epoch_schedules(cfg, e)
    eng.search()
    cc = eng.candidate_counts()[:n].float().cpu().numpy()
    fl = eng.flags[:n].cpu().numpy()
    tr = (((fl & 0xFF) | ((fl >> 8) & 0xFF) | ((fl >> 16) & 0xFF) | ((fl >> 24) & 0xFF)) & 1).astype(bool)
    bm = eng.bmu[:m].cpu().numpy().copy()
    ref.set_codebook(eng.codebook())
    ref.search()
    rb = ref.bmu[:m].cpu().numpy()
    bad = np.flatnonzero(bm != rb)
    gaps = []
    if len(bad):
        W = torch.from_numpy(eng.codebook()).cuda().double()
        xs = X[:m][torch.from_numpy(bad).cuda()].double()
        d2 = (xs * xs).sum(1, keepdim=True) + (W * W).sum(1)[None] - 2 * xs @ W.T
        top2 = torch.topk(d2, 2, dim=1, largest=False).values
        gaps = ((top2[:, 1] - top2[:, 0]) / top2[:, 0]).cpu().numpy()
    print(f"ep{e} r={st.radius:.1f}: cand mean {cc.mean():.1f} p50 {np.median(cc):.0f} p99 {np.percentile(cc, 99):.0f} "
          f"max {cc.max():.0f}; truncated {tr.mean():.3f}; BMU mismatches {len(bad)}/{m}"
          + (f" max rel gap {np.max(gaps):.2e}" if len(bad) else ""), flush=True)
    eng.qe_sum(); eng.node_sums(); eng.reduce(); eng.update(st.radius, st.scale, 1e-3)
