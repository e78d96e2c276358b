"""Probe: how many 32-node chunks of a row could an epilogue chunk bound
(min_j(r_j - c_j) + min_j c_j) rule out, vs the chunks that truly hold a
window member?  (~1% pass at cfg2 / cfg5; the bound was tried in the
screen epilogue and measured neutral.)
   python tools/prune_probe.py [cfg] [rows] [warm]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200.engine import SomEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 200000
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 4
n, d, nx, ny, mt, grid, nbh, compact, _ = bench.CONFIGS[cfg]
g = torch.Generator(device="cuda")
g.manual_seed(1001)
X = torch.rand((rows, d), generator=g, device="cuda")
eng = SomEngine(X, nx, ny, S.MapType(mt), S.GridType(grid))
eng.init_codebook_device(1)
for e in range(warm + 1):
    if e >= warm - 1:
        eng.prepare()
        r = eng.debug_screen_values().double()[:, : eng.K]      # 128 x K screened r
        c = eng.c[: eng.K].double()
        K32 = (eng.K // 32) * 32
        rr, cc = r[:, :K32].view(128, -1, 32), c[:K32].view(-1, 32)
        bound = (rr - cc).min(2).values + cc.min(1).values        # epilogue chunk bound
        cmin_true = rr.min(2).values
        win = eng.window_coef * eng.xnorm[:128].double() * float(eng.scal[1])
        thr = r.min(1).values + win
        passing = (bound <= thr[:, None]).float().mean().item()
        needed = (cmin_true <= thr[:, None]).float().mean().item()
        print(f"{cfg} epoch {e}: chunks passing the bound {passing:.4f}, holding a window member {needed:.5f}", flush=True)
    r0, sc = bench.schedule_for(cfg, e)
    eng.epoch(r0, sc, 1e-3, S.Neighborhood(nbh), compact)
