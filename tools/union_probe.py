"""Probe: how many distinct candidate nodes do R consecutive rows (previous-BMU
order) share after the screen?  Sizes a tiled re-rank.
   python tools/union_probe.py [rows] [d] [nx] [ny] [warm_epochs]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200 import _lib  # noqa: E402
from paper_1305_1422_b200.engine import SomEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
nx = int(sys.argv[3]) if len(sys.argv) > 3 else 200
ny = int(sys.argv[4]) if len(sys.argv) > 4 else 200
warm = int(sys.argv[5]) if len(sys.argv) > 5 else 4
g = torch.Generator(device="cuda")
g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device="cuda")
eng = SomEngine(X, nx, ny, S.MapType.TOROID)
eng.set_codebook(S.init_codebook(S.TrainConfig(n_columns=nx, n_rows=ny), d).weights)
r0 = max(min(nx, ny) / 2, 1.0)
for e in range(warm + 6):
    if e >= warm:
        eng.search()
        torch.cuda.synchronize()
        cap = _lib.CAND_CAP
        cand = eng.ws[: n * cap * 4].view(torch.int32).view(n, cap)
        off = ((n * cap * 4 + 255) // 256) * 256
        cc = eng.ws[off: off + 4 * n].view(torch.int32)
        a = lambda b: (b + 255) // 256 * 256
        coff = a(n * cap * 4) + 2 * a(n * 4)
        ng = int(eng.ws[coff + 12: coff + 16].view(torch.int32).item()) or 2
        gs = cap // ng
        slot = torch.arange(cap, device="cuda")
        grp = slot // gs
        cnts = torch.stack([(cc >> (8 * k)) & 255 for k in range(ng)], 1)         # n x ng
        valid = (slot % gs)[None, :] < cnts.gather(1, grp[None, :].expand(n, -1))
        c = torch.where(valid, cand, torch.full_like(cand, 1 << 30))
        order = eng.row_order[:n].long() if eng.has_order else torch.arange(n, device="cuda")
        c = c[order]
        out = [f"epoch {e}: cand/row {valid.sum(1).float().mean():.1f}"]
        for R in (8, 16, 32, 64):
            m = (n // R) * R
            t = c[:m].view(m // R, R * cap).sort(1).values
            distinct = ((t[:, 1:] != t[:, :-1]) & (t[:, 1:] < (1 << 30))).sum(1) + (t[:, 0] < (1 << 30)).long()
            pairs = valid[order][:m].view(m // R, -1).sum(1).float()
            out.append(f"R={R}: union mean {distinct.float().mean():.1f} p99 {distinct.float().quantile(0.99):.0f} "
                       f"max {distinct.max()}  (pairs {pairs.mean():.0f}, reuse {pairs.mean() / distinct.float().mean():.1f}x)")
        print("; ".join(out), flush=True)
    f = e / 9
    eng.epoch(r0 + (1 - r0) * f, 1 + (0.01 - 1) * f, 1e-3)
