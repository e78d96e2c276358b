"""Feasibility probe for an fp16 + 2 x fp8 split screen (hi.hi in fp16, the
two cross terms hi.lo + lo.hi in e4m3 at twice the tensor rate): emulate its
arithmetic in torch on 128 rows against the codebook of a cfg-shaped run
after each epoch, and report the screen error (in the 1-pass window units
2^-11 |x'| max|delta| / sqrt(d)) and the window candidate counts, next to
the 3-pass fp16 split.
   python tools/f8_probe.py [cfg5|cfg4] [epochs]"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200.engine import SomEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
E = int(sys.argv[2]) if len(sys.argv) > 2 else 6
n, d, nx, ny, mt, grid, nbh, compact, _ = bench.CONFIGS[cfg]
n = 65536
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device=dev)
eng = SomEngine(X, nx, ny, S.MapType(mt), S.GridType(grid), device=dev)
eng.init_codebook_device(1)
f8 = torch.float8_e4m3fn


def split16(v):
    h = v.half()
    return h.double(), (v - h.double()).half().double()


def e4(v):
    return v.to(f8).double()


for e in range(E):
    r_, sc = bench.schedule_for(cfg, e)
    W = eng.W[: eng.K].double()
    x = X[:128].double()
    nu = X.double().mean(0)
    mu = W.mean(0)
    xc, dc = x - nu, W - mu
    xexp = 13 - math.frexp(float(xc.abs().max()))[1]
    sexp = 13 - math.frexp(float(dc.abs().max()))[1]
    xs, ds = xc * 2.0 ** xexp, dc * 2.0 ** sexp
    xh, xl = split16(xs)
    wh, wl = split16(ds)
    m = 2.0 ** -(xexp + sexp)
    exact = (xc @ dc.T)
    p3 = (xh @ wh.T + xh @ wl.T + xl @ wh.T) * m
    p2 = (xh @ wh.T + e4(xh / 32) @ e4(wl * 32).T + e4(xl * 32) @ e4(wh / 32).T) * m
    p1 = (xh @ wh.T) * m
    c = (dc * dc).sum(1) + 2 * ((mu - nu) * dc).sum(1)
    rex = c[None] - 2 * exact
    unit = 2.0 ** -11 * xc.norm(dim=1, keepdim=True) * dc.norm(dim=1).max() / math.sqrt(d)
    out = [f"ep{e}"]
    for name, p in (("1-pass", p1), ("3-pass", p3), ("f16+2xf8", p2)):
        r = c[None] - 2 * p
        err = ((r - rex).abs() / unit).max().item()
        rmin = r.min(1, keepdim=True).values
        cnt = [(r <= rmin + k * unit).sum(1).float().mean().item() for k in (0.5, 1, 2, 4)]
        out.append(f"{name}: max err {err:.3f} units, cand@k0.5/1/2/4 " + "/".join(f"{v:.1f}" for v in cnt))
    print("; ".join(out), flush=True)
    eng.epoch(r_, sc, 1e-3, S.Neighborhood(nbh), compact)
