"""CPU emulation of the screen's operand rounding on structured data (no GPU):
how wide must the screening window be, per row, to keep the exact BMU?

For each dataset family and epoch (a small exact fp64 batch SOM supplies
realistic codebooks) it quantises the centred operands like prep.cu -- fp16
round-to-nearest (the round-1 scheme) or stochastic rounding (dither) -- and
forms the screened values r~ with fp32 accumulation per 16-feature MMA step,
then reports, per row, need_i = r~_{j*} - min_j r~_j (the smallest window that
keeps the exact argmin j*) in two units:
  old  2^-11 |x'_i| max_j|delta_j| / sqrt(d)           (round-1 window unit)
  sig  the per-row Hoeffding scale of the dither       (engine._window_sigma)
   python tools/window_emul.py [d] [rows] [passes] [epochs...]"""
import math
import os
import sys

import numpy as np
import torch

torch.set_num_threads(os.cpu_count() or 8)
D = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
N = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
PASSES = int(sys.argv[3]) if len(sys.argv) > 3 else 1
EPOCHS = [int(a) for a in sys.argv[4:]] or [0, 1, 3, 6, 9]
NX = NY = 40
K = NX * NY
f64 = torch.float64


def datasets(n, d, seed=1001):
    rng = np.random.default_rng(seed)
    u = rng.random((n, d), dtype=np.float32)
    dup = np.repeat(rng.random((n, d // 8), dtype=np.float32), 8, axis=1)[:, :d]
    const = (rng.random((n, 1)) + 1e-3 * rng.standard_normal((n, d))).astype(np.float32)
    cen = rng.random((20, d))
    blobs = (cen[rng.integers(0, 20, n)] + 0.05 * rng.standard_normal((n, d))).astype(np.float32)
    onehot = np.zeros((n, d), np.float32)
    for i in range(n):
        onehot[i, rng.choice(d, 10, replace=False)] = 1.0
    ints = rng.integers(0, 6, (n, d)).astype(np.float32)
    offs = (u + np.float32(1000.0)).astype(np.float32)
    lowrank = (rng.random((n, 4)) @ rng.random((4, d))).astype(np.float32)
    return {"uniform": u, "dupcols": dup, "nearconst": const, "blobs": blobs, "onehot10": onehot,
            "int0-5": ints, "offset1000": offs, "rank4": lowrank}


def grid_h(radius):
    c = torch.arange(K)
    x, y = (c % NX).to(f64), (c // NX).to(f64)
    dx = (x[:, None] - x[None]).abs()
    dy = (y[:, None] - y[None]).abs()
    dx, dy = torch.minimum(dx, NX - dx), torch.minimum(dy, NY - dy)
    h = torch.exp(-torch.hypot(dx, dy) / radius)
    h[h < 1e-3] = 0
    return h


def som_epoch(X, W, radius):
    d2 = (X * X).sum(1, keepdim=True) + (W * W).sum(1)[None] - 2 * X @ W.T
    b = d2.argmin(1)
    S = torch.zeros_like(W).index_add_(0, b, X)
    cnt = torch.bincount(b, minlength=K).to(f64)
    h = grid_h(radius)
    num, den = h @ S, h @ cnt
    m = den > 0
    W = W.clone()
    W[m] = num[m] / den[m, None]
    return W.float().double()


def ulp16(v):
    a = v.abs()
    e = torch.floor(torch.log2(torch.where(a > 0, a, torch.ones_like(a))))
    return torch.where(a > 0, torch.exp2(torch.clamp(e, min=-14) - 10), torch.zeros_like(a))


def q16(v, mode, gen):
    if mode == "rn":
        return v.half().double()
    u = ulp16(v)
    lo = torch.where(u > 0, torch.floor(v / torch.where(u > 0, u, 1)) * u, v)
    p = torch.where(u > 0, (v - lo) / torch.where(u > 0, u, 1), torch.zeros_like(v))
    return lo + u * (torch.rand(v.shape, generator=gen, dtype=f64) < p)


def e4(v):
    return v.to(torch.float8_e4m3fn).double()


def acc32(A, B, k=16):
    """fp32 accumulation per k-feature MMA step (products exact)."""
    acc = torch.zeros((A.shape[0], B.shape[0]), dtype=torch.float32)
    for s in range(0, A.shape[1], k):
        acc = (acc.double() + A[:, s:s + k] @ B[:, s:s + k].T).float()
    return acc.double()


def screen(Xf, W, mode, gen, passes):
    nu = Xf.mean(0).float().double()
    mu = W.mean(0).float().double()
    xc, dc = Xf - nu, W - mu
    top = 13 if passes == 2 else 14
    xexp = top - math.frexp(float(xc.abs().max()))[1]
    sexp = top - math.frexp(float(dc.abs().max()))[1]
    y, z = xc * 2.0 ** xexp, dc * 2.0 ** sexp
    yh, zh = q16(y, mode, gen), q16(z, mode, gen)
    acc = acc32(yh, zh)
    if passes == 2:
        cross = acc32(torch.cat([e4(yh / 32), e4((y - yh) * 32)], 1), torch.cat([e4((z - zh) * 32), e4(zh / 32)], 1), 32)
        acc = (cross + acc)          # (the device accumulates hi.hi on top of the fp8 cross terms)
    m = -2.0 * 2.0 ** -(xexp + sexp)
    c = ((dc * dc).sum(1) + 2 * (dc * (mu - nu)).sum(1)).float().double()
    r = (acc * m + c[None]).float().double()
    rex = c[None] - 2 * xc @ dc.T
    # per-row scales
    old = 2.0 ** -11 * xc.norm(dim=1) * dc.norm(dim=1).max() / math.sqrt(xc.shape[1])
    # dither scale (dot-product units): x side sum_k ulp_x^2 delta^2 and delta side sum_k x'^2 ulp_d^2,
    # each bounded by the min of its two Hoelder forms; ulps of the scaled values mapped back
    ux, ud = ulp16(y) * 2.0 ** -xexp, ulp16(z) * 2.0 ** -sexp
    dn2, dinf = dc.norm(dim=1).max(), dc.abs().max()
    sx = torch.minimum(ux.abs().max(1).values * dn2, ux.norm(dim=1) * dinf)
    sd = torch.minimum(xc.abs().max(1).values * ud.norm(dim=1).max(), xc.norm(dim=1) * ud.max())
    sig = torch.sqrt(sx ** 2 + sd ** 2)
    return r, rex, old, sig


def main():
    gen = torch.Generator().manual_seed(7)
    print(f"d={D} rows={N} K={K} passes={PASSES}")
    for name, X in datasets(N, D).items():
        Xf = torch.from_numpy(X).double()
        W = torch.from_numpy(np.random.default_rng(1).random((K, D), dtype=np.float32)).double()
        rows = []
        for e in range(max(EPOCHS) + 1):
            radius = 20 + (1 - 20) * e / 9
            if e in EPOCHS:
                for mode in ("rn", "sr"):
                    r, rex, old, sig = screen(Xf, W, mode, gen, PASSES)
                    js = rex.argmin(1)
                    need = r.gather(1, js[:, None])[:, 0] - r.min(1).values
                    rel_gap = torch.topk(rex, 2, dim=1, largest=False).values
                    err = (r - rex)
                    err = err - err.median(1, keepdim=True).values
                    rows.append(f"  ep{e} {mode}: need/old max {float((need / old).max()):7.2f}  "
                                f"need/sig max {float((need / sig).max()):6.2f}  "
                                f"|err|/old max {float((err.abs() / old[:, None]).max()):7.2f}  "
                                f"|err|/sig max {float((err.abs() / sig[:, None]).max()):6.2f}  "
                                f"sig/old med {float((sig / old).median()):5.2f}  "
                                f"cand@10old {float((r <= r.min(1, keepdim=True).values + 10 * old[:, None]).sum(1).double().mean()):6.1f}  "
                                f"cand@6sig {float((r <= r.min(1, keepdim=True).values + 6 * sig[:, None]).sum(1).double().mean()):6.1f}")
            W = som_epoch(Xf, W, radius)
        print(name)
        print("\n".join(rows), flush=True)


if __name__ == "__main__":
    main()
