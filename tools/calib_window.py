"""Calibrate the screening window on hardware, per data family: the tcgen05
screened values r~ (the kernel's own dump) against the exact fp64 r, in units
of each row's sigma_i (csrc/cand.cuh screen_sigma).

For sampled 128-row blocks after each epoch it reports
  need = r~_{j*} - min_j r~_j   (the window that keeps the exact argmin j*)
  err  = |r~ - r|               (single-node screen error)
both divided by sigma_i, plus the candidates a window of kappa * sigma_i
would keep, and the full-N screen's candidate statistics.  The engine trains
with the tensor screen; its BMUs are checked against an exact scan of the
sampled rows.
   python tools/calib_window.py FAMILY [cfg] [rows] [epochs] [passes] [blocks]
FAMILY: uniform dupcols nearconst blobs onehot10 int05 offset1000 rank4"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200 import _lib  # noqa: E402
from paper_1305_1422_b200.engine import EngineOptions, SomEngine, _ptr, _stream  # noqa: E402

FAMILIES = ("uniform", "dupcols", "nearconst", "blobs", "onehot10", "int05", "offset1000", "rank4")


def family_data(name, n, d, dev, seed=1001):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    r = lambda *s: torch.rand(s, generator=g, device=dev)
    if name == "uniform":
        return r(n, d)
    if name == "dupcols":
        return r(n, -(-d // 8)).repeat_interleave(8, dim=1)[:, :d].contiguous()
    if name == "nearconst":
        return r(n, 1) + 1e-3 * torch.randn((n, d), generator=g, device=dev)
    if name == "blobs":   # reference test_acceptance.py:304-327 style clusters
        cen = r(20, d)
        lab = torch.randint(0, 20, (n,), generator=g, device=dev)
        return cen[lab] + 0.05 * torch.randn((n, d), generator=g, device=dev)
    if name == "onehot10":
        x = torch.zeros((n, d), device=dev)
        idx = torch.argsort(r(n, d), dim=1)[:, :10]
        return x.scatter_(1, idx, 1.0)
    if name == "int05":
        return torch.randint(0, 6, (n, d), generator=g, device=dev).float()
    if name == "offset1000":
        return r(n, d) + 1000.0
    if name == "rank4":
        return r(n, 4) @ r(4, d)
    raise SystemExit(f"unknown family {name}")


def sigma(xs, scal):
    """host restatement of cand.cuh screen_sigma (fp64)."""
    xs, sc = xs.double(), scal.double()
    sx = torch.minimum(xs[:, 2] * sc[1], xs[:, 3] * sc[3])
    sd = torch.minimum(xs[:, 1] * sc[5], xs[:, 0] * sc[6])
    return torch.sqrt(sx * sx + sd * sd) + 2.0 ** -20 * (sc[4] + 2 * xs[:, 0] * sc[1])


def dump_block(eng, r0):
    """screened values of rows [r0, r0 + 128) (the kernel dumps its first 128 rows)."""
    m = min(128, eng.n - r0)
    dump = torch.full((128, eng.kp), float("nan"), dtype=torch.float32, device=eng.dev)
    rb = eng.Xh.element_size() * eng.Xh.shape[1]
    xl_ptr = C_void(eng.Xl.data_ptr() + r0 * eng.Xl.element_size() * eng.Xl.shape[1]) if eng.Xl is not None else None
    _lib.call("somb_debug_screen_dump", C_void(eng.Xh.data_ptr() + r0 * rb), xl_ptr,
              C_void(eng.xstat.data_ptr() + r0 * 16), m, eng.dp, _ptr(eng.Wh), _ptr(eng.Wl), _ptr(eng.c), eng.kp,
              _ptr(eng.scal), C_float(eng.window_coef), eng.passes, _ptr(dump), _ptr(eng.ws), _stream(eng.dev))
    return dump[:m, : eng.K]


def main():
    fam = sys.argv[1]
    cfg = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
    n0, d, nx, ny, mt, grid, nbh, compact, _ = bench.CONFIGS[cfg]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else n0
    E = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    passes = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    blocks = int(sys.argv[6]) if len(sys.argv) > 6 else 32
    dev = torch.device("cuda", 0)
    X = family_data(fam, n, d, dev)
    eng = SomEngine(X, nx, ny, S.MapType(mt), S.GridType(grid), device=dev,
                    options=EngineOptions(screen_passes=passes))
    eng.init_codebook_device(1)
    kap = (0.25, 0.5, 1.0, 2.0) if eng.passes == 2 else (2.0, 4.0, 6.0, 8.0)
    step = max(1, (n // 128) // blocks)
    out = {"family": fam, "config": cfg, "rows": n, "d": d, "K": eng.K, "passes": eng.passes,
           "window_kappa": eng.window_coef, "epochs": []}
    for e in range(E):
        eng.prepare()
        W = eng.W[: eng.K].double()
        mu = W.mean(0).float().double()
        dl = W - mu
        nu = eng.nu.double()
        c = (dl * dl).sum(1) + 2 * (dl * (mu - nu)).sum(1)
        need_max = err_max = 0.0
        cand = {k: 0.0 for k in kap}
        nrows = 0
        wrong = 0
        for b in range(0, (n // 128) * 128, step * 128):
            rt = dump_block(eng, b).double()
            xb = X[b: b + rt.shape[0]].double()
            xc = xb - nu
            r = c[None] - 2 * xc @ dl.T
            d2 = ((xb * xb).sum(1, keepdim=True) - 2 * xb @ W.T) + (W * W).sum(1)[None]
            js = d2.argmin(1)
            sg = sigma(eng.xstat[b: b + rt.shape[0]], eng.scal)
            fin = torch.isfinite(rt)
            need = rt.gather(1, js[:, None])[:, 0] - torch.where(fin, rt, torch.inf).min(1).values
            need_max = max(need_max, float((need / sg).max()))
            err = torch.where(fin, (rt - r).abs(), torch.zeros_like(rt))
            err_max = max(err_max, float((err / sg[:, None]).max()))
            rmin = torch.where(fin, rt, torch.inf).min(1, keepdim=True).values
            for k in kap:
                cand[k] += float((rt <= rmin + k * sg[:, None]).sum())
            nrows += rt.shape[0]
        st = bench.schedule_for(cfg, e)
        eng.search()
        cc = eng.candidate_counts()[: n].float()
        rep = eng.repaired_rows()
        # the engine's BMUs on the sampled rows vs an exact scan
        rows = torch.arange(0, (n // 128) * 128, step * 128, device=dev)[:, None] + torch.arange(128, device=dev)
        rows = rows.reshape(-1)[:4096]
        xb = X[rows].double()
        d2 = ((xb * xb).sum(1, keepdim=True) - 2 * xb @ W.T) + (W * W).sum(1)[None]
        wrong = int((d2.argmin(1).int() != eng.bmu[rows]).sum())
        rec = {"epoch": e, "need_over_sigma_max": need_max, "err_over_sigma_max": err_max,
               "cand_mean_at_kappa": {str(k): cand[k] / nrows for k in kap},
               "screen_cand_mean": float(cc.mean()), "screen_cand_max": int(cc.max()),
               "repaired_rows": rep, "bmu_vs_exact_mismatch_4096": wrong}
        print(json.dumps(rec), flush=True)
        out["epochs"].append(rec)
        eng.qe_sum()
        eng.node_sums()
        eng.update(st[0], st[1], 1e-3, S.Neighborhood(nbh), compact)
    out["need_over_sigma_max"] = max(r["need_over_sigma_max"] for r in out["epochs"])
    out["err_over_sigma_max"] = max(r["err_over_sigma_max"] for r in out["epochs"])
    out["bmu_mismatch_total"] = sum(r["bmu_vs_exact_mismatch_4096"] for r in out["epochs"])
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open(f"gpurun_out/calib_{fam}_{cfg}_p{eng.passes}.json", "w"), indent=1)
    print("SUMMARY", fam, cfg, "passes", eng.passes, "need/sigma max %.3f err/sigma max %.3f mismatches %d" % (
        out["need_over_sigma_max"], out["err_over_sigma_max"], out["bmu_mismatch_total"]), flush=True)


from ctypes import c_float as C_float, c_void_p as C_void  # noqa: E402

if __name__ == "__main__":
    main()
