"""Full-scale exactness sweep of the screened BMU search (Next 1-2).

Trains a bench config for 10 epochs with the production path (tcgen05 screen
+ fp64 re-rank + node sums + spectral update) and, EVERY epoch, compares the
engine's BMU of EVERY row with an exact fp64 argmin over all nodes computed
independently with cuBLAS/cuSPARSE fp64 GEMMs (torch): the reference's blocked
formula ((-2 x.w) + |x|^2) + |w|^2 clamped >= 0 (kernels.py:196-202) with
first-minimum ties (kernels.py:27-28), teacher-forced on the engine's own
codebook of that epoch.  A BMU that differs from the exact argmin is a screen
miss unless the two nodes' exact distances tie to fp64 summation order; the
relative gap of every mismatch is reported.

   python tools/parity_sweep.py CFG FAMILY [rows] [epochs]
FAMILY: a tools/calib_window.py family (dense configs) or "sparse" (cfg3).
Writes gpurun_out/parity_CFG_FAMILY_ROWS.json."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200.engine import SomEngine  # noqa: E402

TIE_GAP = 1e-12   # relative gap below which two exact fp64 distances are summation-order ties


def exact_argmin_dense(X, x2, W, w2, rows_per_chunk):
    """first-minimum argmin of ((-2 x.w) + |x|^2) + |w|^2, clamp 0, in fp64, plus the
    distance table rows needed to judge mismatches (returned lazily via a closure)."""
    W64 = W.double()
    out = torch.empty(X.shape[0], dtype=torch.int64, device=X.device)
    for a in range(0, X.shape[0], rows_per_chunk):
        xb = X[a: a + rows_per_chunk].double()
        d2 = torch.clamp((-2.0 * (xb @ W64.T) + x2[a: a + rows_per_chunk, None]) + w2[None, :], min=0.0)
        out[a: a + rows_per_chunk] = torch.argmin(d2, dim=1)
    return out


def gaps_dense(X, x2, W, w2, rows, got, want):
    W64 = W.double()
    xb = X[rows].double()
    dg = torch.clamp((-2.0 * (xb * W64[got]).sum(1) + x2[rows]) + w2[got], min=0.0)
    dw = torch.clamp((-2.0 * (xb * W64[want]).sum(1) + x2[rows]) + w2[want], min=0.0)
    scale = x2[rows] + w2.max()
    return ((dg - dw) / scale).tolist()


def main():
    cfg = sys.argv[1]
    fam = sys.argv[2]
    n0, d, nx, ny, mt, grid, nbh, compact, desc = bench.CONFIGS[cfg]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else n0
    E = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    dev = torch.device("cuda", 0)
    sparse = cfg == "cfg3"
    t0 = time.time()
    if sparse:
        from paper_1305_1422_b200.sparse import SparseEngine
        rp, cl, vl = bench.sparse_rows_device(n, d, bench.SPARSE_NNZ, 1001, dev)
        eng = SparseEngine(S.SparseDataset(d, rp.cpu().numpy(), cl.cpu().numpy(), vl.cpu().numpy()), nx, ny,
                           S.MapType(mt), S.GridType(grid), device=dev)
        x2 = torch.zeros(n, dtype=torch.float64, device=dev).index_add_(
            0, torch.repeat_interleave(torch.arange(n, device=dev), rp[1:] - rp[:-1]), vl.double() ** 2)
    else:
        from calib_window import family_data
        X = family_data(fam, n, d, dev)
        eng = SomEngine(X, nx, ny, S.MapType(mt), S.GridType(grid), device=dev)
        x2 = eng.x2[:n]
    eng.init_codebook_device(1)
    K = eng.K
    chunk = max(256, int(4e9 // (8 * K)))
    res = {"config": desc, "family": fam, "rows": n, "epochs": [], "tie_gap": TIE_GAP,
           "reference": "exact fp64 argmin over all nodes by torch cuBLAS/cuSPARSE GEMMs (kernels.py:196-202, "
                        "first-minimum ties kernels.py:27-28), teacher-forced on the engine's codebook each epoch"}
    for e in range(E):
        radius, scale = bench.schedule_for(cfg, e)
        eng.search()
        W = eng.W[:K]
        w2 = eng.w2[:K]
        if sparse:
            W64 = W.double()
            want = torch.empty(n, dtype=torch.int64, device=dev)
            for a in range(0, n, chunk):
                b = min(n, a + chunk)
                sub = torch.sparse_csr_tensor(rp[a: b + 1].long() - int(rp[a]), cl[int(rp[a]): int(rp[b])].long(),
                                              vl[int(rp[a]): int(rp[b])].double(), size=(b - a, d), device=dev)
                dots = (sub @ W64.T)
                d2 = torch.clamp((x2[a:b, None] - 2.0 * dots) + w2[None, :], min=0.0)
                want[a:b] = torch.argmin(d2, dim=1)
        else:
            want = exact_argmin_dense(X, x2, W, w2, chunk)
        got = eng.bmu[:n].long()
        bad = torch.nonzero(got != want).flatten()
        try:
            rep = eng.repaired_rows()
        except Exception:   # (layout of the sparse workspace)
            rep = None
        rec = {"epoch": e, "mismatches": int(bad.numel()), "repaired_rows": rep,
               "candidates_mean": float(eng.candidate_counts()[:n].float().mean()) if not sparse else None}
        if bad.numel() and not sparse:
            g = gaps_dense(X, x2, W, w2, bad[:4096], got[bad[:4096]], want[bad[:4096]])
            rec["max_rel_gap"] = max(g)
            rec["beyond_tie_gap"] = sum(1 for v in g if v > TIE_GAP)
        elif bad.numel():
            rec["max_rel_gap"] = None
        print(json.dumps(rec), flush=True)
        res["epochs"].append(rec)
        eng.qe_sum()
        eng.node_sums()
        eng.reduce()
        eng.update(radius, scale, 1e-3, S.Neighborhood(nbh), compact)
    res["mismatches_total"] = sum(r["mismatches"] for r in res["epochs"])
    res["beyond_tie_gap_total"] = sum(r.get("beyond_tie_gap", 0) or 0 for r in res["epochs"])
    res["seconds"] = time.time() - t0
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open(f"gpurun_out/parity_{cfg}_{fam}_{n}.json", "w"), indent=1)
    print("SUMMARY", cfg, fam, n, "mismatches", res["mismatches_total"], "beyond tie gap",
          res["beyond_tie_gap_total"], f"{res['seconds']:.0f} s", flush=True)


if __name__ == "__main__":
    main()
