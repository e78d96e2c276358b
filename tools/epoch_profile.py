"""Per-epoch phase profile of a bench config: for epochs 0..9 of the reference
schedule, CUDA-event time of each phase plus the screen's candidate-count
distribution and truncation rate (read before node sums reuses the
workspace).
   python tools/epoch_profile.py [cfg2|cfg4|cfg5] [passes]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200.engine import EngineOptions, SomEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
passes = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n, d, nx, ny, mt, grid, nbh, compact, desc = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device=dev)
eng = SomEngine(X, nx, ny, S.MapType(mt), S.GridType(grid), device=dev,
                options=EngineOptions(screen_passes=passes))
eng.set_codebook(S.init_codebook(S.TrainConfig(n_columns=nx, n_rows=ny, seed=1), d).weights)
rows = []
for e in range(10):
    r, sc = bench.schedule_for(cfg, e)
    eng.timing = {}
    eng.search()
    torch.cuda.synchronize()
    cc = eng.candidate_counts()[: eng.n].float().cpu().numpy()
    fl = eng.flags[: eng.n].cpu().numpy()
    trunc = float((((fl & 0xFF) | ((fl >> 8) & 0xFF) | ((fl >> 16) & 0xFF) | ((fl >> 24) & 0xFF)) & 1).astype(bool).mean())
    spilled = float((((fl & 0xFF) | ((fl >> 8) & 0xFF) | ((fl >> 16) & 0xFF) | ((fl >> 24) & 0xFF)) & 2).astype(bool).mean())
    chunks = eng.overflow_chunks() if eng.screen_impl == 0 and eng.passes >= 1 else 0
    eng._mark("node_sums", True)
    eng.qe_sum()
    eng.node_sums()
    eng._mark("node_sums", False)
    eng._mark("update", True)
    eng.update(r, sc, 1e-3, S.Neighborhood(nbh), compact)
    eng._mark("update", False)
    torch.cuda.synchronize()
    ph = {k: round(v[0][0].elapsed_time(v[0][1]), 2) for k, v in eng.timing.items()}
    row = {"epoch": e, "radius": round(r, 2), "scale": round(sc, 3), **ph,
           "cand_mean": round(float(cc.mean()), 2), "cand_p50": float(np.median(cc)),
           "cand_p99": float(np.percentile(cc, 99)), "cand_max": float(cc.max()), "trunc": trunc,
           "spilled": spilled, "ovf_chunks": chunks}
    rows.append(row)
    print(json.dumps(row), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(rows, open(os.path.join(ROOT, "gpurun_out", f"epoch_profile_{cfg}_p{eng.passes}.json"), "w"), indent=1)
w = eng.W[: eng.K].double()
print(json.dumps({"codebook_sum": float(w.sum()), "codebook_sq": float((w * w).sum()),
                  "bmu_hash": int((eng.bmu[: eng.n].long() * torch.arange(1, eng.n + 1, device=dev)).sum())}))
