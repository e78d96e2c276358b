"""Phase times (sync + wall clock after each) of the sparse train() steps at cfg3.
   python tools/e2e_sparse_phases.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200 import _lib  # noqa: E402
from paper_1305_1422_b200.kernels import make_engine  # noqa: E402

n, d, nx, ny = 500_000, 50_000, 100, 100
rp, cl, vl = bench.sparse_rows_device(n, d, bench.SPARSE_NNZ, 1001, torch.device("cuda", 0))
data = S.SparseDataset(d, rp.cpu().numpy(), cl.cpu().numpy(), vl.cpu().numpy())
cfg = S.resolve_defaults(S.TrainConfig(n_epochs=10, n_columns=nx, n_rows=ny, kernel=S.Kernel.SPARSE, seed=1))
for rep in range(2):
    torch.cuda.synchronize()
    T = {}
    t0 = t = time.perf_counter()

    def lap(name):
        global t
        torch.cuda.synchronize()
        now = time.perf_counter()
        T[name] = round((now - t) * 1e3, 1)
        t = now
    eng = make_engine(data, nx, ny, cfg.map_type, cfg.grid)
    lap("engine+H2D")
    eng.init_codebook_device(cfg.seed)
    lap("init")
    for e in range(cfg.n_epochs):
        st = S.epoch_schedules(cfg, e)
        eng.epoch(st.radius, st.scale, cfg.influence_cutoff)
        lap(f"epoch{e}")
    eng.search(_lib.DIST_BLOCKED)
    lap("final pass")
    b = eng.bmu_coords()
    lap("bmus D2H")
    w = eng.codebook()
    lap("codebook D2H")
    T["total"] = round((time.perf_counter() - t0) * 1e3, 1)
    print(T, flush=True)
    del eng
    torch.cuda.empty_cache()
