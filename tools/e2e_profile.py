"""Where does the end-to-end train() time go?  Replays train()'s steps for the
cfg2 workload from pageable numpy rows with a sync + wall clock after each.
   python tools/e2e_profile.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200 import _lib  # noqa: E402
from paper_1305_1422_b200.kernels import make_engine  # noqa: E402
from paper_1305_1422_b200.train import _to_coords  # noqa: E402

n, d, nx, ny = 1_000_000, 1000, 200, 200
Xh = np.random.default_rng(1001).random((n, d), dtype=np.float32)   # pageable numpy, as a reference user passes it
cfg = S.resolve_defaults(S.TrainConfig(n_epochs=10, n_columns=nx, n_rows=ny, map_type=S.MapType.TOROID))
for rep in range(2):
    torch.cuda.synchronize()
    T = {}
    t0 = t = time.perf_counter()

    def lap(name):
        global t
        torch.cuda.synchronize()
        now = time.perf_counter()
        T[name] = round((now - t) * 1e3, 2)
        t = now
    eng = make_engine(S.DenseDataset(Xh), nx, ny, cfg.map_type, cfg.grid)
    lap("engine+H2D+pack")
    eng.init_codebook_device(cfg.seed)
    lap("init")
    for e in range(cfg.n_epochs):
        st = S.epoch_schedules(cfg, e)
        eng.epoch(st.radius, st.scale, cfg.influence_cutoff)
    lap("10 epochs")
    eng.search(_lib.DIST_NAIVE)
    lap("final pass")
    b = _to_coords(eng.gather_bmus(), nx)
    lap("bmus D2H")
    w = eng.codebook()
    lap("codebook D2H")
    u = eng.umatrix().cpu().numpy()
    lap("umatrix")
    T["total"] = round((time.perf_counter() - t0) * 1e3, 2)
    print(T, flush=True)
    del eng
    torch.cuda.empty_cache()
