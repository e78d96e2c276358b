"""Profile helper: a bench config's BMU search after `warm` epochs.
   python tools/prof_cfg.py [cfg] [warm] [passes]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200.engine import EngineOptions, SomEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
passes = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n, d, nx, ny, mt, grid, nbh, compact, _ = bench.CONFIGS[cfg]
g = torch.Generator(device="cuda")
g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device="cuda")
eng = SomEngine(X, nx, ny, S.MapType(mt), S.GridType(grid), options=EngineOptions(screen_passes=passes))
eng.init_codebook_device(1)
for e in range(warm):
    r, sc = bench.schedule_for(cfg, e)
    eng.epoch(r, sc, 1e-3, S.Neighborhood(nbh), compact)
eng.search()
torch.cuda.synchronize()
print("done")
