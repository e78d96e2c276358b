"""Where does the end-to-end sparse train() time go (cfg3: 500k CSR rows x
50,000, 10x10 ... 100x100 map)?  cProfile of one warm train() call.
   python tools/e2e_sparse_profile.py"""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402

n, d, nx, ny = 500_000, 50_000, 100, 100
rp, cl, vl = bench.sparse_rows_device(n, d, bench.SPARSE_NNZ, 1001, torch.device("cuda", 0))
data = S.SparseDataset(d, rp.cpu().numpy(), cl.cpu().numpy(), vl.cpu().numpy())
cfg = S.TrainConfig(n_epochs=10, n_columns=nx, n_rows=ny, kernel=S.Kernel.SPARSE, seed=1)
S.train(data, S.TrainConfig(n_epochs=1, n_columns=nx, n_rows=ny, kernel=S.Kernel.SPARSE), local_rows=True)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
S.train(data, cfg, local_rows=True)
torch.cuda.synchronize()
pr.disable()
print(f"train(): {time.perf_counter() - t0:.2f} s")
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
