"""Profile helper: cfg3-shaped sparse BMU searches after `warm` epochs.
   python tools/prof_sparse.py [rows] [warm]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200.sparse import SparseEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
d, nx, ny = 50_000, 100, 100
dev = torch.device("cuda", 0)
rp, cl, vl = bench.sparse_rows_device(n, d, bench.SPARSE_NNZ, 1001, dev)
data = S.SparseDataset(d, rp.cpu().numpy(), cl.cpu().numpy(), vl.cpu().numpy())
eng = SparseEngine(data, nx, ny, S.MapType.PLANAR, device=dev)
eng.init_codebook_device(1)
for e in range(warm):
    r, sc = bench.schedule_for("cfg3", e)
    eng.epoch(r, sc, 1e-3)
eng.search()
torch.cuda.synchronize()
print("done")
