"""Pageable numpy -> device upload of a cfg2-size dataset: pinning a full
copy (torch pin_memory) vs the chunked pinned staging of engine.to_device.
   python tools/upload_probe.py [rows] [d]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_1422_b200.engine import to_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
x = np.random.default_rng(1).random((n, d), dtype=np.float32)
dev = torch.device("cuda", 0)
torch.zeros(1, device=dev)
for rep in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    a = torch.from_numpy(x).pin_memory().to(dev, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter() - t
    del a
    t = time.perf_counter()
    b = to_device(x, dev)
    torch.cuda.synchronize()
    t2 = time.perf_counter() - t
    ok = bool(torch.equal(b[:: 9973].cpu(), torch.from_numpy(x[:: 9973])))
    del b
    print(f"{x.nbytes / 1e9:.1f} GB: pin_memory + H2D {t1 * 1e3:.0f} ms, staged {t2 * 1e3:.0f} ms, equal {ok}", flush=True)
