"""Split the cfg2 engine construction (the first ~200 ms of train()) into
the pageable upload, the engine build on resident rows, and its pieces.
   python tools/e2e_init_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200 import engine as E  # noqa: E402

n, d, nx, ny = 1_000_000, 1000, 200, 200
Xn = np.random.default_rng(1001).random((n, d), dtype=np.float32)
dev = torch.device("cuda", 0)
torch.zeros(1, device=dev)
for rep in range(3):
    torch.cuda.synchronize()
    T = {}
    t = time.perf_counter()

    def lap(name):
        global t
        torch.cuda.synchronize()
        now = time.perf_counter()
        T[name] = round((now - t) * 1e3, 2)
        t = now
    X = E.to_device(Xn, dev)
    lap("to_device 4GB")
    orig = E.SomEngine.pack_dataset
    pk = {}

    def timed_pack(self):
        torch.cuda.synchronize()
        a = time.perf_counter()
        orig(self)
        torch.cuda.synchronize()
        pk["pack"] = round((time.perf_counter() - a) * 1e3, 2)
    E.SomEngine.pack_dataset = timed_pack
    eng = E.SomEngine(X, nx, ny, S.MapType.TOROID)
    E.SomEngine.pack_dataset = orig
    lap("SomEngine(resident X)")
    T.update(pk)
    eng.init_codebook_device(1)
    lap("init codebook")
    print(rep, T, flush=True)
    del eng, X
    if rep == 1:
        torch.cuda.empty_cache()
