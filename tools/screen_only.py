"""Time only the screen kernel (CUDA events) at the cfg2 shape after `warm`
reference epochs; env knobs (SOMB_SCREEN_LAG, SOMB_SCREEN_PROFILE, ...) are
read once per process.   python tools/screen_only.py [warm] [reps]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1305_1422_b200 as S  # noqa: E402
from paper_1305_1422_b200 import _lib  # noqa: E402
from paper_1305_1422_b200.engine import SomEngine, _ptr, _stream  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n, d, nx, ny = 1_000_000, 1000, 200, 200
g = torch.Generator(device="cuda")
g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device="cuda")
eng = SomEngine(X, nx, ny, S.MapType.TOROID)
eng.set_codebook(S.init_codebook(S.TrainConfig(n_columns=nx, n_rows=ny, seed=1), d).weights)
for e in range(warm):
    r, sc = bench.schedule_for("cfg2", e)
    eng.epoch(r, sc, 1e-3)
eng.prepare()
lib = _lib.load()


def run(tag, **knobs):
    for k, v in knobs.items():
        assert lib.somb_set_knob(k.encode(), int(v)) == 0
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.call("somb_bmu_screen", _ptr(eng.Xh), _ptr(eng.Xl), _ptr(eng.xnorm), eng.n, eng.dp, _ptr(eng.Wh),
                  _ptr(eng.Wl), _ptr(eng.c), eng.K, eng.kp, _ptr(eng.scal), C.c_float(eng.window_coef),
                  _ptr(eng.bmu), 0, _ptr(eng.flags), _ptr(eng.ws), _stream(eng.dev))
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{tag}: screen ms {[round(t, 2) for t in ts]} min {min(ts):.2f} "
          f"-> {2.0 * n * nx * ny * d / (min(ts) / 1e3) / 1e12:.0f} TF/s", flush=True)


for mc in (1, 2, 1, 2):
    for lag in (8, 0, 16):
        run(f"multicast {mc} lag {lag}", tc_multicast=mc, screen_lag=lag)
run("mc2 lag 8 profile (no epilogue)", tc_multicast=2, screen_lag=8, screen_profile=1)
run("mc1 lag 8 profile (no epilogue)", tc_multicast=1, screen_lag=8, screen_profile=1)
run("back to normal", tc_multicast=2, screen_lag=8, screen_profile=0)
