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
cfgn = sys.argv[3] if len(sys.argv) > 3 else "cfg2"
passes = int(sys.argv[4]) if len(sys.argv) > 4 else 0
n, d, nx, ny, mt, grid, nbh, compact, _ = bench.CONFIGS[cfgn]
g = torch.Generator(device="cuda")
g.manual_seed(1001)
X = torch.rand((n, d), generator=g, device="cuda")
from paper_1305_1422_b200.engine import EngineOptions  # noqa: E402
eng = SomEngine(X, nx, ny, S.MapType(mt), S.GridType(grid), options=EngineOptions(screen_passes=passes))
eng.init_codebook_device(1)
for e in range(warm):
    r, sc = bench.schedule_for(cfgn, e)
    eng.epoch(r, sc, 1e-3, S.Neighborhood(nbh), compact)
eng.prepare()
lib = _lib.load()


def run(tag, **knobs):
    for k, v in knobs.items():
        assert lib.somb_set_knob(k.encode(), int(v)) == 0
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.call("somb_bmu_screen", _ptr(eng.Xh), _ptr(eng.Xl), _ptr(eng.xstat), eng.n, eng.dp, _ptr(eng.Wh),
                  _ptr(eng.Wl), _ptr(eng.c), eng.K, eng.kp, _ptr(eng.scal), C.c_float(eng.window_coef),
                  _ptr(eng.bmu), eng.screen_impl, _ptr(eng.flags), _ptr(eng.ws), _stream(eng.dev))
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{tag}: screen ms {[round(t, 2) for t in ts]} min {min(ts):.2f} "
          f"-> {2.0 * n * nx * ny * d / (min(ts) / 1e3) / 1e12:.0f} TF/s", flush=True)


if cfgn == "cfg2":
    for mc in (1, 2, 1, 2):
        for lag in (8, 0, 16):
            run(f"multicast {mc} lag {lag}", tc_multicast=mc, screen_lag=lag)
for lag in (8, 0):
    run(f"{cfgn} passes {eng.passes} lag {lag}", screen_lag=lag)
run(f"{cfgn} passes {eng.passes} profile 1 (no epilogue)", screen_lag=8, screen_profile=1)
run(f"{cfgn} passes {eng.passes} profile 2 (TMEM loads only)", screen_lag=8, screen_profile=2)
run(f"{cfgn} passes {eng.passes} profile 3 (loads + window arithmetic)", screen_lag=8, screen_profile=3)
run("back to normal", screen_lag=8, screen_profile=0)
