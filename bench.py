#!/usr/bin/env python
"""Benchmark of the batch-SOM epoch hot path (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config cfg2|cfg1|cfg4|cfg5]

A step is one training epoch (tcgen05 BMU screen + fp64 re-rank + node sums
+ [NCCL all-reduce] + fp64 neighbourhood convolution + blend) over the whole
synthetic dataset of the config, following the config's 10-epoch radius/scale
schedule (step s runs epoch s mod 10).  Default workload: BASELINE cfg2 --
200x200 toroid (K = 40,000), 1M x 1000 fp32, rows sharded over the N ranks
(strong scaling).  `value` = N_rows * K / epoch time (BMU distance
evaluations per second, whole job); X (4 GB) exceeds L2, so no flush is needed.

--impl reference times the CPU path of the reference algorithm (the numpy
oracle port, all host cores) on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n_rows, d, nx, ny, map, grid, neighborhood, compact, description)
    "cfg1": (10_000, 100, 50, 40, "planar", "rectangular", "gaussian", False,
             "cfg1: dense 50x40 planar rect map, 10k x 100 fp32 uniform, gaussian"),
    "cfg2": (1_000_000, 1000, 200, 200, "toroid", "rectangular", "gaussian", False,
             "cfg2: emergent 200x200 toroid, 1M x 1000 fp32 uniform, gaussian"),
    "cfg3": (500_000, 50_000, 100, 100, "planar", "rectangular", "gaussian", False,
             "cfg3: sparse 100x100 planar, 500k x 50k CSR, 250 nnz/row (0.5%), gaussian"),
    "cfg4": (2_000_000, 256, 300, 300, "toroid", "hexagonal", "bubble", True,
             "cfg4: hexagonal toroid 300x300, 2M x 256 fp32 uniform, bubble, compact support"),
    "cfg5": (4_000_000, 128, 500, 500, "planar", "rectangular", "gaussian", False,
             "cfg5: large emergent 500x500 planar, 4M x 128 fp32 uniform, gaussian"),
}
METRIC = "epoch time & BMU dist-evals/s (N·K·D) at 1/2/4/8 B200, % of roofline"
UNIT = "dist-evals/s"
N_EPOCHS = 10
L2_FLUSH_BYTES = 256 << 20   # > the 126 MB L2


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def measure_l2_gbs(dev):
    """Achievable L2 read bandwidth: somb_l2_probe (float4 loads, 4 blocks per
    SM) over a 48 MB fp32 buffer, L2-resident after the first pass, 40 passes
    timed with CUDA events.  The denominator of the L2-bound kernels'
    rooflines (sparse gather, re-rank candidate rows); no driver-written L2
    peak exists."""
    import ctypes as C
    import torch
    from paper_1305_1422_b200 import _lib
    buf = torch.rand(12 << 20, device=dev)
    out = torch.zeros(4 * 1024, device=dev)
    st = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    _lib.call("somb_l2_probe", C.c_void_p(buf.data_ptr()), buf.numel(), 4, C.c_void_p(out.data_ptr()), st)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    _lib.call("somb_l2_probe", C.c_void_p(buf.data_ptr()), buf.numel(), 40, C.c_void_p(out.data_ptr()), st)
    b.record()
    torch.cuda.synchronize()
    return 40 * buf.numel() * 4 / (a.elapsed_time(b) / 1e3) / 1e9


def schedule_for(cfg_name, epoch):
    n, d, nx, ny, *_ = CONFIGS[cfg_name]
    r0 = max(min(nx, ny) / 2.0, 1.0)
    e = epoch % N_EPOCHS
    frac = e / (N_EPOCHS - 1)
    radius = r0 + (1.0 - r0) * frac if 0 < e < N_EPOCHS - 1 else (r0 if e == 0 else 1.0)
    scale = 1.0 + (0.01 - 1.0) * frac if 0 < e < N_EPOCHS - 1 else (1.0 if e == 0 else 0.01)
    return radius, scale


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        post = False
        if not out.strip():   # region shorter than one sampling period: one query right after it
            post = True
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=10).stdout
            except (OSError, subprocess.SubprocessError):
                out = ""
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                **({"sampled": "once, right after a timed region shorter than 200 ms"} if post else {})}


def init_dist(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SOMB_EXCHANGE=always: a 1-rank NCCL group, so the sharded exchange
    # (reduce-scatter / all-reduce / all-gather) runs and is timed on one GPU
    if world > 1 or os.environ.get("SOMB_EXCHANGE") == "always":
        import torch.distributed as dist
        if world == 1:   # a 1-rank group outside torchrun: env:// rendezvous defaults
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        # SOMB_DIST_BACKEND=gloo (+ ranks sharing a GPU) exercises the sharded
        # path on a 1-GPU box; production runs use NCCL, one rank per GPU
        backend = os.environ.get("SOMB_DIST_BACKEND", "nccl")
        local = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


SPARSE_NNZ = 250


def sparse_rows_device(n, d, nnz, seed, dev):
    """Synthetic text-like CSR rows on the device: nnz distinct sorted columns
    per row (one uniform pick in each of nnz equal column bins), values U[0,1)."""
    import torch
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    width = d // nnz
    base = torch.arange(nnz, device=dev, dtype=torch.int64) * width
    cols = (base[None, :] + torch.randint(0, width, (n, nnz), generator=g, device=dev)).to(torch.int32)
    vals = torch.rand((n, nnz), generator=g, device=dev)
    rowptr = torch.arange(n + 1, device=dev, dtype=torch.int64) * nnz
    return rowptr, cols.reshape(-1), vals.reshape(-1)


def reference_rows(first, count, d, seed=1001):
    """Rows [first, first + count) of the reference generator's dataset
    gen_random_dense(n, d, seed) (reference bench.py:85-88, synth.py here):
    numpy default_rng(seed).random((n, d), float32) consumes one 32-bit half
    of a PCG64 output per value, so a rank's slice starts after advancing the
    bit generator first*d/2 outputs (bit-identical to slicing the full array)."""
    import numpy as np
    skip = first * d
    bg = np.random.PCG64(seed)
    bg.advance(skip // 2)
    g = np.random.Generator(bg)
    if skip % 2:
        g.random(1, dtype=np.float32)
    return g.random((count, d), dtype=np.float32)


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return None


def cpu_reference_rate(cfg_name, n_sub, steps, warmup, seed=1001):
    """Oracle port (numpy restatement of the reference path, kernels.py:365-450)
    on all host cores: search_accumulate(DENSE_BLOCKED) over an n_sub-row
    sample plus the full-codebook blend; the epoch time at full N is
    (N / n_sub) * t_search_accumulate + t_blend (cost is linear in N,
    SURVEY.md 8d)."""
    import numpy as np
    import oracle as O
    n, d, nx, ny, mt, grid, nbh, compact, _ = CONFIGS[cfg_name]
    rng = np.random.default_rng(seed)
    if cfg_name == "cfg3":
        x = O.gen_random_sparse(n_sub, d, SPARSE_NNZ / d, seed)
        kern = O.SPARSE
    else:
        x = rng.random((n_sub, d), dtype=np.float32)
        kern = O.DENSE_BLOCKED
    w = O.init_codebook(nx, ny, d, 1)
    og = O.HEX if grid == "hexagonal" else O.RECT
    workers = os.cpu_count() or 1
    t_sa, t_bl = [], []
    for s in range(warmup + steps):
        radius, scale = schedule_for(cfg_name, s)
        t0 = time.perf_counter()
        _, _, num, den = O.search_accumulate(x, w, nx, ny, radius, 1e-3, mt, kern, workers,
                                             True, og, nbh, compact)
        t1 = time.perf_counter()
        w = O.blend(w, num, den, scale)
        t2 = time.perf_counter()
        t_sa.append(t1 - t0)
        t_bl.append(t2 - t1)
    k = slice(warmup, None) if steps else slice(None)
    sa, bl = statistics.median(t_sa[k]), statistics.median(t_bl[k])
    t_epoch = (n / n_sub) * sa + bl
    return {"value": n * nx * ny / t_epoch, "unit": UNIT, "cores": workers, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{n_sub} of {n} rows x {nx * ny} nodes x {d} dims: search_accumulate "
                      f"({'SPARSE' if kern == O.SPARSE else 'DENSE_BLOCKED'}, {workers} workers) {sa:.2f} s + blend {bl:.2f} s per step, "
                      f"median of {len(t_sa[k])}; epoch = N/n_sub * search + blend",
            "seconds_per_step": t_epoch}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n, d, nx, ny, *_ , desc = CONFIGS[args.config]
    n_sub = args.ref_rows
    cb = cpu_reference_rate(args.config, n_sub, args.steps, args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": cb["seconds_per_step"] * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic uniform [0,1) fp32 (numpy default_rng seed 1001), bounded row sample",
            "config": {"workload": desc, "rows_sampled": n_sub, "K": nx * ny, "d": d},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    rank, world, local = init_dist(args)
    import paper_1305_1422_b200 as S
    from paper_1305_1422_b200 import _lib
    from paper_1305_1422_b200.engine import EngineOptions, SomEngine
    n, d, nx, ny, mt, grid, nbh, compact, desc = CONFIGS[args.config]
    K = nx * ny
    dev = torch.device("cuda", torch.cuda.current_device())
    first, count = S.partition(n, world)[rank]
    opts = EngineOptions(screen=args.screen, screen_passes=args.passes, rerank_order=not args.no_rerank_order)
    mtype, gtype, nb = S.MapType(mt), S.GridType(grid), S.Neighborhood(nbh)
    sparse = args.config == "cfg3"
    if sparse:
        from paper_1305_1422_b200.sparse import SparseEngine
        rp, cl, vl = sparse_rows_device(count, d, SPARSE_NNZ, 1001 + rank, dev)
        sdata = S.SparseDataset(d, rp.cpu().numpy(), cl.cpu().numpy(), vl.cpu().numpy())
        eng = SparseEngine(sdata, nx, ny, mtype, gtype, device=dev, options=opts)
        X = None
    else:
        # the reference generator's dataset (gen_random_dense(n, d, 1001)), this
        # rank's contiguous row partition, uploaded from pageable numpy
        Xnp = reference_rows(first, count, d)
        eng = SomEngine(S.DenseDataset(Xnp), nx, ny, mtype, gtype, device=dev, options=opts)
        X = None
    w0 = S.init_codebook(S.TrainConfig(n_columns=nx, n_rows=ny, seed=1), d).weights
    eng.set_codebook(w0)
    lib = _lib.load()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            if dist.get_backend() == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    for s in range(args.warmup):
        r, sc = schedule_for(args.config, s)
        eng.epoch(r, sc, 1e-3, nb, compact)
    torch.cuda.synchronize()
    barrier()
    eng.timing = {}
    clocks = ClockSampler(local)
    clocks.start()
    l0 = lib.somb_launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    in_bytes = count * SPARSE_NNZ * 8 if sparse else count * d * 4
    flush = in_bytes < L2_FLUSH_BYTES
    if not flush:   # inputs larger than L2: one event pair around all K steps
        t_start.record()
        for s in range(args.warmup, args.warmup + args.steps):
            r, sc = schedule_for(args.config, s)
            eng.epoch(r, sc, 1e-3, nb, compact)
        t_end.record()
        torch.cuda.synchronize()
        elapsed = t_start.elapsed_time(t_end) / 1e3
    else:           # inputs fit in L2: write a larger-than-L2 buffer between timed steps
        scratch = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        for i, s in enumerate(range(args.warmup, args.warmup + args.steps)):
            scratch.fill_(float(i))
            r, sc = schedule_for(args.config, s)
            ev[i][0].record()
            eng.epoch(r, sc, 1e-3, nb, compact)
            ev[i][1].record()
        torch.cuda.synchronize()
        elapsed = sum(a.elapsed_time(b) for a, b in ev) / 1e3
    barrier()
    launches = lib.somb_launch_count() - l0
    clk = clocks.stop()
    phase_ms = {k: [a.elapsed_time(b) for a, b in v] for k, v in eng.timing.items()}
    eng.timing = None
    tmax = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    elapsed = float(tmax.item())
    ms_step = elapsed * 1e3 / max(args.steps, 1)
    value = n * K / (elapsed / max(args.steps, 1))

    # roofline of the dominant kernel: the tcgen05 screen, algorithmic 2*n*K*d flops
    pk, pk_kind = peaks()
    scr = phase_ms.get("screen", [])
    scr_ms = statistics.mean(scr) if scr else float("nan")
    flops = 2.0 * count * K * d
    achieved = flops / (scr_ms / 1e3) / 1e12
    peak_sus = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    if sparse:   # gather-bound: unique bytes against HBM, gathered bytes and SIMT flops alongside
        gathered = float(count) * SPARSE_NNZ * eng.kp * 4
        unique = float(count) * SPARSE_NNZ * 8 + (count + 1) * 8 + float(d) * eng.kp * 4
        achieved_gbs = unique / (scr_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_screen_{args.config}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    passes = getattr(eng, "passes", 1)
    dpad = -(-d // 8) * 8
    kchunks = -(-dpad // 64) + (-(-2 * dpad // 128) if passes == 2 else 0)
    if passes in (1, 2) and kchunks <= 4:   # A-resident variant (screen_tc.cu g_ares)
        kname = ("screen_tc2a_kernel (tcgen05 cta_group::2, data-row operands resident in shared memory, "
                 + ("kind::f16" if passes == 1 else "fp16 kind::f16 + fp8 kind::f8f6f4 split screen") + ")")
    else:
        kname = {1: "screen_tc4_kernel (tcgen05 cta_group::2 kind::f16, 4-CTA clusters multicasting codebook tiles)",
                 2: "screen_tc2_kernel (tcgen05 cta_group::2, fp16 kind::f16 + fp8 kind::f8f6f4 split screen)",
                 3: "screen_tc2_kernel (tcgen05 cta_group::2 kind::f16, three-pass split screen)"}.get(passes, "screen_tc")
    roofline = {"bound": "tensor", "kernel": kname,
                "achieved": achieved, "peak": peak_sus, "unit": "TFLOP/s", "frac": achieved / peak_sus,
                "peak_kind": f"{pk_kind} bf16 dense sustained (fp16 kind::f16 runs at the bf16 rate)",
                "frac_of_burst": achieved / pk.get("bf16_tflops", peak_sus),
                "traffic": traffic, "flops_per_launch": flops, "avg_launch_ms": scr_ms,
                "mma_passes": getattr(eng, "passes", 1),
                "executed_tflops": achieved * getattr(eng, "passes", 1),
                "executed_frac": achieved * getattr(eng, "passes", 1) / peak_sus,
                "note": "achieved = algorithmic 2*n*K*d flops / screen time; the split screens for "
                        "d <= 128 execute mma_passes x that in fp16-equivalent tensor work (2: fp16 hi.hi "
                        "+ two fp8 cross terms at twice the rate; 3: three fp16 passes)"}
    if not sparse:
        # the epilogue reads every fp32 accumulator once from TMEM: 4*n*kp bytes
        # per launch against 64 B/clk/SM of tcgen05.ld bandwidth (B300_MICROARCH
        # TMEM table; same Blackwell SM) -- the floor that keeps the small-d
        # screens (cfg4/cfg5: 2048 TMEM-read clocks per 128x256 tile, as long
        # as the tile's MMAs) from the tensor peak
        sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
        tm_peak = 148 * 64 * sm_mhz * 1e6 / 1e9
        tm_bytes = 4.0 * count * eng.kp
        tm_gbs = tm_bytes / (scr_ms / 1e3) / 1e9
        roofline["tmem_read"] = {"bytes_per_launch": tm_bytes, "achieved": tm_gbs, "peak": tm_peak, "unit": "GB/s",
                                 "frac": tm_gbs / tm_peak,
                                 "peak_kind": "148 SMs x 64 B/clk (tcgen05.ld throughput) x max SM clock"}
        # serial floor: the tile's MMAs at the measured burst tensor rate PLUS
        # its accumulator reads at the TMEM read rate (outstanding tcgen05.ld
        # was measured to stall the MMAs: the two do not overlap)
        burst = pk.get("bf16_tflops", peak_sus)
        t_mma = flops * passes / (burst * 1e12)
        t_tm = tm_bytes / (tm_peak * 1e9)
        roofline["mma_plus_tmem_floor"] = {"floor_ms": (t_mma + t_tm) * 1e3, "mma_ms": t_mma * 1e3,
                                           "tmem_read_ms": t_tm * 1e3, "frac": (t_mma + t_tm) * 1e3 / scr_ms,
                                           "note": "executed tensor work at the measured burst bf16 rate plus "
                                                   "4*n*kp accumulator bytes at 64 B/clk/SM, serialised"}
    if sparse:
        simt_peak = 148 * 128 * 2 * 1.965e9 / 1e12
        gflops = 2.0 * count * SPARSE_NNZ * K / (scr_ms / 1e3) / 1e12
        roofline = {"bound": "hbm", "kernel": "sp_screen_ls_kernel (fp32 slab-lockstep gather over the transposed codebook)",
                    "achieved": achieved_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": achieved_gbs / pk["hbm_gbs"], "traffic": traffic,
                    "bytes_per_launch": unique, "avg_launch_ms": scr_ms,
                    "gather": {"bytes_per_launch": gathered, "GBps": gathered / (scr_ms / 1e3) / 1e9,
                               "simt_tflops": gflops, "simt_peak_tflops": simt_peak,
                               "simt_frac": gflops / simt_peak},
                    "note": "algorithmic bytes = CSR rows + transposed codebook read once; the kernel "
                            "gathers nnz x kp fp32 codebook values (mostly L2 hits): it is bound by "
                            "the L2 gather rate, far above the HBM floor"}

    # per-phase breakdown (rank-local averages)
    phases = {k: statistics.mean(v) for k, v in phase_ms.items() if v}
    eng.search()     # untimed: the candidate lists live in the workspace until node_sums reuses it
    cc = eng.candidate_counts()[: eng.n].float().cpu().numpy() if eng.n else np.zeros(1)
    cand_stats = {"mean": float(cc.mean()), "p50": float(np.median(cc)), "p99": float(np.percentile(cc, 99)),
                  "max": float(cc.max())}
    # the other phases against their HBM floors (algorithmic bytes per epoch / phase time)
    hbm = pk["hbm_gbs"]

    def hbm_line(name, nbytes, what):
        t = phases.get(name)
        if not t:
            return None
        gbs = nbytes / (t / 1e3) / 1e9
        return {"bound": "hbm", "bytes_per_launch": nbytes, "avg_ms": t, "achieved": gbs, "peak": hbm,
                "unit": "GB/s", "frac": gbs / hbm, "bytes": what}
    xb = float(count) * SPARSE_NNZ * 8 if sparse else float(count) * d * 4
    phase_roofline = {
        "rerank": hbm_line("rerank", xb + float(count) * 12,
                           "data rows once + BMU/d2min out; the candidate codebook rows (candidates_per_row x "
                           "4d bytes per row) are L2 reads on top"),
        "node_sums": hbm_line("node_sums", xb + float(count) * 12 + float(K) * d * 8,
                              "data rows once + BMUs/row order + fp64 node sums S out (radix sort + seg_sum)"),
        "update": hbm_line("update", float(K) * d * (8 + 4 + 4),
                           "fp64 node sums in, codebook in and out (spectral DMMA convolution + blend); the "
                           "DFT planes stay in L2"),
    }
    l2_gbs = measure_l2_gbs(dev)
    if not sparse and phases.get("rerank"):
        l2b = float(count) * cand_stats["mean"] * d * 4
        phase_roofline["rerank"]["l2_candidate_bytes"] = l2b
        phase_roofline["rerank"]["l2_candidate_GBps"] = l2b / (phases["rerank"] / 1e3) / 1e9
        phase_roofline["rerank"]["l2_frac"] = phase_roofline["rerank"]["l2_candidate_GBps"] / l2_gbs
    if sparse:
        roofline["gather"]["l2_read_gbs_measured"] = l2_gbs
        roofline["gather"]["l2_frac"] = roofline["gather"]["GBps"] / l2_gbs
    flags = eng.flags[: eng.n].cpu().numpy()
    trunc = float((((flags & 0xFF) | ((flags >> 8) & 0xFF) | ((flags >> 16) & 0xFF) | ((flags >> 24) & 0xFF)) & 1).astype(bool).mean()) if eng.n else 0.0
    spilled = float((((flags & 0xFF) | ((flags >> 8) & 0xFF) | ((flags >> 16) & 0xFF) | ((flags >> 24) & 0xFF)) & 2).astype(bool).mean()) if eng.n else 0.0

    # end to end through the public API: host (pinned) data -> train() -> host results
    e2e = None
    if not args.no_e2e:
        # the drop-in input type: a DenseDataset over a pageable numpy array
        # (or the SparseDataset of numpy CSR arrays), as a reference user passes it
        data = sdata if sparse else S.DenseDataset(Xnp)
        del eng
        torch.cuda.empty_cache()
        kern = S.Kernel.SPARSE if sparse else S.Kernel.DENSE_BLOCKED
        cfg = S.TrainConfig(n_epochs=args.e2e_epochs, n_columns=nx, n_rows=ny, map_type=mtype,
                            kernel=kern, grid=gtype, neighborhood=nb, compact_support=compact, seed=1)
        S.train(data, S.TrainConfig(n_epochs=1, n_columns=nx, n_rows=ny, map_type=mtype, kernel=kern,
                                    grid=gtype, neighborhood=nb, compact_support=compact),
                options=opts, local_rows=True)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        cb, bmus, u = S.train(data, cfg, options=opts, local_rows=True)
        torch.cuda.synchronize()
        barrier()
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            import torch.distributed as dist
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        te = float(te.item())
        e2e = {"value": n * K * args.e2e_epochs / te, "unit": UNIT,
               "h2d_bytes_per_step": int(count * SPARSE_NNZ * 8 + (count + 1) * 8 if sparse else count * d * 4),
               "d2h_bytes_per_step": int(K * d * 4 + n * 2 * 4 + K * 4),
               "step": f"one public train() call: H2D of the rank's rows from a pageable numpy array, seeded "
                       f"codebook init (on device, numpy-identical), {args.e2e_epochs} epochs, final naive "
                       f"BMU pass, U-matrix, D2H of codebook + BMU table + U-matrix",
               "seconds": te}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference_rate(args.config, args.ref_rows, 3, 1)
        cpu.pop("seconds_per_step", None)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": ("fp32 gather screen + f64 exact re-rank/update" if sparse else
                          {1: "fp16", 2: "fp16 + fp8 split", 3: "fp16 three-pass split"}.get(passes, "fp16")
                          + " tensor-core screen (fp32 accumulate) + f64 exact re-rank/update"),
                "data": ("synthetic text-like CSR (torch.Generator seed 1001+rank), codebook init default_rng(1)"
                         if sparse else "synthetic uniform [0,1) fp32: the reference generator "
                         "gen_random_dense(n, d, seed=1001) (numpy PCG64), rank r its partition rows; codebook "
                         "init default_rng(1)"),
                "config": {"workload": desc, "rows": n, "K": K, "d": d,
                           "schedule": f"{N_EPOCHS}-epoch linear radius {max(min(nx, ny) / 2, 1)}->1, "
                                       f"scale 1->0.01; step s = epoch s mod {N_EPOCHS}",
                           "parallelism": f"dp{world} (rows sharded; per epoch 1 fp64 reduce-scatter of the "
                                          f"node sums by feature columns, 1 small all-reduce, 1 fp32 all-gather "
                                          f"of the updated column blocks)",
                           "l2": (f"L2 flushed between timed steps (inputs {in_bytes / 1e6:.0f} MB per GPU, "
                                  f"{L2_FLUSH_BYTES >> 20} MiB buffer written)") if flush else
                                 f"inputs larger than L2 ({in_bytes / 1e9:.2f} GB per GPU)",
                           "screen": args.screen},
                "roofline": roofline, "cpu_baseline": cpu, "clocks": clk, "e2e": e2e,
                "gpu_launches": int(launches),
                "phase_ms": phases, "phase_roofline": phase_roofline, "l2_read_gbs_measured": l2_gbs,
                "epoch_ms": ms_step,
                "nkd_per_s": value * d, "window_truncated_rows": trunc, "window_spilled_rows": spilled,
                "candidates_per_row": cand_stats}
        emit(line)
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        barrier()
        dist.destroy_process_group()
    return 0


_JSON_FD = None


def emit(line):
    """The one JSON line of the contract, on the real stdout."""
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def _quiet_stdout():
    """Route everything else written to fd 1 (NCCL's version banner, library
    prints) to stderr, so stdout carries exactly the one JSON line."""
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--screen", default="tensor", choices=["tensor", "simt", "exact"])
    ap.add_argument("--e2e-epochs", type=int, default=10)
    ap.add_argument("--ref-rows", type=int, default=0, help="CPU sample rows (0: per-config default)")
    ap.add_argument("--passes", type=int, default=0, choices=[0, 1, 2, 3],
                    help="screen passes (0: auto = 2 (fp16 + fp8 cross terms) for d <= 128)")
    ap.add_argument("--no-rerank-order", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    _quiet_stdout()
    if args.ref_rows == 0:
        args.ref_rows = {"cfg3": 256, "cfg5": 512, "cfg4": 1024, "cfg1": 10000}.get(args.config, 4096)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
