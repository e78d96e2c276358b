"""Device-resident epoch engine: one process per GPU, all epoch work on the
stream, one fp64 NCCL all-reduce per epoch when the rows are sharded.

Per epoch:
  somb_codebook_prepare -> somb_bmu_dense (tcgen05 screen + fp64 re-rank)
  -> somb_qe_sum -> somb_node_sums_dense -> [all_reduce(S | cnt | qe)]
  -> somb_hood_update (fp64 convolution + blend, this rank's node slice)
  -> [all_gather(W)].
This replaces the reference epoch loop body train.py:269-277 (search_accumulate
kernels.py:365-435 + blend kernels.py:438-450) and the coordinator/worker fold
distributed.py:492-514 (rank-ordered fp64 merge -> NCCL fp64 sum).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib, errors
from .datasets import DenseDataset, SparseDataset, _is_torch
from .grid import GridType, MapType, Neighborhood, distance_table

# Screening windows, in units of the per-row sigma_i of the stochastically
# rounded fp16 operands (csrc/cand.cuh screen_sigma): the
# window of row i is kappa * sigma_i.  Calibrated on hardware over uniform,
# duplicated-column, near-constant, blob, one-hot, integer, offset and
# low-rank data (tools/calib_screen.py, profiles/r2_window_calib_*.json).
_DEF_WINDOW_KAPPA = float(os.environ.get("SOMB_WINDOW_KAPPA", "5.0"))     # 1-pass fp16
_DEF_WINDOW_KAPPA2 = float(os.environ.get("SOMB_WINDOW_KAPPA2", "0.5"))   # fp16 + fp8 cross terms
_U16 = 2.0 ** -11
# 3-pass split screen (hi.hi + hi.lo + lo.hi, round-to-nearest): its error is
# dominated by fp32 accumulation, measured max ~ D/8192 in units of
# 2^-11 |x'| max|delta| / sqrt(D) (tools/calib_screen.py: 0.01 / 0.03 / 0.09
# at D = 128 / 256 / 1000); the window is 2.6x that + 0.02 (somb_data_pack
# encodes that unit as the row's sigma for the 3-pass operands).
def _kappa3(d: int) -> float:
    return 2.6 * d / 8192.0 + 0.02


@dataclass
class EngineOptions:
    screen: str = "tensor"            # "tensor" (tcgen05), "simt" (reference screen), "exact"
    window_kappa: float = _DEF_WINDOW_KAPPA
    hypot_table: bool = True          # numpy-hypot distances for rect grids (bit parity)
    seed_prev: bool = True            # seed the screen threshold from the previous BMUs
    screen_passes: int = 0            # 0 auto (2 if the padded feature count <= 128), 1, 2 (fp16 + fp8 cross terms) or 3
    window_kappa3: Optional[float] = None     # None: _kappa3(d)
    window_kappa2: float = _DEF_WINDOW_KAPPA2   # 2-pass (fp16 + fp8 cross terms) window, sigma units
    conv: str = "auto"                # neighbourhood convolution: "auto", "direct", "spectral"
    rerank_order: bool = True         # re-rank rows in previous-BMU order (L2 locality; same result)
    shard_update: str = "columns"     # multi-rank update: "columns" (reduce-scatter S by feature columns,
                                      # each rank updates its columns for all nodes) or "nodes" (all-reduce S,
                                      # node-slice update, row all-gather)
    exchange: str = os.environ.get("SOMB_EXCHANGE", "auto")   # "auto": collectives only when world > 1;
                                      # "always": run the sharded exchange (NCCL) even in a 1-rank group
                                      # (tests the NCCL data plane and times it on one GPU)


def _ptr(t: Optional[torch.Tensor]):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _stream(dev: torch.device):
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _round_up(v: int, a: int) -> int:
    return (v + a - 1) // a * a


_STAGE = {}   # (device index, slot, thread) -> two cached page-locked staging halves
_STAGE_EVENTS = {}   # same key -> the events of the last copies that read each upload half


def to_host(t: torch.Tensor, slot: str = "main") -> np.ndarray:
    """Device -> host copy through two cached page-locked staging buffers: the
    D2H of chunk i+1 overlaps the host copy of chunk i (a pageable copy of the
    160 MB cfg2 codebook runs at ~2 GB/s, and pinning a fresh buffer per call
    costs more than the copy)."""
    t = t.contiguous()
    out = np.empty(tuple(t.shape), dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
    nbytes = t.numel() * t.element_size()
    if nbytes == 0:
        return out
    chunk = 16 << 20
    dev = t.device.index if t.device.index is not None else torch.cuda.current_device()
    key = (dev, slot, threading.get_ident())
    bufs = _STAGE.get(key)
    if bufs is None:   # one staging pair per (device, slot, thread): concurrent copies never share one
        bufs = _STAGE[key] = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    src = t.view(-1).view(torch.uint8)
    dst = out.reshape(-1).view(np.uint8)
    stream = torch.cuda.current_stream(t.device)
    events = [None, None]
    offs = list(range(0, nbytes, chunk))
    for i, o in enumerate(offs + [None]):
        if o is not None:   # enqueue D2H of chunk i into half i % 2
            m = min(chunk, nbytes - o)
            bufs[i % 2][:m].copy_(src[o:o + m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            events[i % 2] = ev
        if i > 0:           # host copy of chunk i - 1 while chunk i is in flight
            p = offs[i - 1]
            m = min(chunk, nbytes - p)
            events[(i - 1) % 2].synchronize()
            _host_copy(dst.ctypes.data + p, bufs[(i - 1) % 2].data_ptr(), m)
    return out


def to_device(a: np.ndarray, dev) -> torch.Tensor:
    """Host (pageable numpy) -> device copy through two cached page-locked
    staging chunks: the threaded host copy of chunk i+1 overlaps the H2D of
    chunk i, instead of pinning a full-size copy of the array first."""
    a = np.ascontiguousarray(a)
    out = torch.empty(a.shape, dtype=torch.from_numpy(np.empty(0, a.dtype)).dtype, device=dev)
    nbytes = a.nbytes
    if nbytes < (8 << 20):
        return out.copy_(torch.from_numpy(a)) if nbytes else out
    chunk = _UP_CHUNK
    key = (out.device.index, "up", threading.get_ident())
    bufs = _STAGE.get(key)
    if bufs is None:
        bufs = _STAGE[key] = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    src = a.reshape(-1).view(np.uint8)
    dst = out.view(-1).view(torch.uint8)
    stream = torch.cuda.current_stream(out.device)
    # the last H2D of the previous call may still be reading a half: its
    # events persist with the buffers (a back-to-back upload -- the CSR cols
    # then vals -- must not overwrite a half that is still in flight)
    events = _STAGE_EVENTS.setdefault(key, [None, None])
    for i, o in enumerate(range(0, nbytes, chunk)):
        b = bufs[i % 2]
        if events[i % 2] is not None:
            events[i % 2].synchronize()   # the H2D that last read this half is done
        m = min(chunk, nbytes - o)
        _host_copy(b.data_ptr(), src.ctypes.data + o, m)
        dst[o:o + m].copy_(b[:m], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        events[i % 2] = ev
    return out


_POOL = None
_D2H_POOL = None


# upload staging chunk and host-copy threads (SOMB_STAGE_CHUNK_MB / SOMB_HOST_COPY_THREADS, tools/upload_probe.py)
_UP_CHUNK = int(os.environ.get("SOMB_STAGE_CHUNK_MB", "32")) << 20
_COPY_THREADS = int(os.environ.get("SOMB_HOST_COPY_THREADS", "8"))   # 4 GB pageable upload: 146 ms at 4 threads, 102 ms at 8


def _host_copy(dst: int, src: int, nbytes: int, parts: int = 0) -> None:
    """memcpy split over threads (ctypes.memmove releases the GIL)."""
    global _POOL
    parts = parts or _COPY_THREADS
    if nbytes < (4 << 20):
        C.memmove(dst, src, nbytes)
        return
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(parts)
    step = -(-nbytes // parts)
    futs = [_POOL.submit(C.memmove, dst + o, src + o, min(step, nbytes - o)) for o in range(0, nbytes, step)]
    for f in futs:
        f.result()


def pick_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise errors.DeviceError("no CUDA device: somb200 runs only on a B200 (sm_100a)")
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise errors.DeviceError(f"somb200 needs a CUDA device, got {device}")
    idx = device.index if device.index is not None else torch.cuda.current_device()
    _lib.require_device(idx)
    return torch.device("cuda", idx)


def _dist_ready() -> bool:
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized()


def dist_info(group=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


class SomEngine:
    """Resident dataset slice + codebook + buffers for one GPU (one rank)."""

    _sparse = False   # SparseEngine: CSR rows, gather screen (larger BMU workspace)

    def __init__(self, data, n_columns: int, n_rows: int, map_type: MapType,
                 grid: GridType = GridType.RECTANGULAR, device=None, group=None,
                 options: Optional[EngineOptions] = None):
        self.dev = pick_device(device)
        self.opt = options or EngineOptions()
        self.group = group
        self.rank, self.world = dist_info(group)
        # the per-epoch exchange runs when the rows are sharded, or on demand
        # in a 1-rank process group (EngineOptions.exchange = "always")
        self.sharded = self.world > 1 or (self.opt.exchange == "always" and _dist_ready())
        self.nx, self.ny = int(n_columns), int(n_rows)
        self.K = self.nx * self.ny
        self.map_type, self.grid = map_type, grid
        self.cmap = _lib.SombMap(self.nx, self.ny,
                                 _lib.GRID_HEX if grid is GridType.HEXAGONAL else _lib.GRID_RECT,
                                 _lib.TOROID if map_type is MapType.TOROID else _lib.PLANAR)
        self._init_data(data)
        d = self.d
        self.dp = _round_up(d, 8)
        self.kp = _round_up(self.K, 256)
        # node slice of this rank for the update; K padded so all_gather chunks are equal
        self.kc = -(-self.K // self.world)
        self.kpad = self.kc * self.world
        self.node_begin = min(self.K, self.rank * self.kc)
        self.node_end = min(self.K, (self.rank + 1) * self.kc)
        f32, f64, dev = torch.float32, torch.float64, self.dev
        self.W = torch.zeros((self.kpad, d), dtype=f32, device=dev)
        self.W2 = torch.zeros((self.kpad, d), dtype=f32, device=dev)
        self._init_codebook_buffers()
        self.c = torch.empty(self.kp, dtype=f32, device=dev)
        self.w2 = torch.empty(self.K, dtype=f64, device=dev)
        self.scal = torch.zeros(8, dtype=f32, device=dev)
        n = self.n
        self.bmu = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.d2min = torch.empty(max(n, 1), dtype=f64, device=dev)
        self.flags = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        # rows sorted by BMU (written by node_sums): the next re-rank visits rows
        # in this order so concurrently re-ranked rows share codebook rows in L2
        self.row_order = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        self.has_order = False
        # packed [S | cnt (K) | qe (1)] fp64.  S is [K, d], or with the
        # column-sharded exchange column-block-major [P, K, dc] (dc = ceil(d/P),
        # blocks past the last column stay zero): the node-sum kernels write
        # each rank's column block contiguously, so S is reduce-scattered in
        # place, without a restaging copy
        self.cols = self.sharded and self.opt.shard_update == "columns"
        self.dc = -(-d // self.world) if self.cols else d
        ssz = self.world * self.K * self.dc if self.cols else self.K * d
        self.acc = torch.zeros(ssz + self.K + 1, dtype=f64, device=dev)
        self.S = (self.acc[:ssz].view(self.world, self.K, self.dc) if self.cols
                  else self.acc[:ssz].view(self.K, d))
        self.cnt = self.acc[ssz: ssz + self.K]
        self.qe = self.acc[ssz + self.K:]
        self.dist_tab = None
        if self.opt.hypot_table and grid is GridType.RECTANGULAR:
            self.dist_tab = torch.from_numpy(distance_table(self.nx, self.ny, map_type)).to(dev)
        lib = _lib.load()
        ws = max(lib.somb_codebook_ws(self.K, d),
                 lib.somb_bmu_sparse_ws(n) if self._sparse else lib.somb_bmu_ws(n),
                 lib.somb_node_sums_ws(n, d, self.K),
                 lib.somb_hood_ws(C.byref(self.cmap), self.K, d), 1 << 16)
        self.ws = torch.empty(int(ws), dtype=torch.uint8, device=dev)
        self.window_coef = self._window_coef()
        self.screen_impl = {"tensor": 0, "simt": 1, "exact": 2}[self.opt.screen]
        if self.screen_impl == 0 and self.passes == 2:
            self.screen_impl = 3       # tcgen05 fp16 + fp8 cross-term split screen
        self.has_prev = False

    # ------------------------------------------------------- subclass hooks
    def _init_data(self, data):
        if isinstance(data, SparseDataset):
            raise errors.KernelDataMismatch("SomEngine(dense): got sparse data")
        x = data.values if isinstance(data, DenseDataset) else data
        self._upload_dense(x, dry=True)
        dp0 = _round_up(self.d, 8)
        p = self.opt.screen_passes
        if self.opt.screen != "tensor":
            self.passes = 1
        elif p in (1, 2, 3):
            self.passes = p
        else:
            self._adaptive = dp0 <= 256   # may switch to the split screen (search)
            # split screen only where the 1-pass window holds too many near
            # ties: cfg5 (d = 128, K = 250k) keeps ~360 nodes per row in the
            # 1-pass window (rows truncate, full-scan repairs: 44 s per
            # epoch) against 13 with the fp8 split; at cfg4 (d = 256,
            # K = 90k) the 1-pass screen is the faster one (137 vs 146 ms per
            # epoch, 23 candidates per row) -- tools/r2_p1.sh
            self.passes = 2 if dp0 <= 128 else 1
        self.pack_dataset()

    def _init_codebook_buffers(self):
        self.Wh = torch.empty((self.kp, self.dp), dtype=torch.float16, device=self.dev)
        if self.passes == 3:
            self.Wl = torch.empty((self.kp, self.dp), dtype=torch.float16, device=self.dev)
        elif self.passes == 2:     # fp8 cross operands [w_lo8 | w_hi8]
            self.Wl = torch.empty((self.kp, 2 * self.dp), dtype=torch.uint8, device=self.dev)
        else:
            self.Wl = None

    def _window_coef(self) -> float:
        if self.passes == 3:
            kappa = self.opt.window_kappa3 if self.opt.window_kappa3 is not None else _kappa3(self.d)
        elif self.passes == 2:
            kappa = self.opt.window_kappa2
        else:
            kappa = self.opt.window_kappa
        return float(kappa)

    # ------------------------------------------------------------ dataset
    def _upload_dense(self, x, dry=False):
        if _is_torch(x):
            xt = x.to(self.dev, dtype=torch.float32, non_blocking=True).contiguous()
        else:   # pageable numpy rows: chunked through cached pinned staging
            xt = to_device(np.ascontiguousarray(x, dtype=np.float32), self.dev)
        self.X = xt
        self.n, self.d = int(xt.shape[0]), int(xt.shape[1])
        if not dry:
            self.pack_dataset()

    def pack_dataset(self):
        """Centre + fp16 copy of the resident rows (once per dataset)."""
        lib, dev, st = _lib.load(), self.dev, _stream(self.dev)
        d, n = self.d, self.n
        self.dp = _round_up(d, 8)
        self.nu = torch.empty(d, dtype=torch.float32, device=dev)
        absmax = torch.empty(1, dtype=torch.float32, device=dev)
        ws = torch.empty(int(lib.somb_data_stats_ws(d)), dtype=torch.uint8, device=dev)
        _lib.call("somb_data_stats", _ptr(self.X), n, d, _ptr(self.nu), _ptr(absmax), _ptr(ws), st)
        a = float(absmax.item())                 # one host sync per dataset
        passes = getattr(self, "passes", 1)
        top = 13 if passes == 2 else 14          # the fp8 cross operands need max|hi| <= 2^13
        self.xexp = 0 if a <= 0.0 or not math.isfinite(a) else top - math.frexp(a)[1]
        self.Xh = torch.empty((max(n, 1), self.dp), dtype=torch.float16, device=dev)
        self.Xl = None
        if passes == 3:
            self.Xl = torch.empty((max(n, 1), self.dp), dtype=torch.float16, device=dev)
        elif passes == 2:
            self.Xl = torch.empty((max(n, 1), 2 * self.dp), dtype=torch.uint8, device=dev)
        self.xnorm = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        self.x2 = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        # per-row window terms {|x'|, max|x'_k|, max ulp_k, |ulp|_2} (cand.cuh screen_sigma)
        self.xstat = torch.empty((max(n, 1), 4), dtype=torch.float32, device=dev)
        _lib.call("somb_data_pack_f8" if passes == 2 else "somb_data_pack", _ptr(self.X), n, d, _ptr(self.nu),
                  self.xexp, _ptr(self.Xh), _ptr(self.Xl), self.dp, _ptr(self.xnorm), _ptr(self.x2),
                  _ptr(self.xstat), st)

    # ----------------------------------------------------------- codebook
    def set_codebook(self, w):
        w = torch.as_tensor(w, dtype=torch.float32)
        if tuple(w.shape) != (self.K, self.d):
            raise errors.CodebookShapeMismatch(f"codebook {tuple(w.shape)}, expected {(self.K, self.d)}")
        self.W[: self.K].copy_(w.to(self.dev, non_blocking=True))

    def init_codebook_device(self, seed: int):
        """W = numpy.random.default_rng(seed).random((K, d), float32), generated
        on the device bit for bit (train.py:164-166; somb_uniform_f32)."""
        st = np.random.PCG64(seed).state["state"]
        s, inc, m64 = int(st["state"]), int(st["inc"]), (1 << 64) - 1
        _lib.call("somb_uniform_f32", s >> 64, s & m64, inc >> 64, inc & m64, self.K * self.d, _ptr(self.W),
                  _stream(self.dev))

    def codebook(self) -> np.ndarray:
        return to_host(self.W[: self.K])

    def codebook_async(self):
        """Future of codebook(): the D2H runs on a side stream (ordered after
        the work enqueued so far) from a helper thread, so it overlaps what
        the caller enqueues next -- train() overlaps it with the final BMU
        pass.  The codebook must not be updated until the future resolves."""
        global _D2H_POOL
        if _D2H_POOL is None:
            from concurrent.futures import ThreadPoolExecutor
            _D2H_POOL = ThreadPoolExecutor(1)
        if self._side is None:
            self._side = torch.cuda.Stream(self.dev)
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(self.dev))
        W, K, dev, side = self.W, self.K, self.dev, self._side

        def work():
            with torch.cuda.device(dev), torch.cuda.stream(side):
                side.wait_event(ready)
                return to_host(W[:K], slot="side")
        return _D2H_POOL.submit(work)

    # ------------------------------------------------------------- phases
    def prepare(self):
        _lib.call("somb_codebook_prepare_f8" if self.passes == 2 else "somb_codebook_prepare", _ptr(self.W),
                  self.K, self.d, _ptr(self.nu), self.xexp,
                  _ptr(self.Wh), _ptr(self.Wl), self.dp, self.kp, _ptr(self.c), _ptr(self.w2),
                  _ptr(self.scal), _ptr(self.ws), _stream(self.dev))

    # optional per-phase CUDA-event timing (bench.py): name -> [(start, end), ...]
    timing = None
    _side = None   # side stream of codebook_async (created on first use)

    def _mark(self, name, start):
        if self.timing is None:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.current_stream(self.dev))
        if start:
            self.timing.setdefault(name, []).append([ev, None])
        else:
            self.timing[name][-1][1] = ev

    def search(self, dist_mode=_lib.DIST_BLOCKED):
        """BMU + d2min for the resident rows against the current codebook."""
        self._mark("prepare", True)
        self.prepare()
        self._mark("prepare", False)
        if self.n == 0:
            return
        st = _stream(self.dev)
        self._mark("screen", True)
        prev = self.bmu if (self.has_prev and self.opt.seed_prev) else None
        _lib.call("somb_bmu_screen", _ptr(self.Xh), _ptr(self.Xl), _ptr(self.xstat), self.n, self.dp,
                  _ptr(self.Wh), _ptr(self.Wl), _ptr(self.c), self.K, self.kp, _ptr(self.scal),
                  C.c_float(self.window_coef),
                  _ptr(prev), self.screen_impl, _ptr(self.flags), _ptr(self.ws), st)
        self._mark("screen", False)
        self._mark("rerank", True)
        order = _ptr(self.row_order if (self.has_order and self.opt.rerank_order) else None)
        _lib.call("somb_bmu_rerank", _ptr(self.X), _ptr(self.x2), self.n, self.d, _ptr(self.W),
                  _ptr(self.w2), self.K, dist_mode, self.screen_impl, order, _ptr(self.bmu),
                  _ptr(self.d2min), _ptr(self.flags), _ptr(self.ws), st)
        self._mark("rerank", False)
        self.has_prev = True
        if self._adaptive and self.passes == 1 and self.screen_impl == 0:
            # Auto mode, 128 < dp <= 256: the 1-pass screen is the faster one
            # on spread data, but structured data (near-constant rows, a large
            # mean offset) can keep hundreds of nodes inside its window, so
            # rows truncate and are repaired by full scans (exact, but slow:
            # cfg4 near-constant rows, 50% of the rows per epoch).  Then the
            # fp16 + fp8 split screen takes over for the rest of the training.
            # Also when the sets stay complete but large: more spilled
            # 32-entry chunks than half the rows (uniform cfg4 data spills
            # ~0.05 per row).  Two 4-byte host reads per epoch.
            rep = self.repaired_rows()
            if rep > 0.005 * self.n or self.overflow_chunks() > self.n // 2:
                self._switch_to_split()

    _adaptive = False

    def _switch_to_split(self):
        """1-pass -> 2-pass (fp16 + fp8 cross terms) screen from the next
        search on: re-pack the rows with the fp8 cross operands, allocate the
        codebook's, switch the window."""
        self.passes = 2
        self.pack_dataset()
        self._init_codebook_buffers()
        self.window_coef = self._window_coef()
        self.screen_impl = 3
        self.switched_to_split = True

    def debug_screen_values(self) -> torch.Tensor:
        """tcgen05 screened values r~ of rows [0, 128) x all nodes (calibration)."""
        self.prepare()
        m = min(self.n, 128)
        dump = torch.full((m, self.kp), float("nan"), dtype=torch.float32, device=self.dev)
        _lib.call("somb_debug_screen_dump", _ptr(self.Xh), _ptr(self.Xl), _ptr(self.xstat), self.n,
                  self.dp, _ptr(self.Wh), _ptr(self.Wl), _ptr(self.c), self.kp, _ptr(self.scal),
                  C.c_float(self.window_coef), self.passes,
                  _ptr(dump), _ptr(self.ws), _stream(self.dev))
        return dump[:, : self.K]

    def candidate_counts(self) -> torch.Tensor:
        """Per-row candidate counts of the last screen (tcgen05 two-half encoding)."""
        off = ((self.n * _lib.CAND_CAP * 4 + 255) // 256) * 256
        cc = self.ws[off: off + 4 * self.n].view(torch.int32)
        if self.screen_impl in (0, 3):   # one count byte per column group (2 or 4 groups)
            return (cc & 255) + ((cc >> 8) & 255) + ((cc >> 16) & 255) + ((cc >> 24) & 255)
        return cc

    def repaired_rows(self) -> int:
        """Rows of the last screen whose truncated candidate set was replaced
        by an exact scan of every node (host sync)."""
        return int(_lib.load().somb_bmu_repaired_rows(_ptr(self.ws), self.n, _stream(self.dev)))

    def overflow_chunks(self) -> int:
        """Overflow chunks the last tcgen05 screen spilled (bmu.cu workspace counters)."""
        a = lambda b: (b + 255) // 256 * 256
        off = a(self.n * _lib.CAND_CAP * 4) + 2 * a(self.n * 4)
        return int(self.ws[off + 4: off + 8].view(torch.int32).item())

    def qe_sum(self):
        _lib.call("somb_qe_sum", _ptr(self.d2min), self.n, _ptr(self.qe), _ptr(self.ws),
                  _stream(self.dev))

    def node_sums(self):
        _lib.call("somb_node_sums_dense_cols", _ptr(self.X), self.n, self.d, _ptr(self.bmu), self.K, self.dc,
                  _ptr(self.S), _ptr(self.cnt), _ptr(self.row_order), _ptr(self.ws), _stream(self.dev))
        self.has_order = True

    def _col_buffers(self):
        """Staging for the column-sharded exchange (allocated on first use)."""
        if getattr(self, "_Sr", None) is None:
            dc, K, P, dev = self.dc, self.K, self.world, self.dev
            self._Sr = torch.empty((K, dc), dtype=torch.float64, device=dev)
            self._Wst = torch.empty((P, K, dc), dtype=torch.float32, device=dev)
            self._Wold = torch.zeros((K, dc), dtype=torch.float32, device=dev)
            self._Wnew = torch.empty((K, dc), dtype=torch.float32, device=dev)

    def reduce(self):
        if self.sharded:
            from .parallel import allreduce_sum, reduce_scatter_blocks
            if self.cols:
                # this rank's feature columns of S, summed over ranks; the
                # counts and qe (the contiguous tail of acc) on every rank
                self._col_buffers()
                reduce_scatter_blocks(self.S, self._Sr, self.group)
                allreduce_sum(self.acc[self.S.numel():], self.group)
            else:
                allreduce_sum(self.acc, self.group)

    def update(self, radius, scale, cutoff, neighborhood=Neighborhood.GAUSSIAN, compact=False,
               num_out=None, den_out=None, all_nodes=False):
        hood = _lib.SombHood(_lib.NBH_BUBBLE if neighborhood is Neighborhood.BUBBLE
                             else _lib.NBH_GAUSSIAN, int(bool(compact)), float(radius), float(cutoff),
                             {"auto": 0, "direct": 1, "spectral": 2}[self.opt.conv], 0)
        if self.cols and not all_nodes:
            # all nodes, this rank's columns: the update is independent per
            # feature column, so each column is computed exactly as on one GPU
            from .parallel import allgather_columns
            self._col_buffers()
            a, b = min(self.d, self.rank * self.dc), min(self.d, (self.rank + 1) * self.dc)
            if b > a:
                self._Wold[:, : b - a].copy_(self.W[: self.K, a:b])
            _lib.call("somb_hood_update", _ptr(self._Sr), _ptr(self.cnt), self.dc, C.byref(self.cmap),
                      C.byref(hood), C.c_double(scale), _ptr(self.dist_tab), _ptr(self._Wold), 0, self.K,
                      _ptr(self._Wnew), None, None, _ptr(self.ws), _stream(self.dev))
            allgather_columns(self._Wnew, self._Wst, self.W2[: self.K], self.d, self.group)
            self.W, self.W2 = self.W2, self.W
            return
        nb, ne = (0, self.K) if all_nodes else (self.node_begin, self.node_end)
        S = self.S
        if self.cols:   # column blocks -> [K, d] (the all-nodes update of the functional API)
            S = S.permute(1, 0, 2).reshape(self.K, -1)[:, : self.d].contiguous()
        _lib.call("somb_hood_update", _ptr(S), _ptr(self.cnt), self.d, C.byref(self.cmap),
                  C.byref(hood), C.c_double(scale), _ptr(self.dist_tab), _ptr(self.W), nb, ne,
                  _ptr(self.W2), _ptr(num_out), _ptr(den_out), _ptr(self.ws), _stream(self.dev))
        if self.sharded and not all_nodes:
            from .parallel import allgather_rows
            allgather_rows(self.W2, self.kc, self.group)
        self.W, self.W2 = self.W2, self.W

    def epoch(self, radius, scale, cutoff, neighborhood=Neighborhood.GAUSSIAN, compact=False):
        """One full training epoch; returns the device qe-sum tensor (no sync)."""
        self.search(_lib.DIST_BLOCKED)
        self._mark("node_sums", True)
        self.qe_sum()
        self.node_sums()
        self._mark("node_sums", False)
        self._mark("allreduce", True)
        self.reduce()
        self._mark("allreduce", False)
        self._mark("update", True)
        self.update(radius, scale, cutoff, neighborhood, compact)
        self._mark("update", False)
        return self.qe

    def umatrix(self) -> torch.Tensor:
        u = torch.empty(self.K, dtype=torch.float32, device=self.dev)
        _lib.call("somb_umatrix", _ptr(self.W), self.d, C.byref(self.cmap), _ptr(u),
                  _stream(self.dev))
        return u.view(self.ny, self.nx)

    def global_rows(self) -> int:
        if self.world == 1:
            return self.n
        import torch.distributed as dist
        t = torch.tensor([self.n], dtype=torch.int64, device=self.dev)
        dist.all_reduce(t, group=self.group)
        return int(t.item())

    def bmu_coords(self) -> np.ndarray:
        """(n, 2) int32 [row, col] of ALL rows' BMUs (rank order), computed on
        the device (kernels.py:257-262) and copied through pinned memory."""
        if self.world == 1:
            b = self.bmu[: self.n]
            return to_host(torch.stack((b // self.nx, b % self.nx), dim=1).to(torch.int32))
        from .kernels import _to_coords
        return _to_coords(self.gather_bmus(), self.nx)

    def gather_bmus(self) -> np.ndarray:
        """Flat BMU indices of ALL rows (rank order), on every rank."""
        local = self.bmu[: self.n].to(torch.int64)
        if self.world == 1:
            return to_host(local)
        import torch.distributed as dist
        counts = [torch.zeros(1, dtype=torch.int64, device=self.dev) for _ in range(self.world)]
        dist.all_gather(counts, torch.tensor([self.n], dtype=torch.int64, device=self.dev),
                        group=self.group)
        cn = [int(c.item()) for c in counts]
        m = max(cn)
        buf = torch.zeros(m, dtype=torch.int64, device=self.dev)
        buf[: self.n] = local
        outs = [torch.empty(m, dtype=torch.int64, device=self.dev) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        return torch.cat([o[:c] for o, c in zip(outs, cn)]).cpu().numpy()
