"""Command line with the reference's training flags (cli.py:61-93, local
role), plus the B200 extensions.  Multi-GPU replaces the reference's
coordinator / worker roles (distributed.py:450-628, cli.py:138-201): launch
one process per GPU with torchrun; every rank reads the input, trains its
row partition (distributed.py:424-434) with one NCCL all-reduce per epoch,
and rank 0 prints progress and writes the artifacts.

    python -m paper_1305_1422_b200 -x 200 -y 200 -m toroid -k 1 data.txt out
    torchrun --nproc-per-node 8 -m paper_1305_1422_b200 -k 1 data.txt out
"""
from __future__ import annotations

import argparse
import os
import sys
from typing import Optional

from . import errors


class _Parser(argparse.ArgumentParser):
    def error(self, message):            # argparse exits 2; the reference maps usage errors to 1
        raise errors.UsageError(message)


def build_parser() -> argparse.ArgumentParser:
    p = _Parser(prog="somb200", description="B200 batch self-organizing map trainer", allow_abbrev=False)
    p.add_argument("-c", "--initial-codebook", metavar="FILE", default=None,
                   help="initial codebook file (default: seeded random init)")
    p.add_argument("-e", "--epochs", type=int, default=10, metavar="N", help="training epochs (default 10)")
    p.add_argument("-k", "--kernel", type=int, choices=(0, 1, 2), default=0,
                   help="0 dense naive, 1 dense blocked, 2 sparse (default 0)")
    p.add_argument("-m", "--map", choices=("planar", "toroid"), default="planar",
                   help="map topology (default planar)")
    p.add_argument("-t", "--radius-cooling", choices=("linear", "exponential"), default="linear")
    p.add_argument("-r", "--radius0", type=float, default=0, metavar="R",
                   help="start radius (0 = half the smaller map side)")
    p.add_argument("-R", "--radiusN", type=float, default=0, metavar="R", help="end radius (0 = 1)")
    p.add_argument("-T", "--scale-cooling", choices=("linear", "exponential"), default="linear")
    p.add_argument("-l", "--scale0", type=float, default=0, metavar="S", help="start learning scale (0 = 1.0)")
    p.add_argument("-L", "--scaleN", type=float, default=0, metavar="S", help="end learning scale (0 = 0.01)")
    p.add_argument("-s", "--snapshots", type=int, choices=(0, 1, 2), default=0,
                   help="0 none, 1 interim U-matrix, 2 also codebook and BMUs")
    p.add_argument("-x", "--columns", type=int, default=50, metavar="N", help="map columns (default 50)")
    p.add_argument("-y", "--rows", type=int, default=50, metavar="N", help="map rows (default 50)")
    p.add_argument("--seed", type=int, default=1, metavar="N", help="codebook init seed (default 1)")
    p.add_argument("--threads", type=int, default=os.cpu_count() or 1, metavar="N",
                   help="accepted for compatibility (the GPU is the parallelism)")
    # extensions (defaults reproduce the reference)
    p.add_argument("--grid", choices=("rectangular", "hexagonal"), default="rectangular")
    p.add_argument("--neighborhood", choices=("gaussian", "bubble"), default="gaussian")
    p.add_argument("--compact-support", action="store_true", help="h = 0 beyond the radius")
    p.add_argument("--cache", action="store_true",
                   help="keep a binary copy of the input (INPUT_FILE.sombc) and reuse it while the input is unchanged")
    p.add_argument("input_file", metavar="INPUT_FILE")
    p.add_argument("output_prefix", metavar="OUTPUT_PREFIX")
    return p


def config_from(ns):
    from .grid import GridType, MapType, Neighborhood
    from .kernels import Kernel
    from .train import Cooling, TrainConfig
    return TrainConfig(n_epochs=ns.epochs, n_columns=ns.columns, n_rows=ns.rows, map_type=MapType(ns.map),
                       kernel=Kernel(ns.kernel), radius0=ns.radius0, radiusN=ns.radiusN,
                       radius_cooling=Cooling(ns.radius_cooling), scale0=ns.scale0, scaleN=ns.scaleN,
                       scale_cooling=Cooling(ns.scale_cooling), snapshot_level=ns.snapshots, seed=ns.seed,
                       grid=GridType(ns.grid), neighborhood=Neighborhood(ns.neighborhood),
                       compact_support=ns.compact_support)


def _progress(state, qe: float) -> None:
    print(f"epoch {state.epoch} radius {state.radius:.6g} scale {state.scale:.6g} qe {qe:.6g}", flush=True)


def _init_distributed():
    """torchrun environment -> one NCCL rank per GPU (gloo with
    SOMB_DIST_BACKEND=gloo); returns (rank, world)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1:
        return 0, 1
    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    backend = os.environ.get("SOMB_DIST_BACKEND", "nccl")
    if not dist.is_initialized():
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return dist.get_rank(), dist.get_world_size()


def run(argv) -> int:
    if argv and argv[0] in ("coordinator", "worker"):
        raise errors.UsageError(f"the {argv[0]} role is replaced by torchrun: "
                                "torchrun --nproc-per-node N -m paper_1305_1422_b200 [OPTIONS] INPUT OUTPUT")
    ns = build_parser().parse_args(argv)
    cfg = config_from(ns)
    rank, world = _init_distributed()
    from .ingest import read_dataset
    from .train import FileSinks, load_codebook, train
    data, fmt = read_dataset(ns.input_file, cache=ns.cache)
    if rank == 0:
        print(f"somb200: read {data.n_vectors} x {data.n_dimensions} {fmt} input from {ns.input_file}"
              + (f" ({world} ranks)" if world > 1 else ""), file=sys.stderr)
    initial = load_codebook(ns.initial_codebook) if ns.initial_codebook else None
    sinks = FileSinks(ns.output_prefix) if rank == 0 else None
    train(data, cfg, sinks, workers=ns.threads, initial_codebook=initial,
          progress=_progress if rank == 0 else None)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main(argv: Optional[list] = None) -> int:
    """Exit codes of the reference (cli.py:208-221): 0 ok, 1 usage/config,
    2 input, 3 runtime (CUDA, missing device)."""
    args = sys.argv[1:] if argv is None else argv
    try:
        return run(args)
    except errors.UsageError as exc:
        print(f"somb200: {exc}", file=sys.stderr)
        print("usage: somb200 [OPTIONS] INPUT_FILE OUTPUT_PREFIX (see --help)", file=sys.stderr)
        return 1
    except errors.SomkitError as exc:
        print(f"somb200: {exc}", file=sys.stderr)
        return exc.exit_code
    except KeyboardInterrupt:
        return 3
