"""Data-parallel plumbing: the reference's row partition (distributed.py:424-434)
and per-rank dataset slicing.  The per-epoch exchange (one fp64 all-reduce
of [S | cnt | qe] + an all-gather of the updated codebook slices) lives in
engine.SomEngine.reduce / update and replaces the coordinator fold of
distributed.py:492-514."""
from __future__ import annotations

import numpy as np

from .datasets import DenseDataset, SparseDataset


def partition(n_vectors: int, p: int) -> list[tuple[int, int]]:
    """Contiguous near-equal (first, count) slices; remainder to early ranks."""
    base, extra = divmod(n_vectors, p)
    out, first = [], 0
    for r in range(p):
        count = base + (1 if r < extra else 0)
        out.append((first, count))
        first += count
    return out


def slice_rows(data, first: int, count: int):
    if isinstance(data, SparseDataset):
        a, b = int(data.row_offsets[first]), int(data.row_offsets[first + count])
        return SparseDataset(data.n_dimensions, data.row_offsets[first:first + count + 1] - a,
                             data.col_indices[a:b], data.values[a:b])
    vals = data.values if isinstance(data, DenseDataset) else data
    return DenseDataset(vals[first:first + count])


def node_slices(n_nodes: int, p: int) -> list[tuple[int, int]]:
    """Update ownership: rank r owns nodes [r*kc, min(K, (r+1)*kc)), kc = ceil(K/p)."""
    kc = -(-n_nodes // p)
    return [(min(n_nodes, r * kc), min(n_nodes, (r + 1) * kc)) for r in range(p)]


def allreduce_sum(buf, group=None) -> None:
    """The one per-epoch exchange of the sharded path: fp64 sum of the packed
    [S | cnt | qe] accumulators over all ranks (replaces the rank-ordered
    fold of distributed.py:502-512).  NCCL on GPUs, gloo in CPU tests."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)


def allgather_rows(buf, rows_per_rank: int, group=None) -> None:
    """Every rank updated rows [r*kc, (r+1)*kc) of `buf` (kpad x d); gather
    all slices so each rank holds the full new codebook (replaces the
    codebook broadcast of distributed.py:494-496)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return
    world = dist.get_world_size(group)
    if world == 1:
        return
    rank = dist.get_rank(group)
    mine = buf[rank * rows_per_rank:(rank + 1) * rows_per_rank].contiguous()
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(buf, mine, group=group)
    else:
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=group)
        buf.copy_(torch.cat(parts, 0))
