"""Data-parallel plumbing: the reference's row partition (distributed.py:424-434)
and per-rank dataset slicing.  The per-epoch exchange lives in
engine.SomEngine.reduce / update and replaces the coordinator fold of
distributed.py:492-514: a column-block reduce-scatter of the fp64 node sums
S, an all-reduce of [cnt | qe], every rank's update of its feature columns
for all nodes, and a column-block all-gather of the new codebook (the
legacy node-slice scheme -- all-reduce of [S | cnt | qe], node-slice update,
row all-gather -- stays available as EngineOptions(shard_update="nodes"))."""
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
    if dist.is_available() and dist.is_initialized():
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
    rank = dist.get_rank(group)
    mine = buf[rank * rows_per_rank:(rank + 1) * rows_per_rank].contiguous()
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(buf, mine, group=group)
    else:
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=group)
        buf.copy_(torch.cat(parts, 0))


def column_blocks(d: int, p: int) -> list[tuple[int, int]]:
    """Feature-column ownership: rank r updates columns [r*dc, min(d, (r+1)*dc)), dc = ceil(d/p)."""
    dc = -(-d // p)
    return [(min(d, r * dc), min(d, (r + 1) * dc)) for r in range(p)]


def reduce_scatter_blocks(S_blocks, out, group=None) -> None:
    """out [K, dc] <- sum over ranks of block `rank` of S_blocks [p, K, dc]
    (the column-block-major node sums written by somb_node_sums_*_cols: the
    blocks are already contiguous, so NCCL reduce-scatters S in place; the
    gloo backend has no reduce-scatter: all-reduce, then take the block)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    if dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(out, S_blocks, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.all_reduce(S_blocks, op=dist.ReduceOp.SUM, group=group)
        out.copy_(S_blocks[rank])


def allgather_columns(mine, staging, W, d: int, group=None) -> None:
    """W[:, :d] <- the column blocks [K, dc] of every rank, in rank order."""
    import torch
    import torch.distributed as dist
    p, K, dc = staging.shape
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(staging, mine, group=group)
    else:
        parts = [torch.empty_like(mine) for _ in range(p)]
        dist.all_gather(parts, mine, group=group)
        staging.copy_(torch.stack(parts, 0))
    full = min(p, d // dc)
    if full:
        W[:, : full * dc].view(K, full, dc).copy_(staging[:full].permute(1, 0, 2))
    rem = d - full * dc
    if full < p and rem:
        W[:, full * dc: d].copy_(staging[full, :, :rem])
