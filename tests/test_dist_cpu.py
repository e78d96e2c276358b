"""Multi-process (gloo, world_size 2, CPU) test of the sharded epoch: rows
partitioned like distributed.partition, local node sums, one all-reduce of
the packed fp64 [S | cnt | qe] buffer, per-rank node-slice update, one
all-gather of the codebook rows -- the exact decomposition the NCCL path of
engine.SomEngine runs -- must reproduce the single-process reference epoch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_1305_1422_b200.parallel import (allgather_columns, allgather_rows, allreduce_sum,
                                           column_blocks, node_slices, partition,
                                           reduce_scatter_blocks, slice_rows)
from paper_1305_1422_b200.datasets import DenseDataset


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, x, w, nx, ny, radius, scale, mt, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        k, d = w.shape
        first, count = partition(len(x), world)[rank]
        xs = slice_rows(DenseDataset(x), first, count).values
        # local search + node sums (the oracle stands in for the device kernels)
        bmu, qe, _, _ = O.search_accumulate(xs, w, nx, ny, radius, 0.0, mt, with_accumulators=False)
        s, c = O.node_sums(xs, bmu, k)
        acc = torch.from_numpy(np.concatenate([s.ravel(), c, [qe]]))
        allreduce_sum(acc)
        S = acc[: k * d].view(k, d).numpy()
        C = acc[k * d: k * d + k].numpy()
        qe_all = float(acc[-1])
        kc = -(-k // world)
        buf = torch.zeros((kc * world, d), dtype=torch.float32)
        nb, ne = node_slices(k, world)[rank]
        num, den = O.conv_update(S, C, nx, ny, radius, 1e-3, mt, nodes=np.arange(nb, ne))
        buf[nb:ne] = torch.from_numpy(O.blend(w[nb:ne], num, den, scale))
        allgather_rows(buf, kc)
        out[rank] = (buf[:k].numpy().copy(), qe_all, bmu)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mt", [O.PLANAR, O.TOROID])
def test_sharded_epoch_matches_single_process(world, mt):
    rng = np.random.default_rng(4)
    nx, ny, d = 9, 7, 5
    x = rng.random((301, d), dtype=np.float32)
    w = rng.random((nx * ny, d), dtype=np.float32)
    radius, scale = 2.5, 0.6
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), x, w, nx, ny, radius, scale, mt, out),
             nprocs=world, join=True)
    _, qe, num, den = O.search_accumulate(x, w, nx, ny, radius, 1e-3, mt)
    want = O.blend(w, num, den, scale)
    for r in range(world):
        got, qe_r, _ = out[r]
        np.testing.assert_array_max_ulp(got, want, maxulp=1)
        assert qe_r == pytest.approx(qe, rel=1e-12)
    assert all(np.array_equal(out[0][0], out[r][0]) for r in range(world))   # bit-identical replicas


def _worker_cols(rank, world, port, x, w, nx, ny, radius, scale, mt, out):
    """The column-sharded exchange (engine default): reduce-scatter of S by
    feature columns, all-reduce of [cnt | qe], update of all nodes on this
    rank's columns, all-gather of the column blocks."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        k, d = w.shape
        first, count = partition(len(x), world)[rank]
        xs = slice_rows(DenseDataset(x), first, count).values
        bmu, qe, _, _ = O.search_accumulate(xs, w, nx, ny, radius, 0.0, mt, with_accumulators=False)
        s, c = O.node_sums(xs, bmu, k)
        dc = -(-d // world)
        # S column-block-major [world, k, dc], as somb_node_sums_*_cols writes it
        sp = np.zeros((k, world * dc))
        sp[:, :d] = s
        blocks = torch.from_numpy(np.ascontiguousarray(sp.reshape(k, world, dc).transpose(1, 0, 2)))
        mine = torch.empty((k, dc), dtype=torch.float64)
        reduce_scatter_blocks(blocks, mine)
        tail = torch.from_numpy(np.concatenate([c, [qe]]))
        allreduce_sum(tail)
        C, qe_all = tail[:k].numpy(), float(tail[-1])
        a, b = column_blocks(d, world)[rank]
        blk = np.zeros((k, dc), np.float32)
        if b > a:
            num, den = O.conv_update(mine.numpy()[:, : b - a], C, nx, ny, radius, 1e-3, mt)
            blk[:, : b - a] = O.blend(w[:, a:b], num, den, scale)
        W = torch.zeros((k, d), dtype=torch.float32)
        allgather_columns(torch.from_numpy(blk), torch.empty((world, k, dc), dtype=torch.float32), W, d)
        out[rank] = (W.numpy().copy(), qe_all, bmu)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mt", [O.PLANAR, O.TOROID])
def test_column_sharded_epoch_matches_single_process(world, mt):
    rng = np.random.default_rng(5)
    nx, ny, d = 9, 7, 5        # d = 5 over 2 / 3 ranks: padded last blocks
    x = rng.random((301, d), dtype=np.float32)
    w = rng.random((nx * ny, d), dtype=np.float32)
    radius, scale = 2.5, 0.6
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_cols, args=(world, _free_port(), x, w, nx, ny, radius, scale, mt, out),
             nprocs=world, join=True)
    _, qe, num, den = O.search_accumulate(x, w, nx, ny, radius, 1e-3, mt)
    want = O.blend(w, num, den, scale)
    for r in range(world):
        got, qe_r, _ = out[r]
        np.testing.assert_array_max_ulp(got, want, maxulp=1)
        assert qe_r == pytest.approx(qe, rel=1e-12)
    assert all(np.array_equal(out[0][0], out[r][0]) for r in range(world))


def test_node_slices_cover_and_pad():
    for k, p in [(40000, 8), (7, 3), (5, 8)]:
        sl = node_slices(k, p)
        assert sl[0][0] == 0 and sl[-1][1] == k
        assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
