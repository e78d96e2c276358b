"""Sharded training through the real CUDA kernels on ONE GPU: two ranks
(gloo process group, both on cuda:0) run train() on partition(n, 2) slices
with the per-epoch exchange of engine.SomEngine (column-block
reduce-scatter of the node sums, [cnt | qe] all-reduce, column all-gather
of the codebook), and must reproduce the single-process run (the
reference's distributed equivalence test, test_distributed.py:257-265,
promises 1e-5; only the fp64 summation order across ranks differs)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cfg(S, kernel, big=False):
    if big:   # >= 2048 nodes: the spectral update; hex toroid, bubble, compact support
        return S.TrainConfig(n_epochs=4, n_columns=64, n_rows=48, map_type=S.MapType.TOROID, kernel=kernel,
                             grid=S.GridType.HEXAGONAL, neighborhood=S.Neighborhood.BUBBLE,
                             compact_support=True)
    return S.TrainConfig(n_epochs=5, n_columns=20, n_rows=16, map_type=S.MapType.TOROID, kernel=kernel)


def _worker(rank, world, port, x, sparse, out_dir, big=False):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1305_1422_b200 as S
        if sparse:
            data = S.SparseDataset(*x)
            kernel = S.Kernel.SPARSE
        else:
            data = S.DenseDataset(x)
            kernel = S.Kernel.DENSE_BLOCKED
        cb, bmus, u = S.train(data, _cfg(S, kernel, big), device="cuda:0")
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), w=cb.weights, b=bmus, u=u.heights)
    finally:
        dist.destroy_process_group()


def _run(tmp_path, x, sparse, big=False):
    import torch.multiprocessing as mp
    import paper_1305_1422_b200 as S
    mp.spawn(_worker, args=(2, _free_port(), x, sparse, str(tmp_path), big), nprocs=2, join=True)
    data = S.SparseDataset(*x) if sparse else S.DenseDataset(x)
    kernel = S.Kernel.SPARSE if sparse else S.Kernel.DENSE_BLOCKED
    cb, bmus, u = S.train(data, _cfg(S, kernel, big), device="cuda:0")
    r0, r1 = np.load(tmp_path / "r0.npz"), np.load(tmp_path / "r1.npz")
    # every rank holds the same replica
    assert np.array_equal(r0["w"], r1["w"]) and np.array_equal(r0["b"], r1["b"])
    rel = np.max(np.abs(r0["w"].astype(np.float64) - cb.weights) / np.maximum(np.abs(cb.weights), 1e-12))
    assert rel <= 1e-5, f"sharded vs single codebook rel err {rel}"
    assert np.mean(np.any(r0["b"] != bmus, axis=1)) <= 1e-3
    urel = np.max(np.abs(r0["u"] - u.heights) / np.maximum(np.abs(u.heights), 1e-12))
    assert urel <= 1e-4


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_sharded_train_dense_two_ranks_one_gpu(tmp_path):
    rng = np.random.default_rng(5)
    centers = rng.random((8, 48)).astype(np.float32)
    x = (centers[rng.integers(0, 8, 6000)] + 0.05 * rng.standard_normal((6000, 48))).astype(np.float32)
    _run(tmp_path, x, sparse=False)


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_sharded_train_spectral_hex_two_ranks_one_gpu(tmp_path):
    """3072-node hex toroid (spectral update, bubble, compact support), d = 47:
    the two column blocks are 24 + 23 columns (one padded)."""
    rng = np.random.default_rng(6)
    centers = rng.random((12, 47)).astype(np.float32)
    x = (centers[rng.integers(0, 12, 8000)] + 0.05 * rng.standard_normal((8000, 47))).astype(np.float32)
    _run(tmp_path, x, sparse=False, big=True)


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_sharded_train_sparse_two_ranks_one_gpu(tmp_path):
    import oracle as O
    sp = O.gen_random_sparse(3000, 400, 0.02, 11)
    _run(tmp_path, (sp.n_dimensions, sp.row_offsets, sp.col_indices, sp.values), sparse=True)


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_cli_local_and_torchrun_two_ranks(tmp_path):
    """The CLI (reference flags) trains and writes .wts/.bm/.umx (+ -s 2
    snapshots); under torchrun with two ranks on one GPU (gloo) rank 0 writes
    artifacts matching the single-process run."""
    import subprocess
    import sys
    from conftest import ROOT
    import paper_1305_1422_b200 as S
    from paper_1305_1422_b200 import fileio
    rng = np.random.default_rng(3)
    x = rng.random((3000, 12), dtype=np.float32)
    inp = tmp_path / "data.txt"
    inp.write_text("".join(" ".join(f"{v:.6g}" for v in row) + "\n" for row in x))
    args = ["-x", "9", "-y", "7", "-m", "toroid", "-k", "1", "-e", "4", "-s", "2", str(inp)]
    env = dict(os.environ, PYTHONPATH=ROOT)
    one = subprocess.run([sys.executable, "-m", "paper_1305_1422_b200"] + args + [str(tmp_path / "one")],
                         capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert one.returncode == 0, one.stderr[-2000:]
    assert one.stdout.count("epoch ") == 4
    for ext in ("wts", "bm", "umx"):
        assert (tmp_path / f"one.{ext}").exists() and (tmp_path / f"one.3.{ext}").exists()
    env2 = dict(env, SOMB_DIST_BACKEND="gloo")
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "-m",
                          "paper_1305_1422_b200"] + args + [str(tmp_path / "two")],
                         capture_output=True, text=True, timeout=600, env=env2, cwd=ROOT)
    assert two.returncode == 0, two.stderr[-3000:]
    n1, m1, w1 = fileio.load_codebook(str(tmp_path / "one.wts"))
    n2, m2, w2 = fileio.load_codebook(str(tmp_path / "two.wts"))
    assert (n1, m1) == (n2, m2) == (9, 7)
    assert np.max(np.abs(w1.astype(np.float64) - w2) / np.maximum(np.abs(w1), 1e-6)) <= 1e-4
    assert (tmp_path / "two.bm").read_text().count("\n") == 3001


def _nccl_single_worker(rank, port, x, out_dir):
    """One rank, NCCL: the sharded exchange forced on (exchange="always"), so
    reduce_scatter_tensor / all_gather_into_tensor / all_reduce /
    barrier(device_ids) run over NCCL on the GPU (the data plane the 8-GPU
    run uses; distributed.py:492-514)."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        import paper_1305_1422_b200 as S
        from paper_1305_1422_b200.engine import EngineOptions
        assert dist.get_backend() == "nccl"
        dist.barrier(device_ids=[0])
        out = {}
        for mode in ("columns", "nodes"):
            for big in (False, True):
                cb, bmus, u = S.train(S.DenseDataset(x), _cfg(S, S.Kernel.DENSE_BLOCKED, big), device="cuda:0",
                                      options=EngineOptions(exchange="always", shard_update=mode))
                out[f"{mode}{int(big)}_w"], out[f"{mode}{int(big)}_b"], out[f"{mode}{int(big)}_u"] = \
                    cb.weights, bmus, u.heights
        dist.barrier(device_ids=[0])
        np.savez(os.path.join(out_dir, "nccl1.npz"), **out)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_nccl_single_rank_exchange_matches_local(tmp_path):
    """The NCCL branches of the exchange (column reduce-scatter + all-gather,
    node-slice all-reduce + row all-gather) on hardware, in a 1-rank NCCL
    group: the result must equal the local run bit for bit (with one rank
    the collectives are identities, the column update is the same
    arithmetic per column)."""
    import torch.multiprocessing as mp
    import paper_1305_1422_b200 as S
    rng = np.random.default_rng(9)
    centers = rng.random((10, 47)).astype(np.float32)
    x = (centers[rng.integers(0, 10, 5000)] + 0.05 * rng.standard_normal((5000, 47))).astype(np.float32)
    mp.spawn(_nccl_single_worker, args=(_free_port(), x, str(tmp_path)), nprocs=1, join=True)
    got = np.load(tmp_path / "nccl1.npz")
    for big in (False, True):
        cb, bmus, u = S.train(S.DenseDataset(x), _cfg(S, S.Kernel.DENSE_BLOCKED, big), device="cuda:0")
        for mode in ("columns", "nodes"):
            assert np.array_equal(got[f"{mode}{int(big)}_w"], cb.weights), (mode, big)
            assert np.array_equal(got[f"{mode}{int(big)}_b"], bmus), (mode, big)
            assert np.array_equal(got[f"{mode}{int(big)}_u"], u.heights), (mode, big)
