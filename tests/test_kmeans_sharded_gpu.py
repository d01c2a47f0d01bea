"""Sharded GPU k-means (``kmeans_sharded`` over ``CudaShard``, C-ABI
``dpp_kmeans_shard_*``): two ranks sharing the one GPU (gloo for the
collectives) against the single-GPU trainer ``dpp_kmeans`` on the same points
and seed.  Equal up to summation order: same iteration count, codebooks within
1e-5, and the SSE trace within 1e-9 relative."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _points(n: int = 20000) -> np.ndarray:
    rng = np.random.default_rng(21)
    centers = rng.normal(0, 2, (64, 16))
    return centers[rng.integers(0, 64, n)] + rng.normal(0, 0.6, (n, 16))


def _worker(rank, world, port, k, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1203_4938_b200.distributed import shard_range
        from paper_1203_4938_b200.kmeans import kmeans_sharded
        pts = _points()
        lo, hi = shard_range(len(pts), world, rank)
        trace: list[float] = []
        cb = kmeans_sharded(torch.from_numpy(pts[lo:hi]).cuda(), k, seed=5, trace=trace)
        q.put((rank, cb.cpu().numpy(), trace))
    finally:
        dist.destroy_process_group()


def test_two_ranks_match_single_gpu_trainer():
    import torch.multiprocessing as mp

    from paper_1203_4938_b200.kmeans import kmeans_device
    k, world = 128, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        got = {}
        for _ in range(world):
            r, cb, tr = q.get(timeout=300)
            got[r] = (cb, tr)
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    trace: list[float] = []
    ref = kmeans_device(_points(), k, 5, trace=trace).cpu().numpy()
    for r in range(world):
        cb, tr = got[r]
        assert len(tr) == len(trace)
        assert np.allclose(tr, trace, rtol=1e-9)
        assert np.abs(cb - ref).max() < 1e-5


def test_one_rank_matches_single_gpu_trainer(cuda):
    from paper_1203_4938_b200.kmeans import kmeans_device, kmeans_sharded
    pts = torch.from_numpy(_points(5000)).to(cuda)
    t1: list[float] = []
    t2: list[float] = []
    a = kmeans_sharded(pts, 64, seed=2, trace=t1).cpu().numpy()
    b = kmeans_device(pts, 64, 2, trace=t2).cpu().numpy()
    assert len(t1) == len(t2) and np.allclose(t1, t2, rtol=1e-9)
    assert np.abs(a - b).max() < 1e-5
