"""Sharded k-means driver (kmeans.kmeans_sharded) with world_size 2 on CPU
(gloo): per-shard steps from a numpy stand-in of the CUDA shard
(tests/kmeans_shard_np.py), so the collectives — d2 totals, owner broadcast of
the drawn point, Lloyd accumulator all-reduce, farthest-point MAX — are the
product code.  The result must equal the single-process run up to summation
order, and reach the reference trainer's quality."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from kmeans_shard_np import NumpyShard


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _points(seed: int = 4, n: int = 900) -> np.ndarray:
    rng = np.random.default_rng(seed)
    centers = rng.normal(0, 3, (12, 16))
    return centers[rng.integers(0, 12, n)] + rng.normal(0, 0.5, (n, 16))


def _worker(rank, world, port, split, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1203_4938_b200.kmeans import kmeans_sharded
        pts = _points()
        lo, hi = split[rank], split[rank + 1]
        trace: list[float] = []
        cb = kmeans_sharded(None, k, seed=3, trace=trace, shard=NumpyShard(pts[lo:hi], k))
        q.put((rank, cb.numpy(), trace))
    finally:
        dist.destroy_process_group()


def _single(k):
    from paper_1203_4938_b200.kmeans import kmeans_sharded
    trace: list[float] = []
    cb = kmeans_sharded(None, k, seed=3, trace=trace, shard=NumpyShard(_points(), k))
    return cb.numpy(), trace


@pytest.mark.parametrize("split", [[0, 450, 900], [0, 0, 900], [0, 37, 900]])
def test_two_ranks_match_one(split):
    k, world = 24, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, split, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r, (cb, tr)) for r, cb, tr in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cb1, tr1 = _single(k)
    for r in range(world):
        cb, tr = got[r]
        assert np.allclose(cb, cb1, atol=1e-6), r
        assert len(tr) == len(tr1) and np.allclose(tr, tr1, rtol=1e-9)


def test_sharded_quality_matches_reference_trainer():
    from oracle import imgc_oracle as io
    pts = _points(n=600)
    ref = io.kmeans(pts, 16, 0)
    from paper_1203_4938_b200.kmeans import kmeans_sharded
    got = kmeans_sharded(None, 16, seed=0, shard=NumpyShard(pts, 16)).numpy().astype(np.float64)

    def sse(c):
        return ((pts[:, None, :] - c[None]) ** 2).sum(-1).min(1).sum()

    assert sse(got) <= 1.03 * sse(np.asarray(ref, dtype=np.float64))


def test_duplicate_points_known_answer():  # test_imgc.py:90-128 pattern
    from paper_1203_4938_b200.kmeans import kmeans_sharded
    pts = np.repeat(np.arange(6, dtype=np.float64)[:, None], 16, 1)
    pts = np.vstack([pts] * 3)
    cb = kmeans_sharded(None, 6, seed=1, shard=NumpyShard(pts, 6)).numpy()
    assert sorted(cb[:, 0].tolist()) == [0, 1, 2, 3, 4, 5]
