"""C4 tile sharding: one frame's block rows split into P bands,
each rank encodes its band, the bitstream is the concatenation at fixed
offsets (imgc.py:295-305).

* CPU, world 2 (gloo): the choreography in ``distributed.compress_tile_sharded``
  with the oracle encoder as the band stand-in — the gathered bitstream equals
  the oracle's single-process bitstream, including uneven bands.
* GPU, world 1/2/3 (ranks sharing the one B200 over gloo): the sm_100a band
  encoder — byte-identical to the single-GPU ``compress``.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import imgc_oracle as io


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _frame(h, w):
    return io.synthetic_image(w, h, seed=5)


def _codebook():
    rng = np.random.default_rng(1)
    cb = rng.standard_normal((32, 16))
    return ((cb - cb.mean(1, keepdims=True)) / cb.std(1, keepdims=True)).astype(np.float32)


def _oracle_band(image, ch, h, w, cents, band):
    lo, hi = band
    sub = image[4 * lo:4 * hi]
    if sub.ndim == 2:
        sub = np.repeat(sub[..., None], 3, 2)
    f = io.encode(sub[..., :3], cents)
    return np.stack([f["means"], f["sigma_idx"], f["indices"]], 1), f["cb"].ravel(), f["cr"].ravel()


def _worker(rank, world, port, h, w, gpu, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if gpu:
        torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1203_4938_b200.distributed import compress_tile_sharded
        img = _frame(h, w)
        ci = compress_tile_sharded(img, _codebook(), encode=None if gpu else _oracle_band)
        q.put((rank, ci.to_bytes()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(world, h, w, gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, h, w, gpu, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        got = dict(q.get(timeout=300) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    return got


@pytest.mark.parametrize("h,w", [(64, 48), (52, 40)])  # 16 and 13 block rows (even and uneven bands)
def test_tile_sharded_bitstream_world2(h, w):
    got = _run(2, h, w, gpu=False)
    ref = io.to_bytes(io.encode(_frame(h, w), _codebook()))
    assert got[0] == ref and got[1] == ref


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3])
def test_tile_sharded_on_gpu_equals_single_gpu(cuda, world):
    from paper_1203_4938_b200.apps import imgc
    h, w = 520, 384  # 130 block rows: uneven bands at 3 ranks
    single = imgc.compress(_frame(h, w), 32, 0, codebook=_codebook()).to_bytes()
    assert single == io.to_bytes(io.encode(_frame(h, w), _codebook()))
    if world == 1:
        from paper_1203_4938_b200.distributed import compress_tile_sharded
        assert compress_tile_sharded(_frame(h, w), _codebook()).to_bytes() == single
        return
    got = _run(world, h, w, gpu=True)
    assert all(b == single for b in got.values())
