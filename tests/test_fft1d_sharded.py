"""Row-sharded large 1-D FFT (distributed.fft1d_row_sharded; north star:
"Large 2D and 1D FFTs shard by rows, with the transpose done as an all-to-all").

* CPU, world 2 (gloo): the choreography (two all-to-alls, twiddle on the
  column slab, natural-order third all-to-all) with the oracle as the local
  transforms — equal to the oracle's fft() of the whole signal.
* GPU, world 1 and 2 (ranks sharing the one B200 over gloo): the sm_100a column
  pass, twiddle kernel and row FFTs — within the north-star tolerance of the
  oracle, and the two output layouts consistent.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import complex_signals, rel_l2
from oracle import fft_oracle as fo


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rows(x: torch.Tensor) -> torch.Tensor:
    return torch.from_numpy(fo.fft_rows(x.numpy()))


def _cols(x: torch.Tensor) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(fo.fft_rows(np.ascontiguousarray(x.numpy().T)).T))


def _twiddle(x: torch.Tensor, rows: int, cols: int, col0: int, n: int) -> torch.Tensor:
    r = np.arange(rows, dtype=np.int64)[:, None]
    c = col0 + np.arange(cols, dtype=np.int64)[None, :]
    w = np.exp(-2j * np.pi * ((r * c) % n) / n).astype(np.complex64)
    return torch.from_numpy((x.numpy().reshape(rows, cols) * w).astype(np.complex64))


def _worker(rank, world, port, n, natural, gpu, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if gpu:
        torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1203_4938_b200.distributed import fft1d_row_sharded
        x = complex_signals(n, (n,))
        part = torch.from_numpy(x[rank * n // world:(rank + 1) * n // world].copy())
        if gpu:
            out = fft1d_row_sharded(part.cuda(), n, natural_output=natural).cpu()
        else:
            out = fft1d_row_sharded(part, n, natural_output=natural, row_fft=_rows, col_fft=_cols, twiddle=_twiddle)
        q.put((rank, out.numpy()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(world, n, natural, gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, natural, gpu, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        got = dict(q.get(timeout=300) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    return got


def _assemble(got, n, world, natural):
    from paper_1203_4938_b200.distributed import fft1d_split
    if natural:
        return np.concatenate([got[r] for r in range(world)])
    r, c = fft1d_split(n, world)
    z = np.concatenate([got[k] for k in range(world)])  # (R, C): Z[k_r][k_c] = X[k_r + R k_c]
    return z.T.reshape(-1)


@pytest.mark.parametrize("n", [1024, 2048])
@pytest.mark.parametrize("natural", [True, False])
def test_sharded_1d_choreography_world2(n, natural):
    got = _run(2, n, natural, gpu=False)
    x = complex_signals(n, (n,))
    assert rel_l2(_assemble(got, n, 2, natural), fo.fft(x)) <= 1e-5 * np.log2(n)


def test_split_rules():
    from paper_1203_4938_b200.distributed import fft1d_split
    assert fft1d_split(1 << 24, 8) == (4096, 4096)
    assert fft1d_split(1 << 25, 2) == (8192, 4096)
    with pytest.raises(ValueError):
        fft1d_split(1 << 10, 64)
    with pytest.raises(ValueError):
        fft1d_split(1000, 2)


@pytest.mark.gpu
@pytest.mark.parametrize("world,n", [(1, 1 << 16), (1, 1 << 22), (2, 1 << 16), (2, 1 << 20)])
def test_sharded_1d_on_gpu_vs_oracle(cuda, world, n):
    x = complex_signals(n, (n,))
    ref = fo.fft(x)
    for natural in (True, False):
        if world == 1:
            from paper_1203_4938_b200.distributed import fft1d_row_sharded
            got = {0: fft1d_row_sharded(torch.from_numpy(x).to(cuda), n, natural_output=natural).cpu().numpy()}
        else:
            got = _run(world, n, natural, gpu=True)
        assert rel_l2(_assemble(got, n, world, natural), ref) <= 1e-5 * np.log2(n), (world, n, natural)
