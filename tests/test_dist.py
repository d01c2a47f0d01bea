"""Row-sharded 2-D FFT choreography with world_size 2 on CPU (gloo).

The exchange (packing, all-to-all, final layout) is the product code in
paper_1203_4938_b200/distributed.py; the local 1-D transforms are injected
from the oracle because this box has no GPU (the GPU runs use the sm_100a
kernels).  Also covers the batch/image shard split used by C2/C4/C5.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fft_oracle as fo


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rows(x: torch.Tensor) -> torch.Tensor:
    return torch.from_numpy(fo.fft_rows(x.numpy()))


def _cols(x: torch.Tensor) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(fo.fft_rows(np.ascontiguousarray(x.numpy().T)).T))


def _worker(rank: int, world: int, port: int, n0: int, n1: int, back: bool, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1203_4938_b200.distributed import fft2d_row_sharded, shard_range
    rng = np.random.default_rng(3)
    full = (rng.standard_normal((n0, n1)) + 1j * rng.standard_normal((n0, n1))).astype(np.complex64)
    lo, hi = shard_range(n0, world, rank)
    out = fft2d_row_sharded(torch.from_numpy(full[lo:hi].copy()), n0, transpose_back=back,
                            row_fft=_rows, col_fft=_cols)
    q.put((rank, out.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("back", [True, False])
def test_row_sharded_2d_fft_world2(back):
    n0, n1, world = 32, 64, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n0, n1, back, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(3)
    full = (rng.standard_normal((n0, n1)) + 1j * rng.standard_normal((n0, n1))).astype(np.complex64)
    ref = fo.fft2(full)
    if back:
        res = np.concatenate([got[0], got[1]], axis=0)
    else:
        res = np.concatenate([got[0], got[1]], axis=1)
    assert np.linalg.norm(res - ref) / np.linalg.norm(ref) < 1e-6


def test_shard_range_covers_everything():
    from paper_1203_4938_b200.distributed import shard_range
    for total in (0, 1, 7, 4096, 4097):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_pack_unpack_round_trip():
    from paper_1203_4938_b200.distributed import pack_column_blocks, unpack_column_blocks
    x = torch.arange(6 * 8, dtype=torch.float32).view(6, 8)
    blocks = pack_column_blocks(x, 4)
    assert blocks.shape == (4, 6, 2)
    assert torch.equal(blocks[1], x[:, 2:4])
    assert torch.equal(unpack_column_blocks(blocks), x)
