"""Row-sharded 2-D FFT with the exchange fused into the column pass
(``PeerShardedFft2d`` -> C-ABI ``dpp_fft2d_columns_sharded``).

The multi-rank cases run P processes on the ONE GPU this harness has: CUDA
IPC maps each process's row slab into the others exactly as across GPUs (the
kernel's TMA loads/stores then hit local HBM instead of NVLink), and the flag
barrier runs between time-sliced contexts.  The result must be bit-identical
to the single-GPU 2-D plan (same kernels, same twiddles, same order of
operations), which is itself parity-tested against the oracle
(test_fft_gpu.py)."""

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


def _input(n0: int, n1: int, batch: int) -> np.ndarray:
    rng = np.random.default_rng(11)
    return (rng.standard_normal((batch, n0, n1)) + 1j * rng.standard_normal((batch, n0, n1))).astype(np.complex64)


def _single_gpu(full: np.ndarray) -> np.ndarray:
    from paper_1203_4938_b200 import ops
    batch, n0, n1 = full.shape
    x = torch.from_numpy(full).cuda()
    out = torch.empty_like(x)
    ops.fft2d_forward(x, n0, n1, out=out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _worker(rank, world, port, n0, n1, batch, back, barrier, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1203_4938_b200.distributed import PeerShardedFft2d
        full = _input(n0, n1, batch)
        r = n0 // world
        sh = PeerShardedFft2d(n0, n1, batch, barrier=barrier, timeout_s=60.0)
        x = torch.from_numpy(full[:, rank * r:(rank + 1) * r].copy()).cuda()
        first = sh(x, transpose_back=back).cpu().numpy()
        again = sh(x, transpose_back=back).cpu().numpy()  # buffers and epochs reused
        torch.cuda.synchronize()
        q.put((rank, first, bool(np.array_equal(first, again))))
        dist.barrier()
        sh.close()
    finally:
        dist.destroy_process_group()


def _run(world, n0, n1, batch, back, barrier="device"):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n0, n1, batch, back, barrier, q))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        got = {}
        for _ in range(world):
            rank, res, stable = q.get(timeout=300)
            got[rank] = res
            assert stable, f"rank {rank}: second call differs from the first"
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    for p in procs:
        assert p.exitcode == 0
    axis = 1 if back else 2
    return np.concatenate([got[r] for r in range(world)], axis=axis)


@pytest.mark.parametrize("back", [True, False])
@pytest.mark.parametrize("n0,n1,batch", [(4096, 256, 2), (16384, 64, 1)])
def test_single_rank_matches_2d_plan(n0, n1, batch, back):
    from paper_1203_4938_b200.distributed import PeerShardedFft2d
    full = _input(n0, n1, batch)
    sh = PeerShardedFft2d(n0, n1, batch)
    out = sh(torch.from_numpy(full).cuda(), transpose_back=back).cpu().numpy()
    assert np.array_equal(out, _single_gpu(full))


@pytest.mark.parametrize("world,n0,n1,batch,back", [
    (2, 4096, 256, 2, True),
    (2, 4096, 256, 2, False),
    (2, 16384, 128, 1, True),
    (4, 4096, 256, 1, False),
    # sub-box layouts of the short rings: one row group per rank (nb = 1),
    # kk = 256 / P output rows per rank, both output modes
    (2, 1024, 64, 1, True),
    (4, 1024, 64, 1, False),
    (4, 1024, 64, 1, True),
    (2, 2048, 32, 1, True),
    (2, 2048, 32, 1, False),
])
def test_ranks_share_one_gpu_bit_exact(world, n0, n1, batch, back):
    full = _input(n0, n1, batch)
    assert np.array_equal(_run(world, n0, n1, batch, back), _single_gpu(full))


def test_host_barrier_mode():
    full = _input(4096, 128, 1)
    assert np.array_equal(_run(2, 4096, 128, 1, True, barrier="host"), _single_gpu(full))


def test_rejects_unsupported_shapes():
    from paper_1203_4938_b200 import _lib, ops
    from paper_1203_4938_b200.errors import PlanError
    import ctypes as C
    plan = ops.fft_plan(2, 4096, 256, 1)
    x = torch.zeros((1, 4096, 256), dtype=torch.complex64, device="cuda")
    arr = (C.c_void_p * 4)(*([x.data_ptr()] * 4))
    lib = _lib.load()
    # 3 ranks: not a power of two
    assert lib.dpp_fft2d_columns_sharded(plan._h, arr, arr, 3, 0, 1, 1, None) == _lib.DPP_EINVAL
    # 256 columns do not split into 16-column tiles over 32 ranks
    assert lib.dpp_fft2d_columns_sharded(plan._h, arr, arr, 32, 0, 1, 1, None) == _lib.DPP_EINVAL
    plan_small = ops.fft_plan(2, 512, 256, 1)  # no column ring for 512 rows
    assert lib.dpp_fft2d_columns_sharded(plan_small._h, arr, arr, 2, 0, 1, 1, None) == _lib.DPP_ENOTSUP
    with pytest.raises((PlanError, ValueError)):
        from paper_1203_4938_b200.distributed import PeerShardedFft2d
        PeerShardedFft2d(4096, 24, 1)


@pytest.mark.parametrize("n0,n1", [(1024, 64), (2048, 32), (8192, 64), (32768, 32)])
def test_single_rank_other_column_lengths(n0, n1):
    """The PEER column pass for the 32- and 128-row-group rings (8192, 32768 rows)."""
    from paper_1203_4938_b200.distributed import PeerShardedFft2d
    full = _input(n0, n1, 1)
    sh = PeerShardedFft2d(n0, n1, 1)
    for back in (True, False):
        out = sh(torch.from_numpy(full).cuda(), transpose_back=back).cpu().numpy()
        assert np.array_equal(out, _single_gpu(full))
