"""Multi-GPU drivers: one process per GPU, NCCL (torch.distributed) for plumbing.

* ``shard_range``: contiguous batch / row / image slabs per rank (C2, C4, C5 —
  independent units, no data-path collective).
* ``fft2d_row_sharded`` (C3): a 2-D transform whose rows are
  split contiguously over P ranks.  Row FFTs run locally; ONE all-to-all
  turns each rank's row slab into a column slab (the send buffer is packed
  so that the received buffer is already the n0 x (n1/P) column slab in
  row-major order); column FFTs run locally; optionally a second all-to-all
  restores the row-sharded layout.

The local transforms default to the sm_100a kernels (``ops``).  They are
parameters only so that the choreography (packing, the exchange, the final
layout) can be tested with world-size-2 gloo groups on CPU, where the tests
inject the oracle as the local transform.
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

__all__ = ["shard_range", "fft2d_row_sharded", "pack_column_blocks", "unpack_column_blocks"]


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of a contiguous near-even split (first ranks take the remainder)."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pack_column_blocks(rows: torch.Tensor, world: int) -> torch.Tensor:
    """(r, n1) -> (world, r, n1/world): block s = columns [s*n1/P, (s+1)*n1/P)."""
    r, n1 = rows.shape
    return rows.view(r, world, n1 // world).transpose(0, 1).contiguous()


def unpack_column_blocks(blocks: torch.Tensor) -> torch.Tensor:
    """(world, r, n1/world) -> (r, n1): inverse of pack_column_blocks."""
    world, r, w = blocks.shape
    return blocks.transpose(0, 1).reshape(r, world * w)


def _default_rows(x: torch.Tensor) -> torch.Tensor:
    from . import ops
    return ops.fft_forward(x, x.shape[-1], out=x)


def _default_cols(x: torch.Tensor) -> torch.Tensor:
    from . import ops
    return ops.fft_columns(x, x.shape[0], x.shape[1])


def fft2d_row_sharded(local_rows: torch.Tensor, n0: int, *, group=None, transpose_back: bool = True,
                      row_fft: Callable | None = None, col_fft: Callable | None = None) -> torch.Tensor:
    """Forward 2-D FFT of an n0 x n1 array whose rows are sharded over the group.

    local_rows: (n0/P, n1) complex64, this rank's contiguous row slab.
    Returns the rank's row slab of the result (transpose_back=True) or its
    column slab, shape (n0, n1/P) (transpose_back=False)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    r, n1 = local_rows.shape
    if r * world != n0:
        raise ValueError(f"{world} ranks x {r} rows != {n0} rows")
    if n1 % world:
        raise ValueError(f"row length {n1} is not divisible by {world} ranks")
    row_fft = row_fft or _default_rows
    col_fft = col_fft or _default_cols
    x = row_fft(local_rows.contiguous())
    send = pack_column_blocks(x, world)             # (P, r, n1/P)
    recv = torch.empty_like(send)
    if world > 1:
        _all_to_all(recv, send, group)
    else:
        recv = send
    slab = recv.view(n0, n1 // world)               # rows in global order: already the column slab
    slab = col_fft(slab)
    if not transpose_back:
        return slab
    back = slab.view(world, r, n1 // world).contiguous()  # block s -> rank s (its rows)
    out = torch.empty_like(back)
    if world > 1:
        _all_to_all(out, back, group)
    else:
        out = back
    return unpack_column_blocks(out)


def _all_to_all(recv: torch.Tensor, send: torch.Tensor, group) -> None:
    """Equal-split all-to-all of complex64 buffers as float32 pairs (NCCL on
    CUDA tensors, gloo on CPU); block s of `send` goes to rank s."""
    as_real = (lambda t: torch.view_as_real(t).reshape(-1)) if send.is_complex() else (lambda t: t.reshape(-1))
    if send.is_cuda and dist.get_backend(group) == "gloo":
        # gloo cannot exchange CUDA buffers: used only by multi-rank tests that
        # share one GPU (NCCL refuses two ranks on one device)
        staged = as_real(send).cpu()
        got = torch.empty_like(staged)
        dist.all_to_all_single(got, staged, group=group)
        as_real(recv).copy_(got)
        return
    dist.all_to_all_single(as_real(recv), as_real(send), group=group)
