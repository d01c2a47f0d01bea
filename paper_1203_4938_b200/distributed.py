"""Multi-GPU drivers: one process per GPU, NCCL (torch.distributed) for plumbing.

* ``shard_range``: contiguous batch / row / image slabs per rank (C2, C4, C5 —
  independent units, no data-path collective).
* ``PeerShardedFft2d`` (C3, the product path): the same
  row-sharded transform with the all-to-all fused into the column pass — every
  rank maps every other rank's row slab (CUDA IPC) and the column kernel reads
  its column block straight out of the peers' HBM over NVLink (TMA loads from
  peer pointers) and, for natural-order output, TMA-stores the results straight
  back into the peers' slabs.  No NCCL and no staging copies on the data path;
  two stream-ordered flag barriers per call.
* ``fft1d_row_sharded`` (large 1-D, north star "large 2D and 1D FFTs shard by
  rows"): one n-point signal split contiguously over P ranks, n = R x C
  four-step — all-to-all to column slabs, R-point column FFTs and the
  W_n^{r c} twiddle on device, all-to-all back, C-point row FFTs; optionally
  a third all-to-all returns natural-order contiguous output.
* ``compress_tile_sharded`` (C4): one frame's block rows split
  into P contiguous bands; each rank encodes its band (records, Cb and Cr rows
  are block-local, so a band is an independent sub-image) and the bitstream is
  the concatenation of the bands at fixed offsets (imgc.py:295-305) — one
  all-gather of the finished bytes, no data-path collective.
* ``fft2d_row_sharded`` (C3, the NCCL baseline): a 2-D transform whose rows are
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

__all__ = ["shard_range", "fft2d_row_sharded", "pack_column_blocks", "unpack_column_blocks",
           "PeerShardedFft2d", "encode_band", "compress_tile_sharded", "fft1d_split", "fft1d_row_sharded"]


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


class PeerShardedFft2d:
    """Row-sharded 2-D FFT, exchange fused into the column pass (C-ABI
    ``dpp_fft2d_columns_sharded``, include/dpp_b200.h; SURVEY §8(b)
    ``dpp_fft2d_c2c_fwd_sharded``).

    Collective: every rank of ``group`` constructs it with the same arguments
    (one process per GPU).  Each rank owns ``slab``, a (batch, n0/P, n1)
    complex64 row slab, and a flag array; their CUDA IPC handles are
    exchanged once (``all_gather_object``) and opened, so a call moves data
    only inside the kernels.  ``barrier="host"`` replaces the device flag
    barrier by stream sync + ``dist.barrier`` (for debugging)."""

    def __init__(self, n0: int, n1: int, batch: int = 1, group=None, device=None,
                 barrier: str = "device", timeout_s: float = 30.0):
        import ctypes as C
        from . import _lib, ops
        self._C, self._lib = C, _lib.load()
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if barrier not in ("device", "host"):
            raise ValueError(f"barrier must be 'device' or 'host', got {barrier!r}")
        if n0 % self.world or n1 % (16 * self.world):
            raise ValueError(f"{n0} x {n1} does not shard over {self.world} ranks")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.n0, self.n1, self.batch, self.device = n0, n1, batch, dev
        self.barrier_mode, self.timeout_s = barrier, timeout_s
        self.rows = n0 // self.world
        self.slab = torch.empty((batch, self.rows, n1), dtype=torch.complex64, device=dev)
        self.cols = torch.empty((batch, n0, n1 // self.world), dtype=torch.complex64, device=dev)
        self.flags = torch.zeros(8, dtype=torch.int32, device=dev)
        self._plan2d = ops.fft_plan(2, n0, n1, batch, dev)
        self._plan_rows = ops.fft_plan(1, n1, 1, batch * self.rows, dev)
        self._epoch = 0
        self._opened: list[int] = []
        self._slabs = self._exchange(self.slab)
        self._flag_ptrs = self._exchange(self.flags)
        P = self._C.c_void_p * self.world
        self._slab_arr = P(*self._slabs)
        self._flag_arr = P(*self._flag_ptrs)
        self._col_arr = P(self.cols.data_ptr(), *([0] * (self.world - 1)))
        self._group = C.c_void_p()
        from ._lib import check
        check(self._lib.dpp_peer_group_create(C.byref(self._group), self.world, self.rank, self._slab_arr,
                                              self._flag_arr, float(timeout_s)), "peer group")

    def _exchange(self, t: torch.Tensor) -> list[int]:
        """Pointers, valid in this process, to every rank's copy of ``t``."""
        C, lib = self._C, self._lib
        if self.world == 1:
            return [t.data_ptr()]
        from ._lib import check
        handle = C.create_string_buffer(64)
        off = C.c_uint64()
        check(lib.dpp_ipc_get_handle(t.data_ptr(), handle, C.byref(off)), "ipc handle")
        got: list = [None] * self.world
        dist.all_gather_object(got, (handle.raw, off.value), group=self.group)
        ptrs = []
        for j, (h, o) in enumerate(got):
            if j == self.rank:
                ptrs.append(t.data_ptr())
                continue
            base = C.c_void_p()
            check(lib.dpp_ipc_open(C.create_string_buffer(h, 64), C.byref(base)), f"ipc open (rank {j})")
            self._opened.append(base.value)
            ptrs.append(base.value + o)
        return ptrs

    def _barrier(self, stream) -> None:
        from ._lib import check
        from .ops import stream_handle
        if self.barrier_mode == "host":
            (stream or torch.cuda.current_stream(self.device)).synchronize()
            if self.world > 1:
                dist.barrier(group=self.group)
            return
        self._epoch += 1
        check(self._lib.dpp_peer_barrier(self._flag_arr, self.world, self.rank, self._epoch, self.timeout_s,
                                         stream_handle(stream)), "peer barrier")

    def __call__(self, local_rows: torch.Tensor | None = None, transpose_back: bool = True,
                 stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """Forward 2-D FFT of the row-sharded batch.  ``local_rows`` (this
        rank's (batch, n0/P, n1) rows; None: ``slab`` already holds them) is
        row-transformed into ``slab``.  Returns ``slab`` (transpose_back: this
        rank's rows of the result) or ``cols`` (this rank's (batch, n0, n1/P)
        column block) — buffers owned by this object, overwritten by the next
        call."""
        from ._lib import check
        from .ops import stream_handle
        src = self.slab if local_rows is None else local_rows
        if src.dtype != torch.complex64 or src.numel() != self.slab.numel() or not src.is_contiguous():
            raise ValueError(f"local rows must be contiguous complex64 of {tuple(self.slab.shape)}")
        if self.barrier_mode == "device":
            # one C-ABI call: rows, barrier, fused column/exchange pass, barrier
            check(self._lib.dpp_fft2d_c2c_fwd_sharded(self._plan2d._h, self._group, src.data_ptr(),
                                                       self.cols.data_ptr(), 1 if transpose_back else 0,
                                                       self.batch, stream_handle(stream)), "sharded 2-D FFT")
            return self.slab if transpose_back else self.cols
        self._plan_rows.execute(src, self.slab, self.batch * self.rows, stream)
        self._barrier(stream)
        outs = self._slab_arr if transpose_back else self._col_arr
        check(self._lib.dpp_fft2d_columns_sharded(self._plan2d._h, self._slab_arr, outs, self.world, self.rank,
                                                   1 if transpose_back else 0, self.batch, stream_handle(stream)),
              "sharded column pass")
        self._barrier(stream)
        return self.slab if transpose_back else self.cols

    def close(self) -> None:
        g = getattr(self, "_group", None)
        if g is not None and g.value:
            self._lib.dpp_peer_group_destroy(g)
            self._group = None
        for base in self._opened:
            self._lib.dpp_ipc_close(base)
        self._opened = []

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass


def encode_band(px: torch.Tensor, channels: int, height: int, width: int, codebook: torch.Tensor,
                band: tuple[int, int], out: tuple | None = None, stream=None):
    """Encode block rows [lo, hi) of one (height, width) frame on this GPU.

    px: the frame's pixels (height * width * channels uint8, CUDA); the band is
    a view (row offset 4*lo), so nothing is copied.  Returns (records
    (blocks, 3), cb (blocks,), cr (blocks,)) of the band: exactly the byte
    ranges [3*lo*bw, 3*hi*bw) and [lo*bw, hi*bw) of the single-GPU outputs."""
    from . import ops
    lo, hi = band
    bw = width // 4
    nb = (hi - lo) * bw
    rows = px.reshape(height, width * channels)[4 * lo:4 * hi]
    rec, cbp, crp = out if out is not None else (
        torch.empty((nb, 3), dtype=torch.uint8, device=px.device),
        torch.empty(nb, dtype=torch.uint8, device=px.device),
        torch.empty(nb, dtype=torch.uint8, device=px.device))
    if nb:
        ops.encode(rows, channels, 4 * (hi - lo), width, codebook, rec, cbp, crp, stream=stream)
    return rec, cbp, crp


def compress_tile_sharded(image, codebook, *, group=None, device=None, encode: Callable | None = None):
    """C4 across the ranks of ``group``: every rank passes the same frame
    ((h, w) gray or (h, w, 3|4) uint8, numpy or CUDA) and codebook; rank r
    encodes block rows shard_range(h/4, P, r) and the finished band bytes are
    all-gathered.  Returns the ``CompressedImage`` on every rank.

    ``encode(px, channels, h, w, codebook, band)`` defaults to the sm_100a
    encoder (``encode_band``); the gloo choreography tests inject a stand-in."""
    import numpy as np

    from .apps.imgc import CompressedImage, _validate_image
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    h, w, ch = _validate_image(image)
    bh, bw = h // 4, w // 4
    lo, hi = shard_range(bh, world, rank)
    cents = codebook.centroids if hasattr(codebook, "centroids") else codebook
    if encode is None:
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        px = image.to(dev).contiguous() if isinstance(image, torch.Tensor) else \
            torch.from_numpy(np.ascontiguousarray(image)).to(dev)
        cb_t = torch.as_tensor(np.ascontiguousarray(cents, np.float32)).to(dev) \
            if not isinstance(cents, torch.Tensor) else cents.to(dev, torch.float32).contiguous()
        rec, cbp, crp = encode_band(px.reshape(-1), ch, h, w, cb_t, (lo, hi))
        mine = torch.cat([rec.reshape(-1), cbp, crp]).cpu()
    else:
        rec, cbp, crp = encode(image, ch, h, w, cents, (lo, hi))
        mine = torch.cat([torch.as_tensor(np.ascontiguousarray(x)).reshape(-1) for x in (rec, cbp, crp)])
    # bands differ by at most one block row: pad to the largest, gather, trim
    most = (bh // world + (1 if bh % world else 0)) * bw * 5
    buf = torch.zeros(most, dtype=torch.uint8)
    buf[:mine.numel()] = mine
    parts = [torch.empty_like(buf) for _ in range(world)]
    if world > 1:
        on_gpu = dist.get_backend(group) == "nccl"  # NCCL gathers device buffers, gloo host ones
        gbuf = buf.to(torch.device("cuda", torch.cuda.current_device())) if on_gpu else buf
        gparts = [torch.empty_like(gbuf) for _ in range(world)]
        dist.all_gather(gparts, gbuf, group=group)
        parts = [p.cpu() for p in gparts]
    else:
        parts = [buf]
    recs, cbs, crs = [], [], []
    for r in range(world):
        a, b = shard_range(bh, world, r)
        nb = (b - a) * bw
        p = parts[r].numpy()
        recs.append(p[:3 * nb])
        cbs.append(p[3 * nb:4 * nb])
        crs.append(p[4 * nb:5 * nb])
    return CompressedImage.from_records(w, h, np.asarray(cents.cpu() if isinstance(cents, torch.Tensor) else cents,
                                                         np.float32),
                                        np.concatenate(recs), np.concatenate(cbs), np.concatenate(crs))


def fft1d_split(n: int, world: int) -> tuple[int, int]:
    """n = R x C for the sharded four-step: R = 2^ceil(lg n / 2) >= C, both
    multiples of the world size (every rank owns R/P rows and C/P columns)."""
    if n < 4 or n & (n - 1):
        raise ValueError(f"transform size must be a power of two >= 4, got {n}")
    lg = n.bit_length() - 1
    r = 1 << ((lg + 1) // 2)
    c = n // r
    if r % world or c % world:
        raise ValueError(f"{n} = {r} x {c} does not shard over {world} ranks")
    return r, c


def _default_twiddle(x: torch.Tensor, rows: int, cols: int, col0: int, n: int) -> torch.Tensor:
    from . import ops
    return ops.fft_twiddle(x, rows, cols, col0, n)


def fft1d_row_sharded(local: torch.Tensor, n: int, *, group=None, natural_output: bool = True,
                      row_fft: Callable | None = None, col_fft: Callable | None = None,
                      twiddle: Callable | None = None) -> torch.Tensor:
    """Forward 1-D FFT (the reference's fft(), apps/fft.py:150-174, unnormalised)
    of one n-point complex64 signal whose samples are split contiguously over
    the ranks of ``group``: ``local`` holds samples [p n/P, (p+1) n/P).

    Four-step with n = R x C (``fft1d_split``), M[r][c] = x[r C + c]:
      X[k_r + R k_c] = sum_c W_C^{c k_c} W_n^{c k_r} sum_r M[r][c] W_R^{r k_r}
    Each rank's row slab goes to column slabs (all-to-all), R-point column
    FFTs + twiddle run there, the result returns to row slabs (all-to-all) and
    C-point row FFTs finish: rank p then holds Z[k_r][k_c] = X[k_r + R k_c]
    for its R/P values of k_r (returned as (R/P, C) if not natural_output).
    natural_output: a third all-to-all and a local transpose give rank p the
    contiguous outputs X[p n/P .. (p+1) n/P).  The local transforms default
    to the sm_100a kernels; the gloo tests inject the oracle."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    r, c = fft1d_split(n, world)
    if local.numel() != n // world:
        raise ValueError(f"rank holds {local.numel()} samples, expected {n // world}")
    cw = c // world
    twiddle = twiddle or _default_twiddle
    inner = col_fft or _default_cols

    def columns(slab: torch.Tensor) -> torch.Tensor:  # (R, C/P): this rank's columns, all rows
        slab = inner(slab)
        return twiddle(slab, r, cw, rank * cw, n)

    z = fft2d_row_sharded(local.reshape(r // world, c), r, group=group, transpose_back=True,
                          row_fft=lambda x: x, col_fft=columns)
    z = (row_fft or _default_rows)(z.contiguous())
    if not natural_output:
        return z
    send = pack_column_blocks(z, world)             # (P, R/P, C/P): block s -> rank s (its k_c)
    recv = torch.empty_like(send)
    if world > 1:
        _all_to_all(recv, send, group)
    else:
        recv = send
    # rows k_r of every rank in order = Z[:, this rank's k_c]; X[k_r + R k_c] natural
    return recv.reshape(r, cw).t().contiguous().reshape(-1)
