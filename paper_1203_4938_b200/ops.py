"""Tensor-level entry points of the native nodes (thin wrappers over the C ABI).

Every function takes CUDA tensors, launches on the current (or given) stream
and returns without synchronising.  Shapes/dtypes are checked here so that a
bad call surfaces as the reference's exception type (``PlanError`` for size
rules, ``EngineRuntimeError``/``DeviceError`` for device faults) instead of a
crash inside the kernel.
"""

from __future__ import annotations

import ctypes as C
import threading

import torch

from . import _lib
from ._torch import require_cuda, stream_handle
from .errors import KernelRuntimeError, PlanError

__all__ = ["FftPlanHandle", "fft_plan", "fft_forward", "fft2d_forward", "leaf_dft",
           "ycbcr", "boxdown", "gradient", "vqnearest", "encode", "encode_planar", "decode", "fft2d_u8_spectrum"]


def _check_cuda(t: torch.Tensor, name: str, dtype: torch.dtype | None = None) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise PlanError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise PlanError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise PlanError(f"{name} must be {dtype}, got {t.dtype}")


def _f32_view(t: torch.Tensor) -> torch.Tensor:
    return torch.view_as_real(t) if t.is_complex() else t


# ---------------------------------------------------------------------------
# FFT

class FftPlanHandle:
    """Owns one dpp_fft_plan (rank 1 or 2) for up to ``batch`` transforms."""

    def __init__(self, rank: int, n0: int, n1: int, batch: int, device: torch.device):
        lib = _lib.load()
        self.rank, self.n0, self.n1, self.batch, self.device = rank, n0, n1, batch, device
        h = C.c_void_p()
        ws = C.c_size_t()
        with torch.cuda.device(device):
            _lib.check(lib.dpp_fft_plan_create(C.byref(h), rank, n0, n1, batch, C.byref(ws)),
                       "fft plan")
        self._h = h
        self.workspace_bytes = ws.value
        buf = C.create_string_buffer(256)
        lib.dpp_fft_plan_describe(h, buf, 256)
        self.description = buf.value.decode()

    @property
    def points(self) -> int:
        return self.n0 * (self.n1 if self.rank == 2 else 1)

    def execute(self, src: torch.Tensor, dst: torch.Tensor, batch: int | None = None,
                stream: torch.cuda.Stream | None = None) -> None:
        batch = self.batch if batch is None else batch
        _lib.check(_lib.load().dpp_fft_c2c_forward_batch(self._h, src.data_ptr(), dst.data_ptr(),
                                                         batch, None, stream_handle(stream)),
                   "fft execute")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().dpp_fft_plan_destroy(h)
            except Exception:  # interpreter shutdown
                pass


_plans: dict[tuple, FftPlanHandle] = {}
_plans_lock = threading.Lock()


def fft_shape_supported(rank: int, n0: int, n1: int = 1) -> bool:
    """Would a plan of this shape be accepted?  Pure shape rules (C ABI
    dpp_fft_plan_supported): no device, no allocation."""
    return bool(_lib.load().dpp_fft_plan_supported(rank, n0, n1))


_pin = threading.local()


class pin_plans:
    """Collect every plan handed out in this thread while active: a CUDA graph
    captured meanwhile (client._Replay) bakes the plans' tables and scratch
    into its kernel nodes, so it keeps them alive even after the cache
    replaces a plan with a larger one."""

    def __enter__(self) -> list:
        self.prev = getattr(_pin, "plans", None)
        _pin.plans = []
        return _pin.plans

    def __exit__(self, *exc):
        _pin.plans = self.prev
        return False


def fft_plan(rank: int, n0: int, n1: int, batch: int, device=None) -> FftPlanHandle:
    """Cached plan with capacity >= batch (grown geometrically)."""
    dev = require_cuda(device)
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (rank, n0, n1 if rank == 2 else 1, dev.index)
    with _plans_lock:
        p = _plans.get(key)
        if p is None or p.batch < batch:
            cap = max(batch, 2 * p.batch if p is not None else batch, 1)
            p = FftPlanHandle(rank, n0, n1 if rank == 2 else 1, cap, dev)
            _plans[key] = p
    pins = getattr(_pin, "plans", None)
    if pins is not None:
        pins.append(p)
    return p


def fft_forward(x: torch.Tensor, n: int, out: torch.Tensor | None = None,
                stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Batched 1-D forward FFT over the last ``n`` complex64 samples of x."""
    _check_cuda(x, "x")
    if x.dtype != torch.complex64:
        raise PlanError(f"x must be complex64, got {x.dtype}")
    total = x.numel()
    if n < 2 or n & (n - 1):
        raise PlanError(f"transform size must be a power of two, got {n}")
    if total % n:
        raise PlanError(f"{total} samples is not a whole number of {n}-point signals")
    out = torch.empty_like(x) if out is None else out
    _check_cuda(out, "out", torch.complex64)
    batch = total // n
    if batch:
        fft_plan(1, n, 1, batch, x.device).execute(x, out, batch, stream)
    return out


def fft2d_forward(x: torch.Tensor, n0: int, n1: int, out: torch.Tensor | None = None,
                  stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Batched 2-D forward FFT of n0 x n1 row-major complex64 images."""
    _check_cuda(x, "x")
    if x.dtype != torch.complex64:
        raise PlanError(f"x must be complex64, got {x.dtype}")
    if x.numel() % (n0 * n1):
        raise PlanError(f"{x.numel()} samples is not a whole number of {n0}x{n1} images")
    out = torch.empty_like(x) if out is None else out
    _check_cuda(out, "out", torch.complex64)
    batch = x.numel() // (n0 * n1)
    if batch:
        fft_plan(2, n0, n1, batch, x.device).execute(x, out, batch, stream)
    return out


def fft_twiddle(x: torch.Tensor, rows: int, cols: int, col0: int, n: int,
                stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """In place: x[r][c] *= W_n^{r (col0 + c)} on a rows x cols complex64 block."""
    _check_cuda(x, "x", torch.complex64)
    if x.numel() != rows * cols:
        raise PlanError(f"twiddle block holds {x.numel()} samples, expected {rows} x {cols}")
    _lib.check(_lib.load().dpp_fft_twiddle(x.data_ptr(), rows, cols, col0, n, stream_handle(stream)),
               "fft twiddle")
    return x


def fft_columns(x: torch.Tensor, n0: int, n1: int, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """In place: n0-point FFT of every column of batched n0 x n1 row-major arrays."""
    _check_cuda(x, "x", torch.complex64)
    if x.numel() % (n0 * n1):
        raise PlanError(f"{x.numel()} samples is not a whole number of {n0}x{n1} arrays")
    batch = x.numel() // (n0 * n1)
    if batch:
        plan = fft_plan(2, n0, n1, batch, x.device)
        _lib.check(_lib.load().dpp_fft_c2c_columns(plan._h, x.data_ptr(), batch, stream_handle(stream)),
                   "fft columns")
    return x


def leaf_dft(k: int, x: torch.Tensor, y: torch.Tensor, stream=None) -> None:
    """dft{2^k} leaf node over float{2^(k+1)} work-items (bit-exact with the reference)."""
    _check_cuda(x, "x", torch.float32)
    _check_cuda(y, "y", torch.float32)
    width = 2 << k
    if x.numel() % width or y.numel() != x.numel():
        raise PlanError("leaf buffers must hold whole work-items of equal count")
    _lib.check(_lib.load().dpp_fft_leaf(k, x.data_ptr(), y.data_ptr(), x.numel() // width,
                                        stream_handle(stream)), f"dft{1 << k}")


# ---------------------------------------------------------------------------
# image codec nodes

def ycbcr(rgba: torch.Tensor, yl, cb, cr, stream=None) -> None:
    _check_cuda(rgba, "rgb", torch.uint8)
    n = rgba.numel() // 4
    for t, name in ((yl, "yl"), (cb, "cb"), (cr, "cr")):
        _check_cuda(t, name, torch.float32)
    _lib.check(_lib.load().dpp_imgc_ycbcr(rgba.data_ptr(), yl.data_ptr(), cb.data_ptr(), cr.data_ptr(),
                                          n, stream_handle(stream)), "ycbcr")


def boxdown(blk: torch.Tensor, avg: torch.Tensor, stream=None) -> None:
    _check_cuda(blk, "blk", torch.float32)
    _check_cuda(avg, "avg", torch.float32)
    _lib.check(_lib.load().dpp_imgc_boxdown(blk.data_ptr(), avg.data_ptr(), blk.numel() // 16,
                                            stream_handle(stream)), "boxdown")


def gradient(lum: torch.Tensor, dx, dy, width: int, height: int, stream=None) -> None:
    _check_cuda(lum, "lum", torch.float32)
    fault = C.c_int64(-1)
    rc = _lib.load().dpp_imgc_gradient(lum.data_ptr(), dx.data_ptr(), dy.data_ptr(), width, height,
                                       lum.numel(), C.byref(fault), stream_handle(stream))
    if rc == _lib.DPP_EINVAL and fault.value >= 0:
        raise KernelRuntimeError(_lib.last_error(), work_item=fault.value)
    _lib.check(rc, "gradient")


def vqnearest(blk: torch.Tensor, cbk: torch.Tensor, idx: torch.Tensor, codebook_size: int,
              stream=None) -> None:
    _check_cuda(blk, "blk", torch.float32)
    _check_cuda(cbk, "cbk", torch.float32)
    _check_cuda(idx, "idx", torch.int32)
    items = blk.numel() // 16
    cbk_items = cbk.numel() // 16
    if items and codebook_size > cbk_items:
        raise KernelRuntimeError(f"index {cbk_items} out of range for point 'cbk' (0..{cbk_items - 1})",
                                 work_item=0)
    _lib.check(_lib.load().dpp_imgc_vqnearest(blk.data_ptr(), cbk.data_ptr(), idx.data_ptr(), items,
                                              cbk_items, codebook_size, stream_handle(stream)),
               "vqnearest")


def encode(px: torch.Tensor, channels: int, height: int, width: int, codebook: torch.Tensor,
           records: torch.Tensor, cb_plane: torch.Tensor, cr_plane: torch.Tensor,
           block_grad: torch.Tensor | None = None, norm32: torch.Tensor | None = None,
           batch: int = 1, shared_codebook: bool = True, sigma_min: float = 0.25,
           stream=None) -> None:
    """Fused forward block transform + quantise + order for `batch` images."""
    _check_cuda(px, "px", torch.uint8)
    _check_cuda(codebook, "codebook", torch.float32)
    ncb = codebook.numel() // 16 if shared_codebook else codebook.numel() // (16 * batch)
    image_bytes = height * width * channels
    if px.numel() < batch * image_bytes:
        raise PlanError(f"pixel buffer holds {px.numel()} bytes, need {batch * image_bytes}")
    _lib.check(_lib.load().dpp_imgc_encode(
        px.data_ptr(), channels, height, width, width * channels, image_bytes, batch,
        codebook.data_ptr(), ncb, 0 if shared_codebook else ncb * 16, float(sigma_min),
        records.data_ptr(), cb_plane.data_ptr(), cr_plane.data_ptr(), _lib.ptr(block_grad),
        _lib.ptr(norm32), stream_handle(stream)), "imgc encode")


def encode_planar(px: torch.Tensor, height: int, width: int, codebook: torch.Tensor, mu: torch.Tensor,
                  sig: torch.Tensor, idx: torch.Tensor, cb_plane: torch.Tensor, cr_plane: torch.Tensor,
                  channels: int = 1, batch: int = 1, shared_codebook: bool = True, sigma_min: float = 0.25,
                  stream=None) -> None:
    """:func:`encode` with the record bytes written as three planes (the graph
    node's mu / sig / idx outputs) instead of the interleaved record run."""
    _check_cuda(px, "px", torch.uint8)
    _check_cuda(codebook, "codebook", torch.float32)
    blocks = (height // 4) * (width // 4) * batch
    for name, t in (("mu", mu), ("sig", sig), ("idx", idx), ("cb_plane", cb_plane), ("cr_plane", cr_plane)):
        _check_cuda(t, name, torch.uint8)
        if t.numel() < blocks:
            raise PlanError(f"{name} holds {t.numel()} bytes, need {blocks}")
    ncb = codebook.numel() // 16 if shared_codebook else codebook.numel() // (16 * batch)
    image_bytes = height * width * channels
    if px.numel() < batch * image_bytes:
        raise PlanError(f"pixel buffer holds {px.numel()} bytes, need {batch * image_bytes}")
    _lib.check(_lib.load().dpp_imgc_encode_planar(
        px.data_ptr(), channels, height, width, width * channels, image_bytes, batch,
        codebook.data_ptr(), ncb, 0 if shared_codebook else ncb * 16, float(sigma_min),
        mu.data_ptr(), sig.data_ptr(), idx.data_ptr(), cb_plane.data_ptr(), cr_plane.data_ptr(),
        stream_handle(stream)), "imgc encode (planar)")


def rounding_ties(px: torch.Tensor, channels: int, height: int, width: int, batch: int = 1,
                  stream=None) -> tuple[int, int]:
    """(mean, sigma) rounding-tie counts of the encoder's binary64 quantisers.

    A tie is a block whose mean (or sigma / 0.25) lies within 1e-9 of a
    half-integer, where rint() (imgc.py:398-401) depends on the last bits; the
    encoder reproduces those bits exactly, so ties are reported, not errors."""
    _check_cuda(px, "px", torch.uint8)
    image_bytes = height * width * channels
    if px.numel() < batch * image_bytes:
        raise PlanError(f"pixel buffer holds {px.numel()} bytes, need {batch * image_bytes}")
    ties = torch.zeros(2, dtype=torch.int64, device=px.device)
    _lib.check(_lib.load().dpp_imgc_rounding_ties(
        px.data_ptr(), channels, height, width, width * channels, image_bytes, batch, ties.data_ptr(),
        stream_handle(stream)), "imgc rounding ties")
    m, s = ties.tolist()
    return int(m), int(s)


def u8_to_complex(x: torch.Tensor, y: torch.Tensor, stream=None) -> None:
    _check_cuda(x, "x", torch.uint8)
    _check_cuda(y, "y")
    _lib.check(_lib.load().dpp_u8_to_complex(x.data_ptr(), y.data_ptr(), x.numel(), stream_handle(stream)),
               "to_complex")


def fft2d_u8_spectrum(x: torch.Tensor, rows: int, cols: int, alpha: float, out: torch.Tensor,
                      stream=None) -> bool:
    """Fused to_complex -> 2-D FFT -> spectrum_u8 over batches of rows x cols u8
    images (two passes; the complex intermediate is a scratch tensor).  Returns
    False (and does nothing) when the shape has no fused schedule."""
    _check_cuda(x, "x", torch.uint8)
    _check_cuda(out, "out", torch.uint8)
    n = rows * cols
    if x.numel() % n or out.numel() != x.numel():
        raise PlanError("fused 2-D spectrum: sizes must be whole images and match")
    batch = x.numel() // n
    if batch == 0:
        return True
    plan = fft_plan(2, rows, cols, batch, x.device)
    work = torch.empty(2 * x.numel(), dtype=torch.float32, device=x.device)
    if stream is not None:
        work.record_stream(stream)
    rc = _lib.load().dpp_fft2d_u8_spectrum(plan._h, x.data_ptr(), out.data_ptr(), float(alpha), work.data_ptr(),
                                           batch, stream_handle(stream))
    if rc == _lib.DPP_ENOTSUP:
        return False
    _lib.check(rc, "fft2d_u8_spectrum")
    return True


def spectrum_u8(z: torch.Tensor, y: torch.Tensor, alpha: float, stream=None) -> None:
    _check_cuda(z, "z")
    _check_cuda(y, "y", torch.uint8)
    _lib.check(_lib.load().dpp_spectrum_u8(z.data_ptr(), y.data_ptr(), y.numel(), float(alpha),
                                           stream_handle(stream)), "spectrum_u8")


def decode(records, cb_plane, cr_plane, codebook, height: int, width: int, rgb, stream=None) -> None:
    _lib.check(_lib.load().dpp_imgc_decode(records.data_ptr(), cb_plane.data_ptr(), cr_plane.data_ptr(),
                                           codebook.data_ptr(), codebook.numel() // 16, height, width,
                                           rgb.data_ptr(), stream_handle(stream)), "imgc decode")
