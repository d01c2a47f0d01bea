"""PyTorch plumbing: device buffers, streams, pinned host staging.

PyTorch is used only to allocate device memory and to own CUDA streams;
every computation on the hot path is a libdpp_b200.so kernel.
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import NativeLibraryError
from .types import DataType

_TORCH_DTYPES = {
    "char": torch.int8, "uchar": torch.uint8, "short": torch.int16, "ushort": torch.uint16,
    "int": torch.int32, "uint": torch.uint32, "long": torch.int64, "ulong": torch.uint64,
    "float": torch.float32,
}


def torch_dtype(dt: DataType) -> torch.dtype:
    return _TORCH_DTYPES[dt.base]


_CUDA_OK: bool | None = None


def require_cuda(device=None) -> torch.device:
    global _CUDA_OK
    if not _CUDA_OK:  # a positive answer is cached (the per-call NVML query showed in C1 latency)
        _CUDA_OK = torch.cuda.is_available()
        if not _CUDA_OK:
            raise NativeLibraryError("no CUDA device: the B200 nodes have no CPU fallback")
    dev = torch.device("cuda" if device is None else device)
    if dev.type != "cuda":
        raise NativeLibraryError(f"device {dev} is not a CUDA device")
    return dev


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def to_device(values: np.ndarray, device="cuda", pinned: bool = True) -> torch.Tensor:
    """Host numpy -> device tensor (via pinned staging for async H2D)."""
    dev = require_cuda(device)
    host = torch.from_numpy(np.ascontiguousarray(values))
    if pinned:
        host = host.pin_memory()
    return host.to(dev, non_blocking=pinned)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


class nvtx_range:
    """NVTX range around host-side launch code (SURVEY §5 tracing): visible in
    nsys / ncu --nvtx timelines as ``dpp:<name>``; a no-op cost when no tool
    is attached (one C call each way)."""

    __slots__ = ("name",)

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        torch.cuda.nvtx.range_push("dpp:" + self.name)
        return self

    def __exit__(self, *exc):
        torch.cuda.nvtx.range_pop()
        return False
