"""C5: the full graph FFT -> compression on a batch of images, device-resident edges.

The chain is defined by SURVEY §8(d) C5 (the reference has no such graph):
gray u8 image -> complex64 (g, 0) -> 2-D FFT -> u8 log-magnitude adapter
``clip(floor(alpha * log(1 + |X|)), 0, 255)`` -> block compression.

``chain_program`` builds it as ONE reference-format document (four
instances, three arrows).  ``to_complex`` and ``spectrum_u8`` are written in
the kernel language so the reference engine can run them; ``fft2d_RxC`` is
the self-describing naive-DFT node and ``imgc_encode`` the fused codec node
(apps/fft.py, apps/imgc.py).  Executed by this framework, every edge is a
device tensor handed from producer to consumer (executor.run_chunk) — the
host only ships pixels in and records out.
"""

from __future__ import annotations

import numpy as np

from ..client import CudaBackend, run
from ..model import Arrow, Instance, Node, Program
from ..types import DataType, Direction, IOPoint
from ..wire import DeviceStream, StreamFile
from .fft import fft2d_kernel
from .imgc import encode_kernel

__all__ = ["ALPHA", "to_complex_kernel", "spectrum_u8_kernel", "chain_program", "run_chain"]

ALPHA = 11.5  # 255 / log(1 + 2^31): the DC of a 4096^2 u8 image stays below 255


def to_complex_kernel() -> Node:
    body = ("int i = get_global_id(0);\n"
            "y[i] = (float2)((float)(x[i]), 0.0f);\n")
    return Node("to_complex", body, (IOPoint("x", DataType("uchar"), Direction.INPUT),
                                      IOPoint("y", DataType("float", 2), Direction.OUTPUT)))


def spectrum_u8_kernel(alpha: float = ALPHA) -> Node:
    lit = np.format_float_positional(np.float32(alpha), unique=True)
    body = ("int i = get_global_id(0);\n"
            "float2 z = x[i];\n"
            "float m = sqrt(z.x * z.x + z.y * z.y);\n"
            f"float v = floor({lit}f * log(1.0f + m));\n"
            "y[i] = (uchar)(fmin(fmax(v, 0.0f), 255.0f));\n")
    return Node("spectrum_u8", body, (IOPoint("x", DataType("float", 2), Direction.INPUT),
                                       IOPoint("y", DataType("uchar"), Direction.OUTPUT)))


def chain_program(width: int, height: int, codebook_size: int = 256, alpha: float = ALPHA) -> Program:
    """gray -> complex -> fft2d -> spectrum_u8 -> imgc_encode, one document."""
    nodes = [to_complex_kernel(), fft2d_kernel(height, width), spectrum_u8_kernel(alpha),
             encode_kernel(width, height, codebook_size)]
    return Program({n.name: n for n in nodes},
                   tuple(Instance(i, n.name) for i, n in enumerate(nodes)),
                   (Arrow((0, "y"), (1, "x")), Arrow((1, "y"), (2, "x")), Arrow((2, "y"), (3, "px"))))


def run_chain(images, codebooks, *, backend: CudaBackend | None = None, alpha: float = ALPHA) -> dict:
    """Run the chain over (B, h, w) gray images with (B, n, 16) or (n, 16) codebooks.

    Accepts numpy arrays (staged once) or CUDA tensors (nothing crosses the
    bus on the way in); returns the encode node's free outputs keyed
    mu/sig/idx/cb/cr (host arrays, or device tensors with
    ``CudaBackend(outputs="device")``)."""
    import torch
    b, h, w = images.shape
    ncb = codebooks.shape[-2]
    prog = chain_program(w, h, ncb, alpha)
    if isinstance(images, torch.Tensor):
        px = DeviceStream(DataType("uchar"), images.reshape(-1))
        cbk = DeviceStream(DataType("float", 16), codebooks.reshape(-1).to(images.device, torch.float32))
    else:
        px = StreamFile(DataType("uchar"), np.ascontiguousarray(images, np.uint8).reshape(-1))
        cbk = StreamFile(DataType("float", 16), np.ascontiguousarray(codebooks, np.float32).reshape(-1))
    out = run(backend or CudaBackend(), prog, {"0.x": px, "3.cbk": cbk})
    return {k.split(".")[1]: (v.tensor if isinstance(v, DeviceStream) else v.values) for k, v in out.items()}
