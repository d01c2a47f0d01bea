"""GPU k-means codebook training.

The reference trains the codebook on the host (imgc.py:384-393 + kmeans
imgc.py:221-273).  Here both steps run on the device:

1. ``dpp_imgc_block_stats``: per block the gradient training filter and the
   binary64 normalised block (bit-identical to the reference's values);
2. selection of blocks with gradient >= grad_min (all blocks if none);
3. ``dpp_kmeans``: k-means++ seeding driven by the SAME numpy RNG stream the
   reference consumes (``default_rng(seed)``: one ``integers(n)`` then one
   ``random()`` per further centroid), then Lloyd iterations in binary64.

The codebook is tolerance-equal to the reference's, not bit-equal: the
reference's nearest-centroid step uses an OpenBLAS GEMM and its k-means++
sampling a sequential cumulative sum, both CPU/BLAS dependent.
Bit-exact bitstream parity therefore feeds the node the oracle's codebook.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._torch import require_cuda, stream_handle
from .errors import PlanError

__all__ = ["kmeans_device", "block_stats_device", "train_codebook_device"]


def block_stats_device(px: torch.Tensor, channels: int, h: int, w: int, sigma_min: float = 0.25):
    """(norm64 (blocks, 16) float64, block_grad (blocks,) float32) on the device."""
    nb = (h // 4) * (w // 4)
    norm64 = torch.empty((nb, 16), dtype=torch.float64, device=px.device)
    grad = torch.empty(nb, dtype=torch.float32, device=px.device)
    _lib.check(_lib.load().dpp_imgc_block_stats(px.data_ptr(), channels, h, w, w * channels, h * w * channels,
                                                1, float(sigma_min), norm64.data_ptr(), grad.data_ptr(),
                                                stream_handle()), "block stats")
    return norm64, grad


def kmeans_device(blocks, size: int, seed: int, max_iter: int = 20, trace: list | None = None,
                  device=None) -> torch.Tensor:
    """k-means++ + Lloyd on the GPU; returns (size, 16) float32 centroids on the device."""
    dev = require_cuda(device if not isinstance(blocks, torch.Tensor) else blocks.device)
    pts = blocks if isinstance(blocks, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(blocks, np.float64))
    pts = pts.to(dev, torch.float64).contiguous()
    n = pts.shape[0]
    if n == 0:
        raise ValueError("no blocks to cluster")
    if size > n:
        raise ValueError(f"codebook size {size} exceeds {n} training blocks")
    if pts.dim() != 2 or pts.shape[1] != 16:
        raise PlanError("k-means points must be (n, 16)")
    rng = np.random.default_rng(seed)
    first = int(rng.integers(n))
    uniforms = (C.c_double * max(size - 1, 1))(*rng.random(max(size - 1, 0)).tolist())
    out = torch.empty((size, 16), dtype=torch.float32, device=dev)
    tr = (C.c_double * max(max_iter, 1))()
    iters = C.c_int(0)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().dpp_kmeans(pts.data_ptr(), n, size, first, uniforms, max_iter, out.data_ptr(),
                                          tr, C.byref(iters), stream_handle()), "kmeans")
    if trace is not None:
        trace.extend(float(tr[i]) for i in range(iters.value))
    return out


def train_codebook_device(px: torch.Tensor, channels: int, h: int, w: int, size: int, seed: int,
                          sigma_min: float = 0.25, grad_min: float = 1.0) -> torch.Tensor:
    """imgc.py:384-393 on the device: filter by gradient, then k-means."""
    norm64, grad = block_stats_device(px, channels, h, w, sigma_min)
    keep = torch.nonzero(grad >= grad_min).squeeze(1)
    train = norm64.index_select(0, keep) if keep.numel() else norm64
    return kmeans_device(train, min(size, train.shape[0]), seed)
