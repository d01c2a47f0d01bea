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

__all__ = ["kmeans_device", "block_stats_device", "train_codebook_device", "kmeans_sharded", "CudaShard"]


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


# ---------------------------------------------------------------------------
# multi-GPU: points sharded across ranks, one all-reduce per step


class CudaShard:
    """This rank's slice of the training points on its GPU (C-ABI
    ``dpp_kmeans_shard_*``, include/dpp_b200.h)."""

    def __init__(self, pts: torch.Tensor, k: int):
        self.pts = pts.to(torch.float64).contiguous()
        self.n, self.k, self.device = self.pts.shape[0], k, self.pts.device
        self._lib = _lib.load()
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._lib.dpp_kmeans_shard_create(C.byref(h), self.pts.data_ptr(), self.n, k,
                                                         stream_handle()), "k-means shard")
        self._h = h

    def seed(self, centroid: torch.Tensor, first: bool) -> float:
        t = C.c_double()
        _lib.check(self._lib.dpp_kmeans_shard_seed(self._h, centroid.data_ptr(), int(first), C.byref(t)),
                   "k-means++ step")
        return t.value

    def pick(self, target: float, local_index: int, out: torch.Tensor) -> int:
        got = C.c_int64()
        _lib.check(self._lib.dpp_kmeans_shard_pick(self._h, float(target), int(local_index), out.data_ptr(),
                                                   C.byref(got)), "k-means++ pick")
        return got.value

    def assign(self, cents: torch.Tensor) -> torch.Tensor:
        acc = torch.empty(self.k * 16 + self.k + 2, dtype=torch.float64, device=self.device)
        _lib.check(self._lib.dpp_kmeans_shard_assign(self._h, cents.data_ptr(), acc.data_ptr()), "Lloyd assign")
        return acc

    def far(self, cents: torch.Tensor, base: int) -> torch.Tensor:
        packed = torch.empty(1, dtype=torch.int64, device=self.device)
        _lib.check(self._lib.dpp_kmeans_shard_far(self._h, cents.data_ptr(), int(base), packed.data_ptr()),
                   "farthest point")
        return packed

    def set_assign(self, local_index: int, cluster: int) -> None:
        _lib.check(self._lib.dpp_kmeans_shard_set_assign(self._h, int(local_index), int(cluster)), "reseed")

    def point(self, local_index: int) -> torch.Tensor:
        return self.pts[local_index]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.dpp_kmeans_shard_destroy(h)
            except Exception:  # interpreter shutdown
                pass


def kmeans_sharded(local_pts: torch.Tensor, size: int, seed: int, max_iter: int = 20, trace: list | None = None,
                   group=None, shard=None) -> torch.Tensor:
    """imgc.py:221-273 over training points split contiguously across the
    ranks of ``group`` (rank r holds global points [offs[r], offs[r] + n_r)).

    Every rank gets the same (size, 16) float32 codebook.  Per k-means++ step
    one all-reduce of the per-rank d2 totals (the owner of the drawn point
    broadcasts it); per Lloyd iteration one all-reduce of the k*16 + k + 2
    accumulator; per empty cluster one MAX all-reduce for the farthest point.
    ``shard`` defaults to the GPU shard (``CudaShard``); the CPU tests inject
    a numpy shard with the same methods to check the choreography with gloo."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    shard = shard if shard is not None else CudaShard(local_pts, size)
    dev = shard.device

    def gather_scalar(v: float) -> list[float]:
        vec = torch.zeros(world, dtype=torch.float64, device=dev)
        vec[rank] = v
        if world > 1:
            dist.all_reduce(vec, group=group)
        return vec.tolist()

    counts = [int(c) for c in gather_scalar(float(shard.n))]
    offs = [sum(counts[:r]) for r in range(world)]
    total_n = sum(counts)
    if total_n == 0:
        raise ValueError("no blocks to cluster")
    if size > total_n:
        raise ValueError(f"codebook size {size} exceeds {total_n} training blocks")

    def owner_of(g: int) -> int:
        for r in range(world):
            if offs[r] <= g < offs[r] + counts[r]:
                return r
        raise AssertionError(g)

    def bcast(t: torch.Tensor, src: int) -> None:
        if world > 1:
            dist.broadcast(t, src=src, group=group)  # group-local src == global rank for the default group

    cents = torch.zeros((size, 16), dtype=torch.float64, device=dev)
    rng = np.random.default_rng(seed)
    first = int(rng.integers(total_n))
    uniforms = rng.random(max(size - 1, 0))

    def take(g: int, j: int) -> None:
        r = owner_of(g)
        if rank == r:
            shard.pick(0.0, g - offs[r], cents[j])
        bcast(cents[j], r)

    take(first, 0)
    for j in range(1, size):
        totals = gather_scalar(shard.seed(cents[j - 1], j == 1))
        total = 0.0
        for t in totals:
            total += t
        u = float(uniforms[j - 1])
        if total <= 0.0:
            take(min(int(u * total_n), total_n - 1), j)
            continue
        target, acc, r = u * total, 0.0, 0
        last = max(q for q in range(world) if counts[q])
        for r in range(world):
            if counts[r] and (r == last or acc + totals[r] > target):
                break
            acc += totals[r]
        if rank == r:
            shard.pick(target - acc, -1, cents[j])
        bcast(cents[j], r)

    def assign_all() -> torch.Tensor:
        a = shard.assign(cents)
        if world > 1:
            dist.all_reduce(a, group=group)
        return a

    k = size
    acc = assign_all()
    it = 0
    while it < max_iter:
        cnt = acc[k * 16:k * 16 + k]
        sums = acc[:k * 16].view(k, 16)
        cents = torch.where(cnt[:, None] > 0, sums / cnt.clamp(min=1)[:, None], cents)
        for j in torch.nonzero(cnt == 0).flatten().tolist():
            packed = shard.far(cents, offs[rank])
            if world > 1:
                dist.all_reduce(packed, op=dist.ReduceOp.MAX, group=group)
            g = 0xFFFFFFFF - (int(packed.item()) & 0xFFFFFFFF)
            r = owner_of(g)
            if rank == r:
                shard.set_assign(g - offs[r], j)
                cents[j] = shard.point(g - offs[r])
            bcast(cents[j], r)
        acc = assign_all()
        if trace is not None:
            trace.append(float(acc[-1]))
        it += 1
        if float(acc[-2]) == 0.0:
            break
    return cents.to(torch.float32)
