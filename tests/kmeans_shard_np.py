"""numpy stand-in for ``kmeans.CudaShard`` (test infrastructure): the same
per-shard steps (k-means++ update / pick, Lloyd assign, farthest point) in
binary64 numpy, so the sharded driver's collectives can be checked with gloo
on CPU."""

from __future__ import annotations

import numpy as np
import torch


class NumpyShard:
    def __init__(self, pts: np.ndarray, k: int):
        self.p = np.ascontiguousarray(pts, dtype=np.float64)
        self.pts = torch.from_numpy(self.p)
        self.n, self.k, self.device = self.p.shape[0], k, torch.device("cpu")
        self.d2 = np.zeros(self.n)
        self.a = np.full(self.n, -1)

    def seed(self, centroid: torch.Tensor, first: bool) -> float:
        d = ((self.p - centroid.numpy()) ** 2).sum(1)
        self.d2 = d if first else np.minimum(self.d2, d)
        return float(self.d2.sum())

    def pick(self, target: float, local_index: int, out: torch.Tensor) -> int:
        i = local_index
        if i < 0:
            i = min(int(np.searchsorted(np.cumsum(self.d2), target, side="right")), self.n - 1)
        out.copy_(self.pts[i])
        return i

    def assign(self, cents: torch.Tensor) -> torch.Tensor:
        k = self.k
        d = ((self.p[:, None, :] - cents.numpy()[None]) ** 2).sum(-1)
        a = d.argmin(1) if self.n else np.zeros(0, dtype=np.int64)
        changed = int((a != self.a).sum())
        self.a = a
        sums = np.zeros((k, 16))
        np.add.at(sums, a, self.p)
        cnt = np.bincount(a, minlength=k).astype(np.float64)
        sse = float(d[np.arange(self.n), a].sum()) if self.n else 0.0
        return torch.from_numpy(np.concatenate([sums.ravel(), cnt, [changed, sse]]))

    def far(self, cents: torch.Tensor, base: int) -> torch.Tensor:
        if self.n == 0:
            return torch.zeros(1, dtype=torch.int64)
        d = ((self.p - cents.numpy()[self.a]) ** 2).sum(1).astype(np.float32)
        key = (d.view(np.uint32).astype(np.int64) << 32) | (0xFFFFFFFF - (base + np.arange(self.n)))
        return torch.tensor([int(key.max())], dtype=torch.int64)

    def set_assign(self, local_index: int, cluster: int) -> None:
        self.a[local_index] = cluster

    def point(self, local_index: int) -> torch.Tensor:
        return self.pts[local_index]
