"""GPU k-means codebook training — see train_codebook_device."""

from __future__ import annotations


def kmeans_device(blocks, size, seed, max_iter=20, trace=None, device=None):
    raise NotImplementedError("GPU k-means is not built yet: pass codebook= to compress()")


def train_codebook_device(px, ch, h, w, size, seed, sigma_min, grad_min):
    raise NotImplementedError("GPU k-means is not built yet: pass codebook= to compress()")
