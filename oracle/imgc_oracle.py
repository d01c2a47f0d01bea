"""CPU oracle for the block-compression node — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU arms may
import this module; the product (``paper_1203_4938_b200``) never does.

Vectorised numpy restatement of /root/reference/pkg/src/dpp/apps/imgc.py,
written independently, reproducing the reference arithmetic bit-for-bit:

* ``ycbcr``          imgc.py:128-140  binary32, left to right, no contraction
* ``boxdown``        imgc.py:143-152 + :374-375   sequential binary32 sum * 0.0625f, rint/clip
* ``gradient``       imgc.py:155-166 + :380-381   forward differences, float32 hypot, block mean
* ``to_blocks``      imgc.py:192-201  raster block order, row-major 16-vectors
* ``block_stats``    imgc.py:384-388  binary64 mean/std (numpy pairwise-8), normalisation
* ``vq_nearest``     imgc.py:169-185 + interp.py:417-419  binary32 dot in pairwise order,
                     strict <, best initialised to float32(3.402823e38)
* ``kmeans``         imgc.py:221-273  k-means++ + Lloyd, binary64, same RNG stream
* ``encode``         imgc.py:343-403  everything above; the codebook may be given
* ``to_bytes``/``from_bytes``  imgc.py:279-337  the DPVQ container
* ``decode``         imgc.py:426-439
* ``synthetic_image``, ``psnr``   imgc.py:92-117 (fixtures)

Parity is pinned by tests/test_oracle.py against bitstreams produced by the
reference ``compress()`` (tests/golden/imgc_golden.npz via
tests/golden/make_golden.py).
"""

from __future__ import annotations

import struct

import numpy as np

__all__ = ["SIGMA_STEP", "MAGIC", "ycbcr", "boxdown", "gradient", "to_blocks", "from_blocks",
           "block_stats", "vq_nearest", "kmeans", "encode", "compress", "to_bytes", "from_bytes",
           "decode", "synthetic_image", "psnr", "train_codebook"]

MAGIC = b"DPVQ"
SIGMA_STEP = 0.25
_HEADER = struct.Struct("<4sIIHf")
_F = np.float32


def ycbcr(rgb: np.ndarray) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(..., 3) uint8 -> three float32 planes."""
    r, g, b = (rgb[..., i].astype(_F) for i in range(3))
    y = (_F(0.299) * r + _F(0.587) * g) + _F(0.114) * b
    cb = ((_F(128.0) - _F(0.168736) * r) - _F(0.331264) * g) + _F(0.5) * b
    cr = ((_F(128.0) + _F(0.5) * r) - _F(0.418688) * g) - _F(0.081312) * b
    return y, cb, cr


def to_blocks(plane: np.ndarray) -> np.ndarray:
    h, w = plane.shape
    return plane.reshape(h // 4, 4, w // 4, 4).swapaxes(1, 2).reshape(-1, 16)


def from_blocks(blocks: np.ndarray, h: int, w: int) -> np.ndarray:
    return blocks.reshape(h // 4, w // 4, 4, 4).swapaxes(1, 2).reshape(h, w)


def boxdown(plane: np.ndarray) -> np.ndarray:
    """Chroma plane -> (h/4, w/4) uint8."""
    h, w = plane.shape
    blk = to_blocks(plane)
    acc = blk[:, 0].copy()
    for m in range(1, 16):
        acc = acc + blk[:, m]
    return np.clip(np.rint(acc * _F(0.0625)), 0, 255).astype(np.uint8).reshape(h // 4, w // 4)


def _pw16(a: np.ndarray) -> np.ndarray:
    r = a[:, :8] + a[:, 8:]
    return ((r[:, 0] + r[:, 1]) + (r[:, 2] + r[:, 3])) + ((r[:, 4] + r[:, 5]) + (r[:, 6] + r[:, 7]))


def gradient(luma: np.ndarray) -> np.ndarray:
    """Per-block mean gradient magnitude (float32)."""
    h, w = luma.shape
    dx = np.zeros_like(luma)
    dy = np.zeros_like(luma)
    dx[:, :-1] = luma[:, 1:] - luma[:, :-1]
    dy[:-1, :] = luma[1:, :] - luma[:-1, :]
    mag = np.hypot(dx, dy)
    return _pw16(to_blocks(mag)) / _F(16)


def block_stats(luma: np.ndarray, sigma_min: float = 0.25):
    blk = to_blocks(luma).astype(np.float64)
    mean = _pw16(blk) / 16.0
    dev = blk - mean[:, None]
    sd = np.sqrt(_pw16(dev * dev) / 16.0)
    norm = (blk - mean[:, None]) / np.maximum(sd, sigma_min)[:, None]
    return mean, sd, norm


def vq_nearest(norm32: np.ndarray, centroids: np.ndarray, chunk: int = 1 << 15) -> np.ndarray:
    norm32 = np.asarray(norm32, _F)
    cents = np.asarray(centroids, _F)
    out = np.empty(len(norm32), np.int64)
    with np.errstate(all="ignore"):
        for lo in range(0, len(norm32), chunk):
            b = norm32[lo:lo + chunk]
            best = np.full(len(b), _F(3.402823e38))
            idx = np.zeros(len(b), np.int64)
            for j, c in enumerate(cents):
                d = b - c
                dist = _pw16(d * d)
                better = dist < best
                best = np.where(better, dist, best)
                idx = np.where(better, j, idx)
            out[lo:lo + chunk] = idx
    return out


def kmeans(points: np.ndarray, size: int, seed: int, max_iter: int = 20,
           trace: list | None = None) -> np.ndarray:
    """k-means++ seeding then Lloyd iterations; returns (size, 16) float32."""
    pts = np.asarray(points, np.float64)
    n = len(pts)
    if n == 0:
        raise ValueError("no blocks to cluster")
    if size > n:
        raise ValueError(f"codebook size {size} exceeds {n} training blocks")
    rng = np.random.default_rng(seed)
    cent = np.empty((size, pts.shape[1]))
    cent[0] = pts[rng.integers(n)]
    closest = ((pts - cent[0]) ** 2).sum(axis=1)
    for j in range(1, size):
        total = closest.sum()
        pick = int(rng.integers(n)) if total <= 0.0 else int(rng.choice(n, p=closest / total))
        cent[j] = pts[pick]
        closest = np.minimum(closest, ((pts - cent[j]) ** 2).sum(axis=1))

    def assign_of(c):
        d = (pts ** 2).sum(axis=1)[:, None] + (c ** 2).sum(axis=1)[None, :] - 2.0 * pts @ c.T
        return np.argmin(d, axis=1)

    assign = assign_of(cent)
    for _ in range(max_iter):
        for j in range(size):
            members = pts[assign == j]
            if len(members):
                cent[j] = members.mean(axis=0)
            else:
                far = int(np.argmax(((pts - cent[assign]) ** 2).sum(axis=1)))
                cent[j] = pts[far]
                assign[far] = j
        fresh = assign_of(cent)
        if trace is not None:
            trace.append(float(((pts - cent[fresh]) ** 2).sum()))
        if np.array_equal(fresh, assign):
            break
        assign = fresh
    return cent.astype(np.float32)


def train_codebook(luma: np.ndarray, codebook_size: int, seed: int, sigma_min: float = 0.25,
                   grad_min: float = 1.0) -> np.ndarray:
    """imgc.py:384-393: training set = normalised blocks whose gradient clears grad_min."""
    _, _, norm = block_stats(luma, sigma_min)
    train = norm[gradient(luma) >= grad_min]
    if len(train) == 0:
        train = norm
    return kmeans(train, min(codebook_size, len(train)), seed)


def encode(image: np.ndarray, codebook: np.ndarray | None = None, codebook_size: int = 256,
           seed: int = 0, sigma_min: float = 0.25, grad_min: float = 1.0) -> dict:
    """imgc.py:343-403 as a dict of container fields (codebook trained if not given)."""
    image = np.asarray(image)
    if image.ndim != 3 or image.shape[2] != 3 or image.dtype != np.uint8:
        raise ValueError("expected an (h, w, 3) uint8 image")
    h, w = image.shape[:2]
    if h % 4 or w % 4:
        raise ValueError(f"dimensions must be multiples of 4, got {w}x{h}")
    y, cb, cr = ycbcr(image)
    if codebook is None:
        codebook = train_codebook(y, codebook_size, seed, sigma_min, grad_min)
    mean, sd, norm = block_stats(y, sigma_min)
    idx = vq_nearest(norm.astype(_F), codebook)
    return dict(width=w, height=h, sigma_step=SIGMA_STEP, codebook=np.asarray(codebook, _F),
                means=np.clip(np.rint(mean), 0, 255).astype(np.uint8),
                sigma_idx=np.clip(np.rint(sd / SIGMA_STEP), 0, 255).astype(np.uint8),
                indices=idx.astype(np.uint8), cb=boxdown(cb), cr=boxdown(cr))


def compress(image, codebook_size: int = 256, seed: int = 0, **kw) -> bytes:
    return to_bytes(encode(image, None, codebook_size, seed, **kw))


def to_bytes(ci: dict) -> bytes:
    rec = np.stack([ci["means"], ci["sigma_idx"], ci["indices"]], axis=1).astype(np.uint8)
    return (_HEADER.pack(MAGIC, ci["width"], ci["height"], len(ci["codebook"]), ci["sigma_step"])
            + np.asarray(ci["codebook"], "<f4").tobytes() + rec.tobytes()
            + ci["cb"].tobytes() + ci["cr"].tobytes())


def from_bytes(blob: bytes) -> dict:
    magic, w, h, ncb, step = _HEADER.unpack_from(blob)
    if magic != MAGIC:
        raise ValueError(f"bad container magic {magic!r}")
    off = _HEADER.size
    cents = np.frombuffer(blob, "<f4", ncb * 16, off).reshape(ncb, 16).astype(_F)
    off += ncb * 64
    nb = (w // 4) * (h // 4)
    rec = np.frombuffer(blob, np.uint8, nb * 3, off).reshape(nb, 3)
    off += nb * 3
    cb = np.frombuffer(blob, np.uint8, nb, off).reshape(h // 4, w // 4)
    cr = np.frombuffer(blob, np.uint8, nb, off + nb).reshape(h // 4, w // 4)
    return dict(width=w, height=h, sigma_step=step, codebook=cents, means=rec[:, 0].copy(),
                sigma_idx=rec[:, 1].copy(), indices=rec[:, 2].copy(), cb=cb.copy(), cr=cr.copy())


def decode(ci: dict) -> np.ndarray:
    h, w = ci["height"], ci["width"]
    sig = ci["sigma_idx"].astype(np.float64) * ci["sigma_step"]
    cents = ci["codebook"].astype(np.float64)[ci["indices"]]
    luma = from_blocks(ci["means"].astype(np.float64)[:, None] + sig[:, None] * cents, h, w)
    up = lambda p: np.repeat(np.repeat(p.astype(np.float64), 4, 0), 4, 1) - 128.0  # noqa: E731
    cb, cr = up(ci["cb"]), up(ci["cr"])
    rgb = np.stack([luma + 1.402 * cr, luma - 0.344136 * cb - 0.714136 * cr, luma + 1.772 * cb], -1)
    return np.clip(np.rint(rgb), 0, 255).astype(np.uint8)


def synthetic_image(width: int = 512, height: int = 512, seed: int = 7) -> np.ndarray:
    """The reference's procedural fixture (imgc.py:92-105)."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:height, 0:width].astype(np.float64)
    rad = np.hypot(xx - width / 2, yy - height / 2) / max(width, height)
    r = 110 + 70 * np.sin(2 * np.pi * xx / 97) * np.cos(2 * np.pi * yy / 181) + 60 * (xx / width)
    g = 100 + 90 * np.exp(-4.0 * rad ** 2) + 50 * (yy / height)
    b = 120 + 80 * np.cos(2 * np.pi * (xx + yy) / 253) - 40 * rad
    img = np.stack([r, g, b], axis=-1)
    img += rng.normal(0.0, 2.0, img.shape)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def psnr(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    mse = np.mean((a - b) ** 2)
    return float("inf") if mse == 0.0 else float(10.0 * np.log10(255.0 ** 2 / mse))
