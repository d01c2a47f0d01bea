"""Block-VQ image codec on the B200 nodes (mirror of dpp.apps.imgc).

Same names, container format and argument meaning as
/root/reference/pkg/src/dpp/apps/imgc.py: PPM IO (:53-89), ``synthetic_image``
(:92-105), ``psnr`` (:108-117), program builders ``ycbcr_program`` /
``chroma_down_program`` / ``gradient_program`` / ``vq_program`` (:128-185),
``Codebook`` (:207-218), ``CompressedImage`` (:279-337), ``compress``
(:343-403), ``decompress`` (:426-439), ``kmeans`` (:221-273).

``compress`` runs the forward block transform, quantisation and ordering as
ONE fused sm_100a kernel (``dpp_imgc_encode``) whose output bytes are
identical to the reference's for the same codebook.  The codebook is an
input of that node: pass ``codebook=`` to encode against a given codebook
(bit-exact parity runs use the oracle's), otherwise it is trained on the
GPU by ``kmeans`` (``codebook_gpu``), which follows the reference algorithm
but is only tolerance-equal to it.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from ..client import CudaBackend
from ..model import Instance, Node, Program
from ..types import DataType, Direction, IOPoint

__all__ = ["read_ppm", "write_ppm", "synthetic_image", "Codebook", "kmeans", "psnr", "compress_to_bytes",
           "decompress_bytes",
           "CompressedImage", "compress", "compress_batch", "decompress", "ycbcr_program",
           "chroma_down_program", "gradient_program", "vq_program", "encode_kernel",
           "encode_program", "SIGMA_STEP", "MAGIC", "NATIVE_TAG"]

MAGIC = b"DPVQ"
SIGMA_STEP = 64.0 / 256.0
NATIVE_TAG = "// dpp-b200 native:"
_HEADER = struct.Struct("<4sIIHf")


# ---------------------------------------------------------------------------
# PPM IO and fixtures (host-side file helpers)

def read_ppm(source: bytes | str | Path) -> np.ndarray:
    """Binary P6 (maxval 255) -> (h, w, 3) uint8 (imgc.py:53-80)."""
    data = source if isinstance(source, bytes) else Path(source).read_bytes()
    if not data.startswith(b"P6"):
        raise ValueError("not a binary PPM (P6) file")
    vals: list[int] = []
    pos = 2
    while len(vals) < 3:
        while pos < len(data) and data[pos:pos + 1].isspace():
            pos += 1
        if data[pos:pos + 1] == b"#":
            pos = data.index(b"\n", pos) + 1
            continue
        end = pos
        while end < len(data) and not data[end:end + 1].isspace():
            end += 1
        if end == pos:
            raise ValueError("truncated PPM header")
        vals.append(int(data[pos:end]))
        pos = end
    pos += 1
    w, h, maxval = vals
    if maxval != 255:
        raise ValueError(f"only maxval 255 supported, got {maxval}")
    need = w * h * 3
    body = data[pos:pos + need]
    if len(body) != need:
        raise ValueError(f"PPM body has {len(body)} bytes, expected {need}")
    return np.frombuffer(body, np.uint8).reshape(h, w, 3).copy()


def write_ppm(image: np.ndarray, path: str | Path | None = None) -> bytes:
    image = np.asarray(image, np.uint8)
    h, w, _ = image.shape
    blob = b"P6\n%d %d\n255\n" % (w, h) + image.tobytes()
    if path is not None:
        Path(path).write_bytes(blob)
    return blob


def synthetic_image(width: int = 512, height: int = 512, seed: int = 7) -> np.ndarray:
    """The reference's procedural fixture (imgc.py:92-105), same RNG stream."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:height, 0:width].astype(np.float64)
    rad = np.hypot(xx - width / 2, yy - height / 2) / max(width, height)
    r = 110 + 70 * np.sin(2 * np.pi * xx / 97) * np.cos(2 * np.pi * yy / 181) + 60 * (xx / width)
    g = 100 + 90 * np.exp(-4.0 * rad ** 2) + 50 * (yy / height)
    b = 120 + 80 * np.cos(2 * np.pi * (xx + yy) / 253) - 40 * rad
    img = np.stack([r, g, b], axis=-1)
    img += rng.normal(0.0, 2.0, img.shape)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    mse = np.mean((a - b) ** 2)
    return float("inf") if mse == 0.0 else float(10.0 * np.log10(255.0 ** 2 / mse))


# ---------------------------------------------------------------------------
# node bodies: the reference's four programs (bit-identical text) + the fused node

def _one_node(name: str, body: str, io) -> Program:
    node = Node(name, body, tuple(io))
    return Program({name: node}, (Instance(0, name),), ())


def ycbcr_program() -> Program:
    body = ("int i = get_global_id(0);\n"
            "uchar4 p = rgb[i];\n"
            "yl[i] = 0.299f*p.x + 0.587f*p.y + 0.114f*p.z;\n"
            "cb[i] = 128.0f - 0.168736f*p.x - 0.331264f*p.y + 0.5f*p.z;\n"
            "cr[i] = 128.0f + 0.5f*p.x - 0.418688f*p.y - 0.081312f*p.z;\n")
    f = DataType("float")
    return _one_node("ycbcr", body, [IOPoint("rgb", DataType("uchar", 4), Direction.INPUT),
                                     IOPoint("yl", f, Direction.OUTPUT),
                                     IOPoint("cb", f, Direction.OUTPUT),
                                     IOPoint("cr", f, Direction.OUTPUT)])


def chroma_down_program() -> Program:
    total = " + ".join("b.s%x" % j for j in range(16))
    body = ("int i = get_global_id(0);\n"
            "float16 b = blk[i];\n"
            f"avg[i] = ({total}) * 0.0625f;\n")
    return _one_node("boxdown", body, [IOPoint("blk", DataType("float", 16), Direction.INPUT),
                                       IOPoint("avg", DataType("float"), Direction.OUTPUT)])


def gradient_program(width: int, height: int) -> Program:
    body = ("int i = get_global_id(0);\n"
            f"int x = i % {width};\n"
            f"int y = i / {width};\n"
            f"dx[i] = (x < {width - 1}) ? lum[i+1] - lum[i] : 0.0f;\n"
            f"dy[i] = (y < {height - 1}) ? lum[i+{width}] - lum[i] : 0.0f;\n")
    f = DataType("float")
    return _one_node("gradient", body, [IOPoint("lum", f, Direction.INPUT),
                                        IOPoint("dx", f, Direction.OUTPUT),
                                        IOPoint("dy", f, Direction.OUTPUT)])


def vq_program(codebook_size: int) -> Program:
    body = ("int i = get_global_id(0);\n"
            "float16 b = blk[i];\n"
            "float best = 3.402823e38f;\n"
            "int bestj = 0;\n"
            f"for (int j = 0; j < {codebook_size}; j = j + 1) {{\n"
            "    float16 d = b - cbk[j];\n"
            "    float dist = dot(d, d);\n"
            "    if (dist < best) { best = dist; bestj = j; }\n"
            "}\n"
            "idx[i] = bestj;\n")
    f16 = DataType("float", 16)
    return _one_node("vqnearest", body, [IOPoint("blk", f16, Direction.INPUT),
                                         IOPoint("cbk", f16, Direction.INPUT),
                                         IOPoint("idx", DataType("int"), Direction.OUTPUT)])


def encode_kernel(width: int, height: int, codebook_size: int) -> Node:
    """Fused node ``imgc_encode``: gray frames in, (mu, sig, idx, cb, cr) per block out.

    px: uchar16 — 16 consecutive raster pixels per work-item, i.e. one
    work-item per 4x4 block; cbk: float16 broadcast side input (the codebook,
    NOT chunked — an executor extension the reference plan rules lack,
    SURVEY §8(b)).  The body is valid kernel language but deliberately
    faults on the reference interpreter: the fused node needs binary64
    block statistics the kernel language cannot express, so it only runs
    natively."""
    if width % 4 or height % 4:
        raise ValueError(f"dimensions must be multiples of 4, got {width}x{height}")
    if not 1 <= codebook_size <= 256:
        raise ValueError("codebook size must be in 1..256")
    body = (f"{NATIVE_TAG} imgc_encode width={width} height={height} ncb={codebook_size}\n"
            "// native-only: needs binary64 statistics; faults on the interpreter\n"
            "int i = get_global_id(0);\n"
            "uchar16 p = px[i - get_global_size(0)];\n"
            "float16 c = cbk[0];\n"
            "mu[i] = p.s0;\nsig[i] = p.s1;\nidx[i] = p.s2;\ncb[i] = p.s3;\ncr[i] = p.s4;\n")
    u = DataType("uchar")
    return Node("imgc_encode", body,
                (IOPoint("px", DataType("uchar", 16), Direction.INPUT),
                 IOPoint("cbk", DataType("float", 16), Direction.INPUT),
                 *(IOPoint(n, u, Direction.OUTPUT) for n in ("mu", "sig", "idx", "cb", "cr"))))


def encode_program(width: int, height: int, codebook_size: int) -> Program:
    node = encode_kernel(width, height, codebook_size)
    return Program({node.name: node}, (Instance(0, node.name),), ())


# ---------------------------------------------------------------------------
# codebook and container

@dataclass(frozen=True)
class Codebook:
    """Normalised 4x4 blocks as row-major 16-vectors (imgc.py:207-218)."""

    centroids: np.ndarray  # (size, 16) float32

    @property
    def size(self) -> int:
        return len(self.centroids)

    def to_bytes(self) -> bytes:
        return np.asarray(self.centroids, "<f4").tobytes()


@dataclass(frozen=True)
class CompressedImage:
    """The DPVQ container (imgc.py:279-337), byte-compatible."""

    width: int
    height: int
    sigma_step: float
    codebook: Codebook
    means: np.ndarray
    sigma_idx: np.ndarray
    indices: np.ndarray
    cb: np.ndarray
    cr: np.ndarray

    @property
    def block_count(self) -> int:
        return (self.width // 4) * (self.height // 4)

    def to_bytes(self) -> bytes:
        rec = np.stack([self.means, self.sigma_idx, self.indices], axis=1).astype(np.uint8)
        head = _HEADER.pack(MAGIC, self.width, self.height, self.codebook.size, self.sigma_step)
        return head + self.codebook.to_bytes() + rec.tobytes() + self.cb.tobytes() + self.cr.tobytes()

    @classmethod
    def from_bytes(cls, blob: bytes) -> "CompressedImage":
        magic, w, h, ncb, step = _HEADER.unpack_from(blob)
        if magic != MAGIC:
            raise ValueError(f"bad container magic {magic!r}")
        off = _HEADER.size
        cents = np.frombuffer(blob, "<f4", ncb * 16, off).reshape(ncb, 16).astype(np.float32)
        off += ncb * 64
        nb = (w // 4) * (h // 4)
        rec = np.frombuffer(blob, np.uint8, nb * 3, off).reshape(nb, 3)
        off += nb * 3
        qh, qw = h // 4, w // 4
        cb = np.frombuffer(blob, np.uint8, qh * qw, off).reshape(qh, qw)
        cr = np.frombuffer(blob, np.uint8, qh * qw, off + qh * qw).reshape(qh, qw)
        return cls(w, h, step, Codebook(cents), rec[:, 0].copy(), rec[:, 1].copy(), rec[:, 2].copy(),
                   cb.copy(), cr.copy())

    @classmethod
    def from_records(cls, width, height, codebook, records, cb, cr) -> "CompressedImage":
        rec = np.asarray(records, np.uint8).reshape(-1, 3)
        return cls(width, height, SIGMA_STEP, Codebook(np.asarray(codebook, np.float32)),
                   rec[:, 0].copy(), rec[:, 1].copy(), rec[:, 2].copy(),
                   np.asarray(cb, np.uint8).reshape(height // 4, width // 4),
                   np.asarray(cr, np.uint8).reshape(height // 4, width // 4))

    def save(self, path: str | Path) -> None:
        Path(path).write_bytes(self.to_bytes())

    @classmethod
    def load(cls, path: str | Path) -> "CompressedImage":
        return cls.from_bytes(Path(path).read_bytes())


# ---------------------------------------------------------------------------
# compress / decompress

def _validate_image(image) -> tuple[int, int, int]:
    shape = tuple(image.shape)
    if len(shape) == 3 and shape[2] in (3, 4):
        ch = shape[2]
    elif len(shape) == 2:
        ch = 1
    else:
        raise ValueError("expected an (h, w, 3) uint8 image")
    h, w = shape[:2]
    if h % 4 or w % 4:
        raise ValueError(f"dimensions must be multiples of 4, got {w}x{h}")
    return h, w, ch


def compress(image, codebook_size: int = 256, seed: int = 0, *, backend: CudaBackend | None = None,
             sigma_min: float = 0.25, grad_min: float = 1.0, codebook=None) -> CompressedImage:
    """Compress an (h, w, 3) uint8 image (imgc.py:343-403); (h, w) = gray, R=G=B.

    The image may be a numpy array or a CUDA uint8 tensor.  With ``codebook``
    given (a ``Codebook`` or (n, 16) float32 array) the result is the
    reference bitstream for that codebook, bit for bit."""
    import torch

    from .. import ops
    from .._torch import require_cuda, to_device
    is_tensor = isinstance(image, torch.Tensor)
    if not is_tensor:
        image = np.asarray(image)
        if image.dtype != np.uint8:
            raise ValueError("expected an (h, w, 3) uint8 image")
    elif image.dtype != torch.uint8:
        raise ValueError("expected an (h, w, 3) uint8 image")
    h, w, ch = _validate_image(image)
    if not 1 <= codebook_size <= 256:
        raise ValueError("codebook size must be in 1..256")
    backend = backend or CudaBackend()
    dev = require_cuda(backend.device)
    px = image.contiguous().to(dev) if is_tensor else to_device(np.ascontiguousarray(image), dev)
    nb = (h // 4) * (w // 4)
    if codebook is None:
        cents = kmeans_codebook(px, ch, h, w, codebook_size, seed, sigma_min, grad_min)
    else:
        arr = codebook.centroids if isinstance(codebook, Codebook) else codebook
        cents = torch.as_tensor(np.ascontiguousarray(arr, np.float32)).to(dev) \
            if not isinstance(arr, torch.Tensor) else arr.to(dev, torch.float32).contiguous()
    rec = torch.empty(nb * 3, dtype=torch.uint8, device=dev)
    cbp = torch.empty(nb, dtype=torch.uint8, device=dev)
    crp = torch.empty(nb, dtype=torch.uint8, device=dev)
    ops.encode(px, ch, h, w, cents, rec, cbp, crp, sigma_min=sigma_min)
    host = torch.cat([rec, cbp, crp]).cpu().numpy()
    return CompressedImage.from_records(w, h, cents.cpu().numpy(), host[:3 * nb], host[3 * nb:4 * nb],
                                        host[4 * nb:])


def compress_batch(images, codebooks, *, backend: CudaBackend | None = None, sigma_min: float = 0.25,
                   out=None):
    """Device-level batch encode: (B, h, w) gray uint8 CUDA tensor + (B, n, 16) codebooks.

    Returns (records (B, blocks, 3), cb (B, blocks), cr (B, blocks)) CUDA
    tensors; nothing leaves the GPU."""
    import torch

    from .. import ops
    b, h, w = images.shape[:3]
    ch = 1 if images.dim() == 3 else images.shape[3]
    nb = (h // 4) * (w // 4)
    dev = images.device
    rec, cbp, crp = out if out is not None else (
        torch.empty((b, nb, 3), dtype=torch.uint8, device=dev),
        torch.empty((b, nb), dtype=torch.uint8, device=dev),
        torch.empty((b, nb), dtype=torch.uint8, device=dev))
    shared = codebooks.dim() == 2
    ops.encode(images, ch, h, w, codebooks.contiguous(), rec, cbp, crp, batch=b,
               shared_codebook=shared, sigma_min=sigma_min)
    return rec, cbp, crp


def compress_to_bytes(image, codebook_size: int = 256, seed: int = 0, *, backend: CudaBackend | None = None,
                      sigma_min: float = 0.25, grad_min: float = 1.0, codebook=None) -> bytes:
    """``compress(...).to_bytes()`` with the container assembled on the device
    (SURVEY §8(f) row 4): the encoder writes the record run and both chroma
    planes at their container offsets in one device buffer, and one D2H
    brings back the payload — no host-side stacking or re-packing of records.
    Byte-identical to ``compress(...).to_bytes()``."""
    import torch

    from .. import ops
    from .._torch import require_cuda, to_device
    is_tensor = isinstance(image, torch.Tensor)
    if not is_tensor:
        image = np.asarray(image)
        if image.dtype != np.uint8:
            raise ValueError("expected an (h, w, 3) uint8 image")
    elif image.dtype != torch.uint8:
        raise ValueError("expected an (h, w, 3) uint8 image")
    h, w, ch = _validate_image(image)
    if not 1 <= codebook_size <= 256:
        raise ValueError("codebook size must be in 1..256")
    dev = require_cuda((backend or CudaBackend()).device)
    px = image.contiguous().to(dev) if is_tensor else to_device(np.ascontiguousarray(image), dev)
    if codebook is None:
        cents = kmeans_codebook(px, ch, h, w, codebook_size, seed, sigma_min, grad_min)
    else:
        arr = codebook.centroids if isinstance(codebook, Codebook) else codebook
        cents = torch.as_tensor(np.ascontiguousarray(arr, np.float32)).to(dev) \
            if not isinstance(arr, torch.Tensor) else arr.to(dev, torch.float32).contiguous()
    nb = (h // 4) * (w // 4)
    payload = torch.empty(5 * nb, dtype=torch.uint8, device=dev)  # records | Cb | Cr, container order
    ops.encode(px, ch, h, w, cents, payload[:3 * nb], payload[3 * nb:4 * nb], payload[4 * nb:],
               sigma_min=sigma_min)
    host = torch.empty(5 * nb, dtype=torch.uint8, pin_memory=True)
    host.copy_(payload)
    head = _HEADER.pack(MAGIC, w, h, cents.shape[0], SIGMA_STEP)
    return head + Codebook(cents.cpu().numpy()).to_bytes() + host.numpy().tobytes()


def decompress_bytes(blob, *, backend: CudaBackend | None = None) -> np.ndarray:
    """``decompress(CompressedImage.from_bytes(blob))`` with the container read
    on the device: the header is checked on the host, the
    whole blob goes H2D once and the decoder reads the codebook, records and
    chroma planes at their container offsets.  Bit-exact with ``decompress``."""
    import torch

    from .. import ops
    from .._torch import require_cuda
    blob = bytes(blob)
    if len(blob) < _HEADER.size:
        raise ValueError("truncated container")
    magic, w, h, ncb, _ = _HEADER.unpack_from(blob)
    if magic != MAGIC:
        raise ValueError(f"bad container magic {magic!r}")
    nb = (w // 4) * (h // 4)
    off = _HEADER.size
    need = off + ncb * 64 + 5 * nb
    if len(blob) < need:
        raise ValueError(f"truncated container: {len(blob)} bytes, need {need}")
    dev = require_cuda((backend or CudaBackend()).device)
    # the codebook floats sit at byte 18: shift the image by 2 bytes so they
    # land 4-byte aligned on the device
    pad = (-off) % 4
    host = torch.empty(need + pad, dtype=torch.uint8, pin_memory=True)
    host.numpy()[pad:] = np.frombuffer(blob, np.uint8, need)
    d = host.to(dev, non_blocking=True)
    cents = d[pad + off:pad + off + ncb * 64].view(torch.float32)
    base = pad + off + ncb * 64
    rgb = torch.empty(h * w * 3, dtype=torch.uint8, device=dev)
    ops.decode(d[base:base + 3 * nb], d[base + 3 * nb:base + 4 * nb], d[base + 4 * nb:base + 5 * nb], cents, h, w,
               rgb)
    return rgb.cpu().numpy().reshape(h, w, 3)


def decompress(ci: CompressedImage, *, backend: CudaBackend | None = None) -> np.ndarray:
    """Reconstruct (h, w, 3) uint8 on the GPU (imgc.py:426-439), bit-exact."""
    import torch

    from .. import ops
    from .._torch import require_cuda
    dev = require_cuda((backend or CudaBackend()).device)
    rec = np.stack([ci.means, ci.sigma_idx, ci.indices], axis=1).astype(np.uint8)
    t = lambda a, dt=torch.uint8: torch.as_tensor(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    rgb = torch.empty(ci.height * ci.width * 3, dtype=torch.uint8, device=dev)
    ops.decode(t(rec), t(ci.cb), t(ci.cr), t(np.asarray(ci.codebook.centroids, np.float32)),
               ci.height, ci.width, rgb)
    return rgb.cpu().numpy().reshape(ci.height, ci.width, 3)


def kmeans(blocks, codebook_size: int, seed: int, max_iter: int = 20, trace: list | None = None,
           *, backend: CudaBackend | None = None) -> Codebook:
    """k-means++ + Lloyd on the GPU (algorithm of imgc.py:221-273)."""
    from ..kmeans import kmeans_device
    cents = kmeans_device(blocks, codebook_size, seed, max_iter, trace, device=(backend or CudaBackend()).device)
    return Codebook(cents.cpu().numpy())


def kmeans_codebook(px, ch, h, w, codebook_size, seed, sigma_min, grad_min):
    """Training set (normalised blocks with gradient >= grad_min) + GPU k-means."""
    from ..kmeans import train_codebook_device
    return train_codebook_device(px, ch, h, w, codebook_size, seed, sigma_min, grad_min)
