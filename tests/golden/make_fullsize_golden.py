"""Full-size golden data for the C4 and C5 parity tests, made by the REFERENCE itself.

Run inside the build container (the reference is importable there, not on the
GPU box); it takes ~15-25 min of CPU and ~21 GB of RAM for C4:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_fullsize_golden.py [c4] [c5]

The outputs are small (codebooks and SHA-256 digests), so the GPU tests can
rebuild the full-size inputs from the seeded recipes of SURVEY §8(d) and check
the device output byte for byte without shipping 21 MB bitstreams:

  c4_golden.npz  C4: g = synthetic_image(8192, 8192, seed=7)[..., 1], image =
                 R=G=B=g; reference compress(image, 256, 0) (imgc.py:343-403):
                 its trained codebook, the SHA-256 and length of its bitstream,
                 SHA-256 of the record / Cb / Cr sections, the binary64
                 rounding-tie counts of its mean and sigma quantisers, and the
                 reference's wall time.
  c5_golden.npz  C5 images i = 0 and 63: g_i = synthetic_image(4096, 4096,
                 seed=1000+i)[..., 1] -> reference fft() over every row then
                 every column (fft.py:150-174) -> the spectrum_u8 adapter node
                 on the reference engine -> reference compress(spec, 256, 0):
                 SHA-256 of the adapter output, the codebook, the bitstream
                 SHA-256, and the wall time of each stage.
"""

from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]


def sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def ties(values: np.ndarray) -> int:
    """binary64 values whose fractional part is within 1e-9 of one half."""
    frac = values - np.floor(values)
    return int((np.abs(frac - 0.5) < 1e-9).sum())


def c4() -> None:
    from dpp.apps import imgc as rimgc
    g = rimgc.synthetic_image(8192, 8192, seed=7)[..., 1]
    img = np.repeat(g[..., None], 3, 2)
    t0 = time.perf_counter()
    ci = rimgc.compress(img, 256, 0)
    secs = time.perf_counter() - t0
    blob = ci.to_bytes()
    rec = np.stack([ci.means, ci.sigma_idx, ci.indices], axis=1).astype(np.uint8)
    # tie counts from the reference's own binary64 statistics (imgc.py:384-386, 398-401)
    luma = (np.float32(0.299) * g.astype(np.float32) + np.float32(0.587) * g.astype(np.float32)) \
        + np.float32(0.114) * g.astype(np.float32)
    blocks = luma.reshape(2048, 4, 2048, 4).swapaxes(1, 2).reshape(-1, 16).astype(np.float64)
    means, sigmas = blocks.mean(axis=1), blocks.std(axis=1)
    np.savez_compressed(
        HERE / "c4_golden.npz", codebook=np.asarray(ci.codebook.centroids, np.float32), blob_sha=sha(blob),
        blob_len=len(blob), records_sha=sha(rec.tobytes()), cb_sha=sha(ci.cb.tobytes()),
        cr_sha=sha(ci.cr.tobytes()), mean_ties=ties(means), sigma_ties=ties(sigmas / 0.25),
        seconds=secs)
    print(f"c4: {len(blob)} B in {secs:.1f} s, sha {sha(blob)[:16]}, ties {ties(means)}/{ties(sigmas / 0.25)}",
          flush=True)


def c5() -> None:
    from dpp import LocalBackend, StreamFile, run
    from dpp.apps import fft as rfft
    from dpp.apps import imgc as rimgc
    from dpp.model import Instance, Node, Program
    from dpp.types import DataType, Direction, IOPoint
    sys.path.insert(0, str(ROOT))
    from paper_1203_4938_b200.apps.chain import ALPHA, spectrum_u8_kernel
    ours = spectrum_u8_kernel(ALPHA)
    node = Node(ours.name, ours.body, tuple(IOPoint(p.name, DataType(p.data.base, p.data.width),
                                                    Direction(p.direction.value)) for p in ours.io))
    prog = Program({node.name: node}, (Instance(0, node.name),), ())
    out = {}
    plan = rfft.FftPlan(4096, 3)
    for i in (0, 63):
        g = rimgc.synthetic_image(4096, 4096, seed=1000 + i)[..., 1]
        t0 = time.perf_counter()
        z = np.stack([rfft.fft(row.astype(np.complex64), plan) for row in g.astype(np.float32)])
        z = np.stack([rfft.fft(np.ascontiguousarray(col), plan) for col in z.T]).T
        t1 = time.perf_counter()
        res = run(LocalBackend(), prog, {"0.x": StreamFile(DataType("float", 2),
                                                           np.ascontiguousarray(z).view(np.float32).ravel())})
        spec = res["0.y"].values.reshape(4096, 4096).astype(np.uint8)
        t2 = time.perf_counter()
        ci = rimgc.compress(np.repeat(spec[..., None], 3, 2), 256, 0)
        t3 = time.perf_counter()
        out[f"spec_sha_{i}"] = sha(spec.tobytes())
        out[f"codebook_{i}"] = np.asarray(ci.codebook.centroids, np.float32)
        out[f"blob_sha_{i}"] = sha(ci.to_bytes())
        out[f"seconds_{i}"] = np.array([t1 - t0, t2 - t1, t3 - t2])
        print(f"c5 image {i}: fft {t1 - t0:.1f} s, adapter {t2 - t1:.1f} s, compress {t3 - t2:.1f} s", flush=True)
    np.savez_compressed(HERE / "c5_golden.npz", **out)


if __name__ == "__main__":
    parts = sys.argv[1:] or ["c4", "c5"]
    if "c4" in parts:
        c4()
    if "c5" in parts:
        c5()
