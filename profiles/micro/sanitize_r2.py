"""compute-sanitizer driver for the kernels added in round 2 (small sizes):
the transposed-output column ring (two-pass 2^24), the k-means trainer with
the tensor-core Lloyd assignment, the encoder's vector mode through it, the
device container write/read and a captured-graph replay."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1203_4938_b200 import ops  # noqa: E402
from paper_1203_4938_b200 import kmeans as km  # noqa: E402
from paper_1203_4938_b200.apps import fft as afft  # noqa: E402
from paper_1203_4938_b200.apps import imgc  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("xp", "all"):
    x = torch.randn((1, 1 << 24), dtype=torch.complex64, device="cuda")
    ops.fft_forward(x, 1 << 24)
    torch.cuda.synchronize()
    print("xp ok", flush=True)
if what in ("km", "all"):
    pts = torch.randn((5000, 16), dtype=torch.float64, device="cuda")
    km.kmeans_device(pts, 64, 3)
    km.kmeans_sharded(pts, 32, seed=1)
    torch.cuda.synchronize()
    print("kmeans ok", flush=True)
if what in ("codec", "all"):
    img = imgc.synthetic_image(96, 64, seed=4)
    blob = imgc.compress_to_bytes(img, 16, 0)
    imgc.decompress_bytes(blob)
    torch.cuda.synchronize()
    print("codec ok", flush=True)
if what in ("replay", "all"):
    v = (np.random.default_rng(0).standard_normal(1024) + 1j).astype(np.complex64)
    for _ in range(3):
        afft.fft(v)
    print("replay ok", flush=True)
