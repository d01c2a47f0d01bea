"""Small driver for ncu captures: launches one hot-path kernel a few times.

    ncu ... python profiles/drive.py fft   [--n 65536 --batch 4096 --iters 3]
    ncu ... python profiles/drive.py encode [--size 8192 --iters 3]
    ncu ... python profiles/drive.py fft2d [--rows 16384 --cols 16384 --iters 2]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main() -> None:
    import torch

    from paper_1203_4938_b200 import ops
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["fft", "encode", "fft2d", "chain"])
    ap.add_argument("--images", type=int, default=64)
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--rows", type=int, default=16384)
    ap.add_argument("--cols", type=int, default=16384)
    ap.add_argument("--size", type=int, default=8192)
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    if a.what == "fft":
        x = torch.randn((a.batch, a.n), dtype=torch.complex64, device=dev, generator=g)
        y = torch.empty_like(x)
        for _ in range(a.iters):
            ops.fft_forward(x, a.n, out=y)
    elif a.what == "chain":
        from paper_1203_4938_b200 import CudaBackend
        from paper_1203_4938_b200.apps import chain
        imgs = torch.randint(0, 256, (a.images, 4096, 4096), dtype=torch.uint8, device=dev, generator=g)
        cbs = torch.randn((a.images, 256, 16), dtype=torch.float32, device=dev, generator=g)
        # codebooks as k-means leaves them: centroids of normalised blocks (zero mean, unit deviation)
        cbs = (cbs - cbs.mean(-1, keepdim=True)) / cbs.std(-1, unbiased=False, keepdim=True)
        for _ in range(a.iters):
            chain.run_chain(imgs, cbs, backend=CudaBackend(outputs="device"))
    elif a.what == "fft2d":
        x = torch.randn((a.rows, a.cols), dtype=torch.complex64, device=dev, generator=g)
        for _ in range(a.iters):
            ops.fft2d_forward(x, a.rows, a.cols, out=x)
    else:
        h = w = a.size
        img = torch.randint(0, 256, (h, w), dtype=torch.uint8, device=dev, generator=g)
        cb = torch.randn((256, 16), dtype=torch.float32, device=dev, generator=g)
        nb = (h // 4) * (w // 4)
        rec = torch.empty(nb * 3, dtype=torch.uint8, device=dev)
        cbp = torch.empty(nb, dtype=torch.uint8, device=dev)
        crp = torch.empty(nb, dtype=torch.uint8, device=dev)
        for _ in range(a.iters):
            ops.encode(img, 1, h, w, cb, rec, cbp, crp)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
