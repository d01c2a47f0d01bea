"""compress(image, 256, 0) end to end with the GPU k-means trainer, per stage.

Images: the C4 frame (synthetic_image(8192, 8192, seed=7) green channel as
gray) and its 4096^2 crop-free sibling synthetic_image(4096, 4096, seed=7).
SSE of the trained codebook over the training blocks against the
reference codebook (tests/golden/c4_golden.npz) for the C4 frame."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def sse(train, cents):
    import torch
    c = cents.to(torch.float64)
    cn = (c * c).sum(1)
    tot = 0.0
    for lo in range(0, train.shape[0], 1 << 18):
        p = train[lo:lo + (1 << 18)]
        d = (p * p).sum(1)[:, None] + cn[None, :] - 2.0 * p @ c.T
        tot += float(d.min(1).values.clamp(min=0).sum())
    return tot


def main():
    import numpy as np
    import torch
    from paper_1203_4938_b200.apps import imgc
    from paper_1203_4938_b200 import kmeans as km
    dev = torch.device("cuda:0")
    for side in (4096, 8192):
        g = imgc.synthetic_image(side, side, seed=7)[..., 1]
        img = np.ascontiguousarray(np.repeat(g[..., None], 3, 2))
        imgc.compress(img[:256, :256], 256, 0)  # warm-up: library, plans
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ci = imgc.compress(img, 256, 0)
        t1 = time.perf_counter()
        # stages
        px = torch.from_numpy(img).to(dev)
        torch.cuda.synchronize()
        s0 = time.perf_counter()
        norm64, grad = km.block_stats_device(px, 3, side, side)
        keep = torch.nonzero(grad >= 1.0).squeeze(1)
        train = norm64.index_select(0, keep) if keep.numel() else norm64
        torch.cuda.synchronize()
        s1 = time.perf_counter()
        tr = []
        cents = km.kmeans_device(train, 256, 0, trace=tr)
        torch.cuda.synchronize()
        s2 = time.perf_counter()
        line = (f"{side}^2: compress {t1 - t0:.3f} s ({len(ci.to_bytes())} B); stats+filter {s1 - s0:.4f} s, "
                f"kmeans {s2 - s1:.3f} s ({len(tr)} Lloyd iterations, n={train.shape[0]})")
        if side == 8192:
            ref = torch.from_numpy(np.load(ROOT / "tests/golden/c4_golden.npz")["codebook"]).to(dev)
            a, b = sse(train, cents), sse(train, ref)
            line += f"; SSE gpu {a:.6e} reference {b:.6e} ratio {a / b:.4f}"
        print(line, flush=True)


if __name__ == "__main__":
    main()
