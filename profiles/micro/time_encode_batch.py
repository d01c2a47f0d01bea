"""TC encoder throughput: image size, batch, shared vs per-image codebooks."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    import torch
    from paper_1203_4938_b200 import ops
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    for (b, side, shared) in ((1, 8192, True), (4, 4096, True), (64, 4096, True), (64, 4096, False), (16, 8192, True)):
        img = torch.randint(0, 256, (b, side, side), dtype=torch.uint8, device=dev, generator=g)
        cb = torch.randn((1 if shared else b, 256, 16), device=dev, generator=g)
        cb = (cb - cb.mean(-1, keepdim=True)) / cb.std(-1, unbiased=False, keepdim=True)
        nb = (side // 4) ** 2
        rec = torch.empty(b * nb * 3, dtype=torch.uint8, device=dev)
        cbp = torch.empty(b * nb, dtype=torch.uint8, device=dev)
        crp = torch.empty(b * nb, dtype=torch.uint8, device=dev)
        run = lambda: ops.encode(img, 1, side, side, cb, rec, cbp, crp, batch=b, shared_codebook=shared)
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"batch {b} x {side}^2 shared={shared}: {ms:.3f} ms  {b * side * side / ms / 1e6:.1f} Gpx/s")


if __name__ == "__main__":
    main()
