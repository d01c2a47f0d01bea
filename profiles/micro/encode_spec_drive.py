"""Drive the TC encoder on C5 spectrum images (mode=spec) or noise images (mode=noise) for ncu."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    import torch
    from paper_1203_4938_b200 import ops
    from paper_1203_4938_b200.apps import chain
    mode = sys.argv[1]
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    b, side = 16, 4096
    imgs = torch.randint(0, 256, (b, side, side), dtype=torch.uint8, device=dev, generator=g)
    if mode == "spec":
        spec = torch.empty_like(imgs)
        ops.fft2d_u8_spectrum(imgs.reshape(-1), side, side, chain.ALPHA, spec.reshape(-1))
        imgs = spec
    cb = torch.randn((b, 256, 16), device=dev, generator=g)
    cb = (cb - cb.mean(-1, keepdim=True)) / cb.std(-1, unbiased=False, keepdim=True)
    nb = (side // 4) ** 2
    rec = torch.empty(b * nb * 3, dtype=torch.uint8, device=dev)
    cbp = torch.empty(b * nb, dtype=torch.uint8, device=dev)
    crp = torch.empty(b * nb, dtype=torch.uint8, device=dev)
    for _ in range(2):
        ops.encode(imgs, 1, side, side, cb, rec, cbp, crp, batch=b, shared_codebook=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.encode(imgs, 1, side, side, cb, rec, cbp, crp, batch=b, shared_codebook=False)
    e1.record()
    torch.cuda.synchronize()
    print(mode, e0.elapsed_time(e1), "ms")


if __name__ == "__main__":
    main()
