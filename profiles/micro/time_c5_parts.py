"""C5 on real inputs: the fused u8 -> 2-D FFT -> spectrum pass and the encode
of the resulting spectra, each timed alone (CUDA events), 64 x 4096^2."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def timed(fn, iters=5):
    import torch
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main() -> None:
    import torch

    from paper_1203_4938_b200 import CudaBackend, ops
    from paper_1203_4938_b200.apps import chain
    dev = torch.device("cuda:0")
    b, side = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 4096
    g = torch.Generator(device=dev).manual_seed(0)
    imgs = torch.randint(0, 256, (b, side, side), dtype=torch.uint8, device=dev, generator=g)
    cbs = torch.randn((b, 256, 16), dtype=torch.float32, device=dev, generator=g)
    cbs = (cbs - cbs.mean(-1, keepdim=True)) / cbs.std(-1, unbiased=False, keepdim=True)
    spec = torch.empty_like(imgs)
    nb = side * side // 16
    rec = torch.empty(b * nb * 3, dtype=torch.uint8, device=dev)
    cbp = torch.empty(b * nb, dtype=torch.uint8, device=dev)
    crp = torch.empty(b * nb, dtype=torch.uint8, device=dev)
    px = b * side * side
    res = {}
    res["fft2d_u8_spectrum"] = timed(lambda: ops.fft2d_u8_spectrum(imgs.reshape(-1), side, side, chain.ALPHA,
                                                                   spec.reshape(-1)))
    one = imgs[:1].reshape(-1)
    res["  one image x b"] = b * timed(lambda: ops.fft2d_u8_spectrum(one, side, side, chain.ALPHA, spec[0].reshape(-1)))
    res["encode(spectra)"] = timed(lambda: ops.encode(spec, 1, side, side, cbs, rec, cbp, crp, batch=b,
                                                      shared_codebook=False))
    res["encode(noise)"] = timed(lambda: ops.encode(imgs, 1, side, side, cbs, rec, cbp, crp, batch=b,
                                                    shared_codebook=False))
    be = CudaBackend(outputs="device")
    res["chain"] = timed(lambda: chain.run_chain(imgs, cbs, backend=be), 3)
    for k, v in res.items():
        print(f"{k:18s} {v:8.3f} ms  {px / v / 1e6:9.1f} Mpx/s")
    print("spectrum value histogram (first image):", torch.bincount(spec[0].reshape(-1).long(), minlength=256)
          .nonzero().flatten()[:8].tolist(), "...")


if __name__ == "__main__":
    main()
