"""Time each node of the C5 chain (64 x 4096^2) alone and the whole graph, CUDA events."""
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
    b, side = 64, 4096
    g = torch.Generator(device=dev).manual_seed(0)
    imgs = torch.randint(0, 256, (b, side, side), dtype=torch.uint8, device=dev, generator=g)
    cbs = torch.randn((b, 256, 16), dtype=torch.float32, device=dev, generator=g)
    # codebooks as k-means leaves them: centroids of normalised blocks (zero mean, unit deviation)
    cbs = (cbs - cbs.mean(-1, keepdim=True)) / cbs.std(-1, unbiased=False, keepdim=True)
    z = torch.empty((b, side, side), dtype=torch.complex64, device=dev)
    spec = torch.empty((b, side, side), dtype=torch.uint8, device=dev)
    nb = side * side // 16
    rec = torch.empty(b * nb * 3, dtype=torch.uint8, device=dev)
    cbp = torch.empty(b * nb, dtype=torch.uint8, device=dev)
    crp = torch.empty(b * nb, dtype=torch.uint8, device=dev)
    px = b * side * side
    res = {}
    res["to_complex"] = timed(lambda: ops.u8_to_complex(imgs.reshape(-1), torch.view_as_real(z).reshape(-1)))
    res["fft2d"] = timed(lambda: ops.fft2d_forward(z, side, side, out=z))
    res["spectrum"] = timed(lambda: ops.spectrum_u8(torch.view_as_real(z).reshape(-1), spec.reshape(-1), chain.ALPHA))
    res["encode"] = timed(lambda: ops.encode(spec, 1, side, side, cbs, rec, cbp, crp, batch=b, shared_codebook=False))
    be = CudaBackend(outputs="device")
    res["chain"] = timed(lambda: chain.run_chain(imgs, cbs, backend=be), 3)
    for k, v in res.items():
        print(f"{k:12s} {v:8.3f} ms  {px / v / 1e6:9.1f} Mpx/s")


if __name__ == "__main__":
    main()
