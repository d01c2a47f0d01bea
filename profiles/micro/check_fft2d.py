"""Quick parity check of the 2-D FFT against numpy (float64) for the ring column shapes."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main() -> None:
    import torch
    from paper_1203_4938_b200 import ops
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(3)
    for (r, c, b) in ((4096, 2048, 3), (16384, 1024, 1), (4096, 16, 2), (16384, 32, 3)):
        x = (rng.standard_normal((b, r, c)) + 1j * rng.standard_normal((b, r, c))).astype(np.complex64)
        xt = torch.from_numpy(x).to(dev)
        got = ops.fft2d_forward(xt, r, c).cpu().numpy()
        ref = np.fft.fft2(x.astype(np.complex128), axes=(-2, -1))
        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        ops.fft2d_forward(xt, r, c, out=xt)
        same = np.array_equal(xt.cpu().numpy(), got)
        print(f"{r}x{c} b{b}: rel-L2 {err:.3e} in-place-equal {same}", "OK" if err < 1e-5 * np.log2(r * c) and same else "FAIL")
    print(ops.fft_plan(2, 16384, 16384, 1, dev).description)


if __name__ == "__main__":
    main()
