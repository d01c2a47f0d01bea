"""Quick parity check of the 1-D FFT against numpy (float64) for a few batches."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main() -> None:
    import torch
    from paper_1203_4938_b200 import ops
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(5)
    worst = 0.0
    for batch in (1, 3, 17, 41, 97, 300):
        x = (rng.standard_normal((batch, n)) + 1j * rng.standard_normal((batch, n))).astype(np.complex64)
        xt = torch.from_numpy(x).to(dev)
        got = ops.fft_forward(xt, n).cpu().numpy()
        ref = np.fft.fft(x.astype(np.complex128), axis=-1)
        err = np.linalg.norm(got - ref, axis=-1) / np.linalg.norm(ref, axis=-1)
        worst = max(worst, float(err.max()))
        # in place
        ops.fft_forward(xt, n, out=xt)
        got2 = xt.cpu().numpy()
        assert np.array_equal(got, got2), "in-place differs"
        print(f"batch {batch}: max rel-L2 {err.max():.3e}")
    print("worst", worst, "OK" if worst < 1e-5 * np.log2(n) else "FAIL")


if __name__ == "__main__":
    main()
