"""16384-point FFT A/B: L2-ring kernel vs the register-resident single-CTA
kernel (DPP_RR16K=1); ms per 2^28 points and the max rel-L2 against numpy.
The register kernel is kept unbuilt as fft16k_rr_experiment.cu; to rerun, build it
into an A/B library (build_variant.py) with its DPP_RR16K hook in fft.cu."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1203_4938_b200 import ops  # noqa: E402

n, batch = 16384, 16384
dev = torch.device("cuda:0")
x = torch.randn((batch, n), dtype=torch.complex64, device=dev, generator=torch.Generator(device=dev).manual_seed(3))
y = torch.empty_like(x)
for _ in range(3):
    ops.fft_forward(x, n, out=y)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.fft_forward(x, n, out=y)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[5]
rows = [0, 1, 777, batch - 1]
err = max(float(np.linalg.norm(y[r].cpu().numpy() - np.fft.fft(x[r].cpu().numpy().astype(np.complex128)))
                / np.linalg.norm(np.fft.fft(x[r].cpu().numpy().astype(np.complex128)))) for r in rows)
small = ops.fft_forward(x[:5].clone(), n)  # batch below the grid
err5 = float((small - y[:5]).abs().max())
print(f"DPP_RR16K={os.environ.get('DPP_RR16K', '-')}: {ms:.4f} ms ({16 * n * batch / ms / 1e6:.0f} GB/s, "
      f"{16 * n * batch / ms / 1e6 / 6556.5:.3f}) rel-L2 {err:.2e} small-batch diff {err5:.2e}", flush=True)
