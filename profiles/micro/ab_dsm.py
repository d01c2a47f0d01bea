"""C2 kernel A/B: the L2-ring kernel vs the DSMEM cluster kernel (DPP_FFT_DSM=2|3
groups), same input; prints ms per launch (median of 20) and an output digest
(the two kernels run the same butterflies: digests must match).
The DSMEM kernel is kept unbuilt as fft_dsm_experiment.cu; to rerun, build it
into an A/B library (build_variant.py) with its DPP_FFT_DSM hook in fft_l2.cu."""
import hashlib
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import torch  # noqa: E402

from paper_1203_4938_b200 import ops  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(42)
x = torch.randn((batch, 65536), dtype=torch.complex64, device=dev, generator=g)
y = torch.empty_like(x)
for _ in range(3):
    ops.fft_forward(x, 65536, out=y)
torch.cuda.synchronize()
ms = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.fft_forward(x, 65536, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
ms.sort()
dig = hashlib.sha256(y.view(torch.uint8).cpu().numpy().tobytes()).hexdigest()[:16]
print(f"DPP_FFT_DSM={os.environ.get('DPP_FFT_DSM', '-')} batch {batch}: {ms[10]:.4f} ms "
      f"({16 * 65536 * batch / ms[10] / 1e6:.0f} GB/s) digest {dig}", flush=True)
