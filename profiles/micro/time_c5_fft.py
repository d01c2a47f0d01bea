"""The fused C5 FFT pass alone, b x 4096^2 (CUDA events, median of 7 x 3 calls)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

from paper_1203_4938_b200 import ops
from paper_1203_4938_b200.apps import chain

b = int(sys.argv[1]) if len(sys.argv) > 1 else 64
imgs = torch.randint(0, 256, (b, 4096, 4096), dtype=torch.uint8, device="cuda")
out = torch.empty_like(imgs)
f = lambda: ops.fft2d_u8_spectrum(imgs.reshape(-1), 4096, 4096, chain.ALPHA, out.reshape(-1))
f()
torch.cuda.synchronize()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        f()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 3)
ts.sort()
print(f"{os.environ.get('DPP_LIB_PATH', 'shipped')}: {ts[3]:.3f} ms per {b} images (min {ts[0]:.3f})")
