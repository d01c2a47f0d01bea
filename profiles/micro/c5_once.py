"""One fused C5 FFT pass over b x 4096^2 images (for ncu launch lists)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

from paper_1203_4938_b200 import ops
from paper_1203_4938_b200.apps import chain

b = int(sys.argv[1]) if len(sys.argv) > 1 else 64
imgs = torch.randint(0, 256, (b, 4096, 4096), dtype=torch.uint8, device="cuda")
out = torch.empty_like(imgs)
for _ in range(2):
    ops.fft2d_u8_spectrum(imgs.reshape(-1), 4096, 4096, chain.ALPHA, out.reshape(-1))
torch.cuda.synchronize()
