"""2-D 4096 x 4096 x 16 images (2^28 points): ms per launch; DPP_LIB_PATH picks the library."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

from paper_1203_4938_b200 import ops  # noqa: E402

dev = torch.device("cuda:0")
x = torch.randn((16, 4096, 4096), dtype=torch.complex64, device=dev)
y = torch.empty_like(x)
for _ in range(3):
    ops.fft2d_forward(x, 4096, 4096, out=y)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.fft2d_forward(x, 4096, 4096, out=y)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(os.environ.get("DPP_LIB_PATH", "tree").split("/")[-1], f"{sorted(ts)[5]:.4f} ms", flush=True)
