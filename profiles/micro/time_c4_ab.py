"""C4 encoder time (CUDA events, median of 5 x 10 launches) on the bench frame
(synthetic_image(8192, 8192, seed=7) green, the reference codebook) and on
uniform noise with a random normalised codebook.  DPP_LIB_PATH picks the library."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from oracle import imgc_oracle as io  # noqa: E402  (test input generator only)
from paper_1203_4938_b200 import ops  # noqa: E402

dev = torch.device("cuda:0")
h = w = 8192
g = np.load("tests/golden/c4_golden.npz")
frames = {
    "bench": (torch.from_numpy(np.ascontiguousarray(io.synthetic_image(w, h, seed=7)[..., 1])).to(dev),
              torch.from_numpy(g["codebook"]).to(dev)),
}
gen = torch.Generator(device=dev).manual_seed(0)
cb = torch.randn((256, 16), device=dev, generator=gen)
cb = (cb - cb.mean(1, keepdim=True)) / cb.std(1, unbiased=False, keepdim=True)
frames["noise"] = (torch.randint(0, 256, (h, w), dtype=torch.uint8, device=dev, generator=gen), cb)
nb = (h // 4) * (w // 4)
rec = torch.empty(nb * 3, dtype=torch.uint8, device=dev)
cbp = torch.empty(nb, dtype=torch.uint8, device=dev)
crp = torch.empty(nb, dtype=torch.uint8, device=dev)
out = []
for name, (img, cbk) in frames.items():
    for _ in range(3):
        ops.encode(img, 1, h, w, cbk, rec, cbp, crp)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ops.encode(img, 1, h, w, cbk, rec, cbp, crp)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 10)
    import hashlib
    out.append(f"{name} {sorted(ts)[2]:.4f} ms sha {hashlib.sha256(rec.cpu().numpy().tobytes()).hexdigest()[:12]}")
print(os.environ.get("DPP_LIB_PATH", "tree").split("/")[-1], " | ".join(out))
