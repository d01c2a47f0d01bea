"""Per-tile timeline of the four-group encoder (alt/prof.so from
make_prof_variant.py): CTA 0, first 64 tiles of each group, clock64 cycles."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1203_4938_b200 import ops, _lib
dev = torch.device("cuda:0"); h = w = 8192
gen = torch.Generator(device=dev).manual_seed(0)
img = torch.randint(0, 256, (h, w), dtype=torch.uint8, device=dev, generator=gen)
cb = torch.randn((256, 16), device=dev, generator=gen); cb = (cb - cb.mean(1, keepdim=True)) / cb.std(1, unbiased=False, keepdim=True)
nb = (h // 4) * (w // 4)
rec = torch.empty(nb * 3, dtype=torch.uint8, device=dev); cbp = torch.empty(nb, dtype=torch.uint8, device=dev); crp = torch.empty(nb, dtype=torch.uint8, device=dev)
for _ in range(3): ops.encode(img, 1, h, w, cb, rec, cbp, crp)
torch.cuda.synchronize()
buf = np.zeros((4, 64, 8), dtype=np.uint64)
_lib.load().dpp_enc_prof_read(ctypes.c_void_p(buf.ctypes.data))
p = buf.astype(np.int64)
names = ["front", "sync", "tmem_wait", "mma_issue", "mma_wait", "rank", "tail"]
for g in range(4):
    d = [np.median(p[g, 2:50, j + 1] - p[g, 2:50, j]) for j in range(7)]
    period = np.median(np.diff(p[g, 2:50, 0]))
    print(f"group {g}: " + " ".join(f"{n} {v:.0f}" for n, v in zip(names, d)) + f" | period {period:.0f}")
