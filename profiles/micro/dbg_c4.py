import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1203_4938_b200 import ops
dev = torch.device("cuda:0")
for (h, w) in [(64, 64), (256, 256), (1024, 1024), (8192, 8192)]:
    gen = torch.Generator(device=dev).manual_seed(0)
    img = torch.randint(0, 256, (h, w), dtype=torch.uint8, device=dev, generator=gen)
    cb = torch.randn((256, 16), device=dev, generator=gen); cb = (cb - cb.mean(1, keepdim=True)) / cb.std(1, unbiased=False, keepdim=True)
    nb = (h // 4) * (w // 4)
    outs = []
    for mode in ("exact", "tc", "tc"):
        os.environ["DPP_IMGC_VQ"] = mode
        rec = torch.empty(nb * 3, dtype=torch.uint8, device=dev); cbp = torch.empty(nb, dtype=torch.uint8, device=dev); crp = torch.empty(nb, dtype=torch.uint8, device=dev)
        ops.encode(img, 1, h, w, cb, rec, cbp, crp)
        torch.cuda.synchronize()
        outs.append(rec.view(-1, 3).cpu().numpy())
    for m in (1, 2):
        bad = np.nonzero((outs[0] != outs[m]).any(1))[0]
        f = [int(((outs[0][:, q] != outs[m][:, q])).sum()) for q in range(3)]
        print(h, w, "run", m, "bad blocks", len(bad), "per field", f, "first", bad[:8], "tiles", np.unique(bad // 128)[:10])
