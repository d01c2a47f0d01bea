import sys, torch
sys.path.insert(0, '.')
from paper_1203_4938_b200 import ops
dev = torch.device("cuda:0"); g = torch.Generator(device=dev).manual_seed(0)
h = w = 8192
img = torch.randint(0, 256, (h, w), dtype=torch.uint8, device=dev, generator=g)
cb = torch.randn((256, 16), device=dev, generator=g); cb = (cb - cb.mean(1, keepdim=True)) / cb.std(1, unbiased=False, keepdim=True)
nb = (h // 4) * (w // 4)
rec = torch.empty(nb * 3, dtype=torch.uint8, device=dev); cbp = torch.empty(nb, dtype=torch.uint8, device=dev); crp = torch.empty(nb, dtype=torch.uint8, device=dev)
for _ in range(3): ops.encode(img, 1, h, w, cb, rec, cbp, crp)
torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): ops.encode(img, 1, h, w, cb, rec, cbp, crp)
e1.record(); torch.cuda.synchronize(); print("C4 ms", e0.elapsed_time(e1) / 10)
