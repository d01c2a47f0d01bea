"""Micro-benchmark: copy bandwidth for L2-resident vs HBM-sized buffers (torch copy_)."""
import torch

dev = torch.device("cuda:0")
for mb in (8, 16, 32, 48, 64, 96, 2048):
    n = mb * 1024 * 1024 // 4
    a = torch.randn(n, device=dev)
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = max(3, int(2000 / mb))
    e0.record()
    for _ in range(it):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    print(f"{mb:5d} MB  {2 * n * 4 / (ms / 1e3) / 1e9:8.1f} GB/s (read+write)")
