"""A/B one FFT size across library builds: CUDA-event median per launch plus
a bitwise digest of the output (same seeded input), so a variant is only
kept when it is both faster and bit-identical.

    DPP_LIB_PATH=alt/x.so python profiles/micro/ab_c2.py [--n 65536 --batch 4096]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main() -> None:
    import torch

    from paper_1203_4938_b200 import ops
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=30)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(1234)
    x = torch.randn((a.batch, a.n), dtype=torch.complex64, device=dev, generator=g)
    y = torch.empty_like(x)
    for _ in range(3):
        ops.fft_forward(x, a.n, out=y)
    torch.cuda.synchronize()
    w = y.view(torch.int32).view(-1)
    digest = int((w.to(torch.int64) * (torch.arange(w.numel(), device=dev) % 1000003 + 1)).sum().item())
    ms = []
    for _ in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.fft_forward(x, a.n, out=y)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    med = ms[len(ms) // 2]
    gbs = 16.0 * a.n * a.batch / med / 1e6
    print(json.dumps({"lib": os.path.basename(os.environ.get("DPP_LIB_PATH", "shipped")), "n": a.n,
                      "batch": a.batch, "ms_median": round(med, 4), "ms_min": round(ms[0], 4),
                      "GBps": round(gbs, 1), "digest": digest}))


if __name__ == "__main__":
    main()
