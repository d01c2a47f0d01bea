"""1-D transforms above 2^20: ms per launch (median of 10) and the plan's schedule."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

from paper_1203_4938_b200 import ops  # noqa: E402

dev = torch.device("cuda:0")
for m, batch in ((21, 32), (22, 16), (23, 8), (24, 4), (25, 2), (26, 1), (27, 1), (28, 1), (29, 1), (30, 1)):
    n = 1 << m
    x = torch.randn((batch, n), dtype=torch.complex64, device=dev)
    y = torch.empty_like(x)
    for _ in range(3):
        ops.fft_forward(x, n, out=y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.fft_forward(x, n, out=y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[5]
    print(f"2^{m} x {batch}: {ms:.3f} ms, {16 * n * batch / ms / 1e6:.0f} GB/s compulsory "
          f"({16 * n * batch / ms / 1e6 / 6556.5:.3f}) | {ops.fft_plan(1, n, 1, batch, dev).description}", flush=True)
    del x, y
    torch.cuda.empty_cache()
