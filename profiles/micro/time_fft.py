"""Time one FFT launch configuration with CUDA events (A/B helper).

    python profiles/micro/time_fft.py [--n 65536 --batch 4096 --iters 20]

Prints ms per launch and the fraction of the measured HBM copy bandwidth.
Set DPP_LIB_PATH to time an alternative build of the library.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main() -> None:
    import torch

    from paper_1203_4938_b200 import ops
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--rank", type=int, default=1)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    x = torch.randn((a.batch, a.n), dtype=torch.complex64, device=dev)
    y = torch.empty_like(x)
    run = (lambda: ops.fft_forward(x, a.n, out=y)) if a.rank == 1 else \
        (lambda: ops.fft2d_forward(x, a.batch, a.n, out=y))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ms = []
    for _ in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    med = ms[len(ms) // 2]
    pfile = Path(__file__).resolve().parents[2] / "MEASURED_PEAKS.json"
    peaks = json.loads(pfile.read_text()) if pfile.exists() else {"hbm_fallback": 6650.0}
    hbm = None
    for k, v in peaks.items():
        if "hbm" in k.lower() and isinstance(v, (int, float)):
            hbm = v
            break
    gbs = 16.0 * a.n * a.batch / med / 1e6
    print(json.dumps({"n": a.n, "batch": a.batch, "ms_median": round(med, 4), "ms_min": round(ms[0], 4),
                      "GBps": round(gbs, 1), "frac": round(gbs / hbm, 4) if hbm else None}))


if __name__ == "__main__":
    main()
