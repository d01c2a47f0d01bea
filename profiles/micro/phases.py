"""Phase timeline of the MODE 7 2^16 kernel from a -DDPP_PHASES build.

    nvcc ... -DDPP_PHASES (see profiles/micro/build_alt.sh phases)
    DPP_LIB_PATH=.../libdpp_phases.so DPP_FFT_CLUSTER_MODE=7 python profiles/micro/phases.py

Per CTA (thread 0): clock64 at start, tile landed, pass 1 done, cluster
barrier passed, scatter issued, receive complete, pass 2 done, store read.
"""
from __future__ import annotations

import ctypes
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main() -> None:
    import torch

    from paper_1203_4938_b200 import _lib, ops
    dev = torch.device("cuda:0")
    batch = 4096
    x = torch.randn((batch, 65536), dtype=torch.complex64, device=dev)
    y = torch.empty_like(x)
    for _ in range(3):
        ops.fft_forward(x, 65536, out=y)
    torch.cuda.synchronize()
    lib = _lib.load()
    n = 65536 * 12
    buf = (ctypes.c_longlong * n)()
    fn = lib.dpp_debug_phases
    fn.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
    assert fn(buf, n) == 0
    a = np.frombuffer(buf, dtype=np.int64).reshape(65536, 12)
    clk = 1.93e3  # cycles per us (approx; sm clock under load)
    names = ["tile wait", "pass 1", "barrier", "scatter", "recv wait", "pass 2", "store+exit"]
    d = np.diff(a[:, :8], axis=1) / clk
    out = {nm: {"mean_us": round(float(d[:, k].mean()), 3), "p50": round(float(np.median(d[:, k])), 3),
                "p90": round(float(np.percentile(d[:, k], 90)), 3)} for k, nm in enumerate(names)}
    life = (a[:, 10] - a[:, 9]) / 1e3
    out["lifetime_us_globaltimer"] = {"mean": round(float(life.mean()), 3), "p50": round(float(np.median(life)), 3)}
    t0 = a[:, 9].min()
    span = (a[:, 10].max() - t0) / 1e3
    out["span_us"] = round(float(span), 1)
    # resident CTAs per SM over time
    sm = a[:, 8]
    ev = []
    for s_, b_, e_ in zip(sm, a[:, 9] - t0, a[:, 10] - t0):
        ev.append((b_, 1))
        ev.append((e_, -1))
    ev.sort()
    cur, acc, last = 0, 0.0, 0
    for tt, dd in ev:
        acc += cur * (tt - last)
        cur += dd
        last = tt
    out["mean_resident_ctas_per_sm"] = round(acc / (a[:, 10].max() - t0) / 148, 2)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
