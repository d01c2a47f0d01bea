"""PCIe ceiling for the C2 e2e line: pinned 2 GiB H2D alone, D2H alone, and
both at once on two streams (full duplex) in chunks of 32 MB / 128 MB /
2 GiB, CUDA events.  Prints one JSON line."""
import json
import sys

import torch


def timed(fn, reps=3):
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    nbytes = 2 << 30
    dev = torch.device("cuda:0")
    h_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d_a = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d_b = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    h_in.fill_(1)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def both(chunk):
        def run():
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            for off in range(0, nbytes, chunk):
                with torch.cuda.stream(s1):
                    d_a[off:off + chunk].copy_(h_in[off:off + chunk], non_blocking=True)
                with torch.cuda.stream(s2):
                    h_out[off:off + chunk].copy_(d_b[off:off + chunk], non_blocking=True)
            cur.wait_stream(s1)
            cur.wait_stream(s2)
        return run

    out = {}
    out["h2d_ms"] = timed(lambda: d_a.copy_(h_in, non_blocking=True))
    out["d2h_ms"] = timed(lambda: h_out.copy_(d_b, non_blocking=True))
    for mb in (32, 128, 2048):
        out[f"duplex_{mb}MB_ms"] = timed(both(mb << 20))
    gb = nbytes / 1e9
    out["h2d_GBps"] = gb / out["h2d_ms"] * 1e3
    out["d2h_GBps"] = gb / out["d2h_ms"] * 1e3
    best = min(v for k, v in out.items() if k.startswith("duplex"))
    out["duplex_GBps_each_way"] = gb / best * 1e3
    flop = 5 * 65536 * 16 * 4096
    out["c2_e2e_ceiling_GFLOPs"] = flop / (best * 1e-3) / 1e9
    print(json.dumps({k: round(v, 3) for k, v in out.items()}))


if __name__ == "__main__":
    sys.exit(main())
