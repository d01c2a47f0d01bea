"""Time the row-sharded C3 path at one rank (PEER column kernel, both output
modes) against the plain single-GPU 2-D plan on 16384^2 — the fused exchange
must cost nothing when there is nothing to exchange."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    import torch
    from paper_1203_4938_b200 import ops
    from paper_1203_4938_b200.distributed import PeerShardedFft2d
    n = 16384
    dev = torch.device("cuda:0")
    x = torch.randn((n, n), dtype=torch.complex64, device=dev)
    sh = PeerShardedFft2d(n, n, 1)
    sh.slab.copy_(x.view(1, n, n))

    def t(fn, k=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k

    print("plan2d in place      %.3f ms" % t(lambda: ops.fft2d_forward(x, n, n, out=x)))
    print("peer  transpose_back %.3f ms" % t(lambda: sh(None, transpose_back=True)))
    print("peer  column slab    %.3f ms" % t(lambda: sh(None, transpose_back=False)))


if __name__ == "__main__":
    main()
