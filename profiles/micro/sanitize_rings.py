"""compute-sanitizer driver: two transforms per ring size (argv: log2 sizes)."""
import sys, torch
sys.path.insert(0, '.')
from paper_1203_4938_b200 import ops
for m in [int(a) for a in sys.argv[1:] if a.isdigit()]:
    n = 1 << m
    x = torch.randn((2, n), dtype=torch.complex64, device="cuda")
    y = ops.fft_forward(x, n)
    torch.cuda.synchronize()
    print(m, "ok", flush=True)


def extra():
    """2-D column ring (plain, TW via the three-pass path), one-rank sharded pass, k-means shard."""
    from paper_1203_4938_b200.distributed import PeerShardedFft2d
    from paper_1203_4938_b200.kmeans import kmeans_sharded
    x = torch.randn((4096, 64), dtype=torch.complex64, device="cuda")
    ops.fft2d_forward(x, 4096, 64)
    y = torch.randn((1, 1 << 21), dtype=torch.complex64, device="cuda")
    ops.fft_forward(y, 1 << 21, out=y)
    sh = PeerShardedFft2d(4096, 64, 1)
    sh(x.view(1, 4096, 64), transpose_back=True)
    sh(x.view(1, 4096, 64), transpose_back=False)
    kmeans_sharded(torch.randn((3000, 16), dtype=torch.float64, device="cuda"), 32, seed=1)
    torch.cuda.synchronize()
    print("extra ok", flush=True)


if __name__ == "__main__" and "--extra" in sys.argv:
    extra()
