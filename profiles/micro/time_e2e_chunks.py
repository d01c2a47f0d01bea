"""C2 end to end from pinned host memory (apps.fft.fft_batch) — the chunk size
of the H2D / FFT / D2H pipeline is read from DPP_PIPE_CHUNK_MB at import."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    import torch
    from paper_1203_4938_b200.apps.fft import fft_batch
    n, b = 65536, 4096
    x = torch.randn((b, n), dtype=torch.complex64).pin_memory()
    y = torch.empty_like(x).pin_memory()
    for _ in range(2):
        fft_batch(x, n, out=y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        fft_batch(x, n, out=y)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    ms = sorted(ts)[len(ts) // 2] * 1e3
    print(f"chunk {sys.argv[1] if len(sys.argv) > 1 else '?'} MB: {ms:.2f} ms  "
          f"{5 * n * 16 * b / ms / 1e6:.1f} GFLOP/s  {2 * 8 * n * b / ms / 1e6:.1f} GB/s over PCIe")


if __name__ == "__main__":
    main()
