"""cProfile of the C1 path: fft(x) for one N=1024 numpy signal through the graph API."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    import numpy as np
    from paper_1203_4938_b200.apps import fft as afft
    rng = np.random.default_rng(42)
    x = (rng.standard_normal(1024) + 1j * rng.standard_normal(1024)).astype(np.complex64)
    for _ in range(20):
        afft.fft(x)
    t = time.perf_counter()
    for _ in range(200):
        afft.fft(x)
    print("median-ish ms", (time.perf_counter() - t) / 200 * 1e3)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        afft.fft(x)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(30)


if __name__ == "__main__":
    main()
