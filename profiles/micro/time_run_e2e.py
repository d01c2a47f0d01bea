"""End-to-end through the graph API: numpy in -> fft65536 node -> numpy out, chunked."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main() -> None:
    from paper_1203_4938_b200 import CudaBackend, DataType, StreamFile, run
    from paper_1203_4938_b200.apps.fft import fft_program
    n, batch = 65536, 4096
    x = np.random.default_rng(0).standard_normal(2 * n * batch).astype(np.float32)
    sf = StreamFile(DataType("float", 2), x)
    for m, chunk in ((1, None), (1, n * 256), (3, n * 256), (4, n * 128)):
        be = CudaBackend(chunk_size=chunk, max_in_flight=m)
        run(be, fft_program(n), {"0.x": sf})
        t0 = time.perf_counter()
        reps = 3
        for _ in range(reps):
            run(be, fft_program(n), {"0.x": sf})
        dt = (time.perf_counter() - t0) / reps
        print(f"max_in_flight={m} chunk={chunk}: {dt * 1e3:.1f} ms  {5 * n * 16 * batch / dt / 1e9:.1f} GFLOP/s")


if __name__ == "__main__":
    main()
