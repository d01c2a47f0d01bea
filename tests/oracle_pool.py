"""Oracle over many rows on every host core (test infrastructure).

The full-size parity tests (tests/test_fullsize_gpu.py) check every row of
the BASELINE-size outputs against the CPU oracle; one process at a time would
take minutes, so the rows are cut into chunks and evaluated by a spawn-context
process pool (spawn: the parent holds a CUDA context, the workers only run
numpy).
"""

from __future__ import annotations

import os
import sys
from concurrent.futures import ProcessPoolExecutor
from multiprocessing import get_context
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def _init():
    if str(ROOT) not in sys.path:
        sys.path.insert(0, str(ROOT))


def _rows(x):
    from oracle import fft_oracle
    return fft_oracle.fft_rows(x)


def _rows_vs(args):
    """Oracle rows of x compared with got: per-row (|d|^2, |ref|^2)."""
    x, got = args
    from oracle import fft_oracle
    ref = fft_oracle.fft_rows(x).astype(np.complex128)
    d = got.astype(np.complex128) - ref
    return (np.abs(d) ** 2).sum(axis=1), (np.abs(ref) ** 2).sum(axis=1)


def workers() -> int:
    return max(1, min(16, len(os.sched_getaffinity(0))))


def pool() -> ProcessPoolExecutor:
    return ProcessPoolExecutor(max_workers=workers(), mp_context=get_context("spawn"), initializer=_init)


def fft_rows(x: np.ndarray, chunk: int, ex: ProcessPoolExecutor) -> np.ndarray:
    """oracle.fft_rows over the rows of x (complex64 result)."""
    parts = ex.map(_rows, [x[i:i + chunk] for i in range(0, len(x), chunk)])
    return np.concatenate(list(parts))


def rows_rel_l2(x: np.ndarray, got: np.ndarray, chunk: int, ex: ProcessPoolExecutor) -> tuple[float, float]:
    """(max per-row rel-L2, whole-array rel-L2) of got against oracle.fft_rows(x)."""
    res = list(ex.map(_rows_vs, [(x[i:i + chunk], got[i:i + chunk]) for i in range(0, len(x), chunk)]))
    num = np.concatenate([r[0] for r in res])
    den = np.concatenate([r[1] for r in res])
    return float(np.sqrt(num / np.maximum(den, 1e-300)).max()), float(np.sqrt(num.sum() / den.sum()))
