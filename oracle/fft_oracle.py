"""CPU oracle for the FFT node — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` arm may import this module.  The product path
(``paper_1203_4938_b200``) never does: it has no CPU fallback.

This is a numpy restatement of the reference radix-2 FFT,
/root/reference/pkg/src/dpp/apps/fft.py, written independently:

* ``naive_dft``            fft.py:32-42   O(N^2) binary64 sum, rounded to complex64
* ``bit_reverse_indices``  fft.py:45-53   bit-reversal permutation
* ``leaf_terms``           fft.py:56-117  the generated dft{2,4,8} body as term lists
* ``leaf_eval``            interp.py:348-358, 432-439  binary32 left-to-right evaluation
* ``fft`` / ``fft_rows``   fft.py:150-174 permute -> leaves (binary32) -> binary64
                           butterflies with twiddles exp(-2 pi i j/span) -> complex64
* ``fft2``                 SURVEY §8(d) C3: fft over every row, then every column

Parity is pinned: tests/test_oracle.py checks ``fft`` against golden outputs of
the reference itself (tests/golden/fft_golden.npz, made by
tests/golden/make_golden.py) bit-for-bit, and ``leaf_eval`` against the
reference engine's leaf outputs bit-for-bit.
"""

from __future__ import annotations

import numpy as np

__all__ = ["naive_dft", "bit_reverse_indices", "leaf_terms", "leaf_eval", "fft", "fft_rows",
           "fft2", "MAX_LEAF_ORDER"]

MAX_LEAF_ORDER = 3


def naive_dft(signal) -> np.ndarray:
    x = np.asarray(signal).astype(np.complex128)
    n = len(x)
    if n < 1:
        raise ValueError("signal must have at least one sample")
    pos = np.arange(n)
    out = np.array([(x * np.exp((-2j * np.pi * k / n) * pos)).sum() for k in range(n)],
                   dtype=np.complex128)
    return out.astype(np.complex64)


def bit_reverse_indices(n: int) -> np.ndarray:
    bits = int(n).bit_length() - 1
    src = np.arange(n, dtype=np.int64)
    out = np.zeros(n, dtype=np.int64)
    for _ in range(bits):
        out = (out << 1) | (src & 1)
        src = src >> 1
    return out


def _snapped(t: int, size: int) -> tuple[float, float]:
    ang = -2.0 * np.pi * (t % size) / size
    c, s = float(np.cos(ang)), float(np.sin(ang))
    for e in (-1.0, 0.0, 1.0):
        c = e if abs(c - e) < 1e-12 else c
        s = e if abs(s - e) < 1e-12 else s
    return c, s


def leaf_terms(k: int) -> list[list[tuple[int, float]]]:
    """Per output lane: ordered (input lane, signed binary32 coefficient) terms.

    Zero coefficients are dropped, +-1 kept as +-1.0, others become the
    binary32 literal of |c| with the sign of c (fft.py:68-83)."""
    size = 1 << k
    rev = bit_reverse_indices(size)
    outs: list[list[tuple[int, float]]] = [[] for _ in range(2 * size)]
    for j in range(size):
        for n in range(size):
            c, s = _snapped(j * n, size)
            at = int(rev[n])
            for lane_out, coeff, lane_in in ((2 * j, c, 2 * at), (2 * j, -s, 2 * at + 1),
                                             (2 * j + 1, s, 2 * at), (2 * j + 1, c, 2 * at + 1)):
                if coeff != 0.0:
                    mag = 1.0 if abs(coeff) == 1.0 else float(np.float32(abs(coeff)))
                    outs[lane_out].append((lane_in, -mag if coeff < 0 else mag))
    return outs


def leaf_eval(k: int, x: np.ndarray) -> np.ndarray:
    """Evaluate the dft{2^k} node over work-items x[items, 2^(k+1)] in binary32."""
    x = np.asarray(x, np.float32).reshape(-1, 2 << k)
    out = np.empty_like(x)
    with np.errstate(all="ignore"):
        for lane, terms in enumerate(leaf_terms(k)):
            acc = None
            for src, coeff in terms:
                mag = np.float32(abs(coeff))
                term = x[:, src] if mag == 1.0 else mag * x[:, src]
                if acc is None:
                    acc = -term if coeff < 0 else term
                else:
                    acc = acc - term if coeff < 0 else acc + term
            out[:, lane] = acc
    return out


def fft_rows(x: np.ndarray, k: int = MAX_LEAF_ORDER) -> np.ndarray:
    """Reference fft() applied independently to every row of a 2-D complex64 array."""
    x = np.ascontiguousarray(x, np.complex64)
    rows, n = x.shape
    if n < 2 or n & (n - 1):
        raise ValueError(f"transform size must be a power of two, got {n}")
    if not 1 <= k <= MAX_LEAF_ORDER or (1 << k) > n:
        raise ValueError("bad leaf order")
    perm = np.ascontiguousarray(x[:, bit_reverse_indices(n)])
    leaves = leaf_eval(k, perm.view(np.float32).reshape(-1, 2 << k))
    data = leaves.reshape(rows, 2 * n).view(np.complex64).astype(np.complex128)
    for stage in range(k + 1, n.bit_length()):
        span = 1 << stage
        half = span // 2
        blk = data.reshape(rows, n // span, span)
        tw = np.exp(-2j * np.pi * np.arange(half) / span)
        lo = blk[..., :half].copy()
        hi = blk[..., half:] * tw
        blk[..., :half] = lo + hi
        blk[..., half:] = lo - hi
    return data.astype(np.complex64)


def fft(signal, n: int | None = None, k: int = MAX_LEAF_ORDER) -> np.ndarray:
    x = np.ascontiguousarray(signal, np.complex64)
    if n is not None and n != len(x):
        raise ValueError(f"plan is for {n} samples, got {len(x)}")
    return fft_rows(x[None, :], k)[0]


def fft2(x: np.ndarray, k: int = MAX_LEAF_ORDER) -> np.ndarray:
    """2-D composition used as the C3/C5 oracle: rows, then columns."""
    x = np.ascontiguousarray(x, np.complex64)
    rows = fft_rows(x, k)
    return np.ascontiguousarray(fft_rows(np.ascontiguousarray(rows.T), k).T)
