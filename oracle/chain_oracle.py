"""CPU oracle for the C5 chain — TEST INFRASTRUCTURE ONLY.

The chain (gray -> complex -> 2-D FFT -> u8 log-magnitude -> compression) is
defined by SURVEY §8(d) C5; the reference has no such graph, so the oracle is
composed from reference pieces:

* ``to_complex`` / ``spectrum_u8``: the adapter node bodies of
  paper_1203_4938_b200/apps/chain.py evaluated the way the reference
  interpreter does (numpy binary32 ops, interp.py:312-366, 408-419), pinned
  bit-for-bit against the reference engine's own outputs
  (tests/golden/docs_golden.npz);
* ``fft_oracle.fft2``: reference fft() over rows then columns;
* ``imgc_oracle.encode``: reference compress() with the given codebook.
"""

from __future__ import annotations

import numpy as np

from . import fft_oracle, imgc_oracle

_F = np.float32


def to_complex(gray: np.ndarray) -> np.ndarray:
    return np.asarray(gray, np.uint8).astype(_F).astype(np.complex64)


def spectrum_u8(z: np.ndarray, alpha: float = 11.5) -> np.ndarray:
    z = np.asarray(z, np.complex64)
    re, im = z.real.astype(_F), z.imag.astype(_F)
    with np.errstate(all="ignore"):
        m = np.sqrt(re * re + im * im)
        v = np.floor(_F(alpha) * np.log(_F(1.0) + m))
        return np.maximum(np.minimum(v, _F(255.0)), _F(0.0)).astype(np.uint8)  # fmin(fmax(v,0),255)


def chain(gray: np.ndarray, codebook: np.ndarray, alpha: float = 11.5) -> tuple[np.ndarray, dict]:
    """(adapter output, container fields) for one gray image."""
    spec = spectrum_u8(fft_oracle.fft2(to_complex(gray)), alpha)
    rgb = np.repeat(spec[..., None], 3, axis=2)
    return spec, imgc_oracle.encode(rgb, codebook)
