"""C5 chain on the B200: FFT -> adapter -> compression, device-resident edges.

Per-edge parity: the 2-D FFT within tolerance, the u8
adapter as a mismatch count (device logf vs numpy log: transcendental), and
the compression records BIT-EXACT on the GPU's own adapter output.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_l2
from oracle import chain_oracle as co
from oracle import fft_oracle as fo
from oracle import imgc_oracle as io

pytestmark = pytest.mark.gpu


def _images(b, h, w):
    return np.stack([io.synthetic_image(w, h, seed=1000 + i)[..., 1] for i in range(b)])


def test_chain_graph_per_edge_parity(cuda):
    import torch

    from paper_1203_4938_b200 import ops
    from paper_1203_4938_b200.apps import chain
    b, h, w = 3, 256, 256
    imgs = _images(b, h, w)
    # edges computed step by step on the device
    px = torch.from_numpy(imgs).to(cuda)
    z = torch.empty((b, h, w), dtype=torch.complex64, device=cuda)
    ops.u8_to_complex(px.reshape(-1), torch.view_as_real(z).reshape(-1))
    ops.fft2d_forward(z, h, w, out=z)
    spec = torch.empty((b, h, w), dtype=torch.uint8, device=cuda)
    ops.spectrum_u8(torch.view_as_real(z).reshape(-1), spec.reshape(-1), chain.ALPHA)
    zs, specs = z.cpu().numpy(), spec.cpu().numpy()
    mismatches = 0
    cbs = []
    for i in range(b):
        ref_z = fo.fft2(co.to_complex(imgs[i]))
        assert rel_l2(zs[i], ref_z) <= 1e-5 * 16
        mismatches += int((co.spectrum_u8(zs[i]) != specs[i]).sum())  # same FFT input: adapter only
        cbs.append(io.train_codebook(io.ycbcr(np.repeat(specs[i][..., None], 3, 2))[0], 64, i))
    assert mismatches <= 1e-4 * imgs.size, mismatches  # logf vs numpy log, counted
    # the whole graph through run(): records must equal the oracle encode of the GPU's adapter output
    cbs = np.stack(cbs)
    out = chain.run_chain(imgs, cbs)
    nb = (h // 4) * (w // 4)
    for i in range(b):
        f = io.encode(np.repeat(specs[i][..., None], 3, 2), cbs[i])
        sl = slice(i * nb, (i + 1) * nb)
        assert np.array_equal(out["mu"][sl], f["means"])
        assert np.array_equal(out["sig"][sl], f["sigma_idx"])
        assert np.array_equal(out["idx"][sl], f["indices"])
        assert np.array_equal(out["cb"][sl], f["cb"].ravel())
        assert np.array_equal(out["cr"][sl], f["cr"].ravel())


def test_chain_device_resident_shared_codebook(cuda):
    import torch

    from paper_1203_4938_b200 import CudaBackend
    from paper_1203_4938_b200.apps import chain
    imgs = torch.from_numpy(_images(2, 512, 256)).to(cuda)
    cb = torch.from_numpy(io.kmeans(np.random.default_rng(0).standard_normal((4096, 16)), 32, 0)).to(cuda)
    out = chain.run_chain(imgs, cb, backend=CudaBackend(outputs="device"))
    assert all(t.is_cuda for t in out.values())
    assert out["mu"].numel() == 2 * 128 * 64
