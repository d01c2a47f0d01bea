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


def _three_nodes(imgs, rows, cols):
    import torch

    from paper_1203_4938_b200 import ops
    from paper_1203_4938_b200.apps import chain
    z = torch.empty((imgs.shape[0], rows, cols), dtype=torch.complex64, device=imgs.device)
    ops.u8_to_complex(imgs.reshape(-1), torch.view_as_real(z).reshape(-1))
    ops.fft2d_forward(z, rows, cols, out=z)
    ref = torch.empty(imgs.numel(), dtype=torch.uint8, device=imgs.device)
    ops.spectrum_u8(torch.view_as_real(z).reshape(-1), ref, chain.ALPHA)
    return ref.view(imgs.shape)


def _point_mirror(spec):
    """S[(-k1) mod R][(-k2) mod C] for a (..., R, C) tensor."""
    import torch
    return torch.roll(torch.flip(spec, dims=(-2, -1)), shifts=(1, 1), dims=(-2, -1))


@pytest.mark.parametrize("rows", [4096, 16384])
def test_fused_pairs_vs_three_nodes(cuda, rows):
    """The fused pass takes real images in pairs (z = a + i b, spectra
    separated in the row pass, each written with its point mirror): within
    float32 rounding of the three separate nodes — off-by-one bytes counted,
    <= 1e-4 of the pixels — and exactly point-symmetric; the odd last image
    takes the single-image schedule and equals the three nodes byte for byte."""
    import torch

    from paper_1203_4938_b200 import ops
    from paper_1203_4938_b200.apps import chain
    g = torch.Generator(device=cuda).manual_seed(rows)
    imgs = torch.randint(0, 256, (3, rows, 4096), dtype=torch.uint8, device=cuda, generator=g)
    imgs[1] = imgs[1] // 4 + 100  # a second image with other statistics (DC, dynamic range)
    fused = torch.empty(imgs.numel(), dtype=torch.uint8, device=cuda)
    assert ops.fft2d_u8_spectrum(imgs.reshape(-1), rows, 4096, chain.ALPHA, fused)
    fused = fused.view(imgs.shape)
    ref = _three_nodes(imgs, rows, 4096)
    assert torch.equal(fused[2], ref[2])  # single-image schedule
    diff = (fused[:2].to(torch.int16) - ref[:2].to(torch.int16)).abs()
    print(f"pair spectra vs three nodes, {rows} rows: {int((diff > 0).sum())} bytes differ of {diff.numel()}")
    assert int(diff.max()) <= 1 and int((diff > 0).sum()) <= 1e-4 * diff.numel()
    assert torch.equal(fused[:2], _point_mirror(fused[:2]))
    # DC / Nyquist columns and rows come from the side fix-up: check them exactly
    # against the three nodes up to the same one-count rounding
    for c in (0, 2048):
        assert int((fused[:2, :, c].to(torch.int16) - ref[:2, :, c].to(torch.int16)).abs().max()) <= 1


def test_fused_chain_graph_records(cuda):
    # 4096-column images: the executor fuses to_complex -> fft2d -> spectrum_u8
    # into two passes (u8 row loads, u8 spectrum stores); the records of the
    # whole graph must equal the encode of the fused pass's own spectra
    import torch

    from paper_1203_4938_b200 import CudaBackend, ops, plan
    from paper_1203_4938_b200.apps import chain
    g = torch.Generator(device=cuda).manual_seed(3)
    imgs = torch.randint(0, 256, (2, 4096, 4096), dtype=torch.uint8, device=cuda, generator=g)
    prog = chain.chain_program(4096, 4096, 256)
    p = plan(prog)
    assert p.fused and len(p.absorbed) == 2
    fused = torch.empty(imgs.numel(), dtype=torch.uint8, device=cuda)
    assert ops.fft2d_u8_spectrum(imgs.reshape(-1), 4096, 4096, chain.ALPHA, fused)
    cbs = torch.randn((2, 256, 16), device=cuda, generator=g)
    out = chain.run_chain(imgs, cbs, backend=CudaBackend(outputs="device"))
    rec = torch.empty(2 * (1024 * 1024) * 3, dtype=torch.uint8, device=cuda)
    cbp = torch.empty(2 * 1024 * 1024, dtype=torch.uint8, device=cuda)
    crp = torch.empty(2 * 1024 * 1024, dtype=torch.uint8, device=cuda)
    ops.encode(fused.view(2, 4096, 4096), 1, 4096, 4096, cbs, rec, cbp, crp, batch=2, shared_codebook=False)
    rec = rec.view(-1, 3)
    for col, key in enumerate(("mu", "sig", "idx")):  # the whole graph, fused, = encode of the fused spectra
        assert torch.equal(out[key].reshape(-1).to(torch.uint8), rec[:, col]), key
