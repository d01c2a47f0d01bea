"""Compression node parity on the B200: bit-exact bitstreams against the reference.

Every bitstream in tests/golden/imgc_golden.npz was produced by the reference
``compress()`` itself; the GPU encoder is fed the codebook stored in that
bitstream (k-means is an input of the node) and must reproduce every byte.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import imgc_oracle as io

pytestmark = pytest.mark.gpu


def _cases(g):
    return sorted(k[:-5] for k in g.files if k.endswith("_blob"))


def test_bitstreams_bit_exact_vs_reference(cuda, imgc_golden):
    from paper_1203_4938_b200.apps import imgc
    for name in _cases(imgc_golden):
        blob = imgc_golden[f"{name}_blob"].tobytes()
        ref = imgc.CompressedImage.from_bytes(blob)
        ci = imgc.compress(imgc_golden[f"{name}_image"], ref.codebook.size, codebook=ref.codebook)
        got = ci.to_bytes()
        if got != blob:
            diff = [f for f in ("means", "sigma_idx", "indices", "cb", "cr")
                    if not np.array_equal(getattr(ci, f), getattr(ref, f))]
            pytest.fail(f"{name}: fields differ: {diff}")


def test_container_written_and_read_on_the_device(cuda, imgc_golden):
    """compress_to_bytes / decompress_bytes (the container assembled and
    parsed on the device) give the reference's own bitstreams and decodes."""
    from paper_1203_4938_b200.apps import imgc
    for name in _cases(imgc_golden):
        blob = imgc_golden[f"{name}_blob"].tobytes()
        ref = imgc.CompressedImage.from_bytes(blob)
        assert imgc.compress_to_bytes(imgc_golden[f"{name}_image"], ref.codebook.size,
                                      codebook=ref.codebook) == blob, name
        assert np.array_equal(imgc.decompress_bytes(blob), imgc_golden[f"{name}_decoded"]), name
    with pytest.raises(ValueError, match="truncated container"):
        imgc.decompress_bytes(blob[:-1])
    with pytest.raises(ValueError, match="bad container magic"):
        imgc.decompress_bytes(b"XXXX" + blob[4:])


@pytest.mark.parametrize("layout", ["gray", "rgb", "rgba"])
def test_channel_layouts_agree(cuda, imgc_golden, layout):
    from paper_1203_4938_b200.apps import imgc
    img3 = imgc_golden["gray256_cb256_s0_image"]
    blob = imgc_golden["gray256_cb256_s0_blob"].tobytes()
    ref = imgc.CompressedImage.from_bytes(blob)
    if layout == "gray":
        img = np.ascontiguousarray(img3[..., 0])
    elif layout == "rgba":
        img = np.concatenate([img3, np.full(img3.shape[:2] + (1,), 200, np.uint8)], axis=2)
    else:
        img = img3
    assert imgc.compress(img, 256, codebook=ref.codebook).to_bytes() == blob


def test_decompress_bit_exact(cuda, imgc_golden):
    from paper_1203_4938_b200.apps import imgc
    for name in _cases(imgc_golden):
        ci = imgc.CompressedImage.from_bytes(imgc_golden[f"{name}_blob"].tobytes())
        assert np.array_equal(imgc.decompress(ci), imgc_golden[f"{name}_decoded"]), name


def test_drop_in_nodes_bit_exact(cuda, imgc_golden):
    import torch

    from paper_1203_4938_b200 import ops
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(cuda)  # noqa: E731
    rgba = t(imgc_golden["ycbcr_in"])
    n = rgba.numel() // 4
    yl, cb, cr = (torch.empty(n, dtype=torch.float32, device=cuda) for _ in range(3))
    ops.ycbcr(rgba, yl, cb, cr)
    assert np.array_equal(yl.cpu().numpy(), imgc_golden["ycbcr_yl"])
    assert np.array_equal(cb.cpu().numpy(), imgc_golden["ycbcr_cb"])
    assert np.array_equal(cr.cpu().numpy(), imgc_golden["ycbcr_cr"])
    blk = t(imgc_golden["box_in"])
    avg = torch.empty(len(imgc_golden["box_in"]), dtype=torch.float32, device=cuda)
    ops.boxdown(blk, avg)
    assert np.array_equal(avg.cpu().numpy(), imgc_golden["box_out"])
    lum = t(imgc_golden["grad_in"])
    dx, dy = torch.empty_like(lum), torch.empty_like(lum)
    ops.gradient(lum, dx, dy, 24, 16)
    assert np.array_equal(dx.cpu().numpy(), imgc_golden["grad_dx"])
    assert np.array_equal(dy.cpu().numpy(), imgc_golden["grad_dy"])
    blocks = t(imgc_golden["vq_blocks"])
    cents = t(imgc_golden["vq_cents"])
    idx = torch.empty(len(imgc_golden["vq_blocks"]), dtype=torch.int32, device=cuda)
    ops.vqnearest(blocks, cents, idx, 64)
    assert np.array_equal(idx.cpu().numpy(), imgc_golden["vq_idx"])


def test_gradient_fault_matches_interpreter(cuda):
    import torch

    from paper_1203_4938_b200 import KernelRuntimeError, ops
    lum = torch.zeros(24 * 15, dtype=torch.float32, device=cuda)  # one row short of 24x16
    dx, dy = torch.empty_like(lum), torch.empty_like(lum)
    with pytest.raises(KernelRuntimeError) as info:
        ops.gradient(lum, dx, dy, 24, 16)
    assert info.value.work_item == 24 * 14  # first lane whose lum[i+24] leaves the chunk
    assert "out of range for point 'lum'" in str(info.value)


def test_block_grad_and_norm32_outputs(cuda):
    import torch

    from paper_1203_4938_b200 import ops
    img = io.synthetic_image(96, 64, seed=21)
    y, _, _ = io.ycbcr(img)
    cents = io.train_codebook(y, 32, 1)
    nb = (64 // 4) * (96 // 4)
    dev = lambda n, dt: torch.empty(n, dtype=dt, device=cuda)  # noqa: E731
    rec, cbp, crp = dev(3 * nb, torch.uint8), dev(nb, torch.uint8), dev(nb, torch.uint8)
    grad, norm = dev(nb, torch.float32), dev(nb * 16, torch.float32)
    ops.encode(torch.from_numpy(img).to(cuda), 3, 64, 96, torch.from_numpy(cents).to(cuda), rec, cbp,
               crp, block_grad=grad, norm32=norm)
    assert np.array_equal(grad.cpu().numpy(), io.gradient(y))
    _, _, n64 = io.block_stats(y)
    assert np.array_equal(norm.cpu().numpy().reshape(-1, 16), n64.astype(np.float32))


def test_batched_encode_equals_single(cuda):
    import torch

    from paper_1203_4938_b200.apps import imgc
    imgs = np.stack([io.synthetic_image(128, 64, seed=s)[..., 1] for s in (1, 2, 3)])
    cbs = np.stack([io.train_codebook(io.ycbcr(np.repeat(g[..., None], 3, 2))[0], 64, 0) for g in imgs])
    rec, cbp, crp = imgc.compress_batch(torch.from_numpy(imgs).cuda(), torch.from_numpy(cbs).cuda())
    for b in range(3):
        f = io.encode(np.repeat(imgs[b][..., None], 3, 2), cbs[b])
        assert np.array_equal(rec[b].cpu().numpy()[:, 0], f["means"])
        assert np.array_equal(rec[b].cpu().numpy()[:, 1], f["sigma_idx"])
        assert np.array_equal(rec[b].cpu().numpy()[:, 2], f["indices"])
        assert np.array_equal(cbp[b].cpu().numpy(), f["cb"].ravel())
        assert np.array_equal(crp[b].cpu().numpy(), f["cr"].ravel())


@pytest.mark.parametrize("mode", ["tc", "exact"])
@pytest.mark.parametrize("shape", [(128, 64), (512, 260), (36, 20)])
def test_planar_records_equal_interleaved(cuda, monkeypatch, mode, shape):
    """dpp_imgc_encode_planar (the graph node's mu / sig / idx outputs) writes
    the same bytes as the interleaved record run, batched, both searches,
    including frames whose tiles straddle block rows."""
    import torch

    from paper_1203_4938_b200 import ops
    if mode == "exact":
        monkeypatch.setenv("DPP_IMGC_VQ", "exact")
    w, h = shape
    imgs = torch.from_numpy(np.stack([io.synthetic_image(w, h, seed=s)[..., 1] for s in (4, 5)])).cuda()
    cb = torch.from_numpy(io.train_codebook(io.ycbcr(np.repeat(imgs[0].cpu().numpy()[..., None], 3, 2))[0],
                                            32, 0)).cuda()
    nb = (w // 4) * (h // 4) * 2
    rec = torch.empty(nb * 3, dtype=torch.uint8, device="cuda")
    cbp, crp = (torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(2))
    ops.encode(imgs, 1, h, w, cb, rec, cbp, crp, batch=2)
    planes = [torch.full((nb,), 7, dtype=torch.uint8, device="cuda") for _ in range(5)]
    ops.encode_planar(imgs, h, w, cb, *planes, batch=2)
    r3 = rec.view(-1, 3)
    for i in range(3):
        assert torch.equal(planes[i], r3[:, i])
    assert torch.equal(planes[3], cbp) and torch.equal(planes[4], crp)


def test_c4_full_size_8192_gray(cuda):
    """C4 at full size: 8192^2 gray (R=G=B).  The oracle (too slow for the whole
    frame) checks the first 64 block rows exactly."""
    import torch

    from paper_1203_4938_b200 import ops
    rng = np.random.default_rng(7)
    base = io.synthetic_image(1024, 1024, seed=7)[..., 1]
    gray = np.tile(base, (8, 8)) ^ (rng.integers(0, 2, (8192, 8192), dtype=np.uint8))
    band = np.repeat(gray[:256, :][..., None], 3, 2)
    cents = io.train_codebook(io.ycbcr(band[:, :1024])[0], 256, 0)
    px = torch.from_numpy(gray).to(cuda)
    nb = 2048 * 2048
    rec = torch.empty(nb * 3, dtype=torch.uint8, device=cuda)
    cbp = torch.empty(nb, dtype=torch.uint8, device=cuda)
    crp = torch.empty(nb, dtype=torch.uint8, device=cuda)
    ops.encode(px, 1, 8192, 8192, torch.from_numpy(cents).to(cuda), rec, cbp, crp)
    got = rec.view(-1, 3)[: 64 * 2048].cpu().numpy()
    f = io.encode(band, cents)
    assert np.array_equal(got[:, 0], f["means"])
    assert np.array_equal(got[:, 1], f["sigma_idx"])
    assert np.array_equal(got[:, 2], f["indices"])
    assert np.array_equal(cbp[: 64 * 2048].cpu().numpy(), f["cb"].ravel())


# -- tensor-core pruned search: identical to the exact search ------------------------

def _encode_tc(cuda, img, cents, delta_scale=1.0):
    import ctypes

    import torch

    from paper_1203_4938_b200 import _lib
    h, w = img.shape[:2]
    ch = 1 if img.ndim == 2 else img.shape[2]
    nb = (h // 4) * (w // 4)
    px = torch.from_numpy(np.ascontiguousarray(img)).to(cuda)
    cb = torch.from_numpy(np.ascontiguousarray(cents, np.float32)).to(cuda)
    rec = torch.empty(nb * 3, dtype=torch.uint8, device=cuda)
    cbp = torch.empty(nb, dtype=torch.uint8, device=cuda)
    crp = torch.empty(nb, dtype=torch.uint8, device=cuda)
    amb = torch.zeros(1, dtype=torch.int64, device=cuda)
    _lib.check(_lib.load().dpp_imgc_encode_tc_debug(px.data_ptr(), ch, h, w, cb.data_ptr(), len(cents),
                                                    rec.data_ptr(), cbp.data_ptr(), crp.data_ptr(),
                                                    ctypes.c_float(delta_scale), amb.data_ptr(), None))
    return rec.view(-1, 3).cpu().numpy(), int(amb.item()), nb


@pytest.mark.parametrize("seed", [0, 1])
def test_tensor_core_search_equals_exact_search(cuda, seed):
    """Whatever the band width, the TC path must give the exact reference
    indices: the re-check makes the result independent of the approximation."""
    img = io.synthetic_image(512, 512, seed=30 + seed)
    y, _, _ = io.ycbcr(img)
    cents = io.train_codebook(y, 256, seed)
    f = io.encode(img, cents)
    for scale in (1.0, 30.0):
        rec, amb, nb = _encode_tc(cuda, img, cents, scale)
        assert np.array_equal(rec[:, 2], f["indices"]), (scale, int((rec[:, 2] != f["indices"]).sum()))
        assert np.array_equal(rec[:, 0], f["means"]) and np.array_equal(rec[:, 1], f["sigma_idx"])
    rec, amb, nb = _encode_tc(cuda, img, cents, 1.0)
    print(f"ambiguous blocks (exact re-check): {amb} of {nb} ({100 * amb / nb:.2f}%)")
    assert amb < 0.1 * nb


def test_tensor_core_search_adversarial_codebooks(cuda):
    """Duplicated centroids (exact ties -> first index), a tiny codebook, a
    codebook with large norms (band scales with |c|max) and one beyond the
    binary16 split's range."""
    rng = np.random.default_rng(4)
    img = io.synthetic_image(256, 128, seed=44)
    y, _, _ = io.ycbcr(img)
    base = io.train_codebook(y, 64, 0)
    dup = np.concatenate([base, base[::-1], base[:5]])       # 133 entries, every vector twice+
    big = (rng.standard_normal((200, 16)) * 6).astype(np.float32)
    # outside the binary16 split's range (|c| > 2^14): every block takes the exact path
    wide = np.concatenate([base, np.full((1, 16), 3.0e4, np.float32), -base[:7] * 1.0e5]).astype(np.float32)
    for cents in (dup, base[:3], big, wide):
        f = io.encode(img, cents)
        rec, amb, nb = _encode_tc(cuda, img, cents)
        assert np.array_equal(rec[:, 2], f["indices"])
    assert amb > 0.5 * nb  # the wide codebook re-checked (almost) every block exactly


def test_flat_blocks_take_the_zero_block_index(cuda):
    """Constant 4x4 blocks normalise to exactly 0; against a normalised codebook
    every centroid is then at |c_j|^2 = 16 (+- rounding), i.e. inside the band.
    The encoder resolves them with the precomputed exact argmin for the zero
    block (no re-check): same indices as the reference, and no ambiguous count."""
    rng = np.random.default_rng(12)
    img = io.synthetic_image(256, 256, seed=51)
    img[:128, :, :] = 117                       # flat half (R=G=B -> constant luma blocks)
    img[128:, :64, :] = rng.integers(0, 256, 3, dtype=np.uint8)
    cents = rng.standard_normal((256, 16)).astype(np.float64)
    cents = ((cents - cents.mean(1, keepdims=True)) / cents.std(1, keepdims=True)).astype(np.float32)
    cents[[17, 200]] = cents[[5, 5]]            # exact duplicates of a candidate
    f = io.encode(img, cents)
    rec, amb, nb = _encode_tc(cuda, img, cents)
    assert np.array_equal(rec[:, 2], f["indices"]) and np.array_equal(rec[:, 1], f["sigma_idx"])
    flat = int((f["sigma_idx"] == 0).sum())
    assert flat >= nb // 2 and amb < nb - flat  # flat blocks never reach the re-check


def test_default_path_is_tensor_core_and_matches_exact(cuda, imgc_golden, monkeypatch):
    from paper_1203_4938_b200.apps import imgc
    blob = imgc_golden["fix512_cb256_s0_blob"].tobytes()
    ref = imgc.CompressedImage.from_bytes(blob)
    image = imgc_golden["fix512_cb256_s0_image"]
    assert imgc.compress(image, 256, codebook=ref.codebook).to_bytes() == blob  # default: TC
    monkeypatch.setenv("DPP_IMGC_VQ", "exact")
    assert imgc.compress(image, 256, codebook=ref.codebook).to_bytes() == blob


# -- GPU k-means codebook (tolerance parity) ----------------------

def test_block_stats_bit_exact(cuda):
    import torch

    from paper_1203_4938_b200.kmeans import block_stats_device
    img = io.synthetic_image(96, 64, seed=22)
    norm64, grad = block_stats_device(torch.from_numpy(img).to(cuda), 3, 64, 96)
    y, _, _ = io.ycbcr(img)
    _, _, ref = io.block_stats(y)
    assert np.array_equal(norm64.cpu().numpy(), ref)
    assert np.array_equal(grad.cpu().numpy(), io.gradient(y))


def test_kmeans_known_answers(cuda):  # test_imgc.py:90-128
    from paper_1203_4938_b200.apps import imgc
    rng = np.random.default_rng(5)
    a = rng.normal(0, 0.01, (300, 16)) + 4.0
    b = rng.normal(0, 0.01, (300, 16)) - 4.0
    cb = imgc.kmeans(np.vstack([a, b]), 2, seed=8)
    lows, highs = sorted(cb.centroids[:, 0])
    assert abs(lows - b[:, 0].mean()) < 1e-2 and abs(highs - a[:, 0].mean()) < 1e-2
    pts = np.array([[float(i)] * 16 for i in range(5)])
    assert sorted(imgc.kmeans(pts, 5, seed=1).centroids[:, 0].tolist()) == [0, 1, 2, 3, 4]
    pts = rng.standard_normal((400, 16))
    trace: list[float] = []
    imgc.kmeans(pts, 16, seed=2, trace=trace)
    assert len(trace) >= 1 and all(y <= x + 1e-9 for x, y in zip(trace, trace[1:]))
    pts = rng.standard_normal((256, 16))
    assert imgc.kmeans(pts, 32, 9).to_bytes() == imgc.kmeans(pts, 32, 9).to_bytes()
    with pytest.raises(ValueError, match="exceeds"):
        imgc.kmeans(np.zeros((3, 16)), 4, seed=0)


def test_kmeans_quality_matches_reference_trainer(cuda):
    """Same training set and seed: the GPU codebook's SSE is within 3% of the
    reference algorithm's (oracle), and the seeding consumes the same RNG stream."""
    from paper_1203_4938_b200.apps import imgc
    img = io.synthetic_image(128, 128, seed=12)
    y, _, _ = io.ycbcr(img)
    _, _, norm = io.block_stats(y)
    train = norm[io.gradient(y) >= 1.0]
    ref = io.kmeans(train, 64, 0)
    got = imgc.kmeans(train, 64, 0).centroids

    def sse(c):
        d = ((train[:, None, :] - c[None].astype(np.float64)) ** 2).sum(-1)
        return d.min(1).sum()

    assert sse(got) <= 1.03 * sse(ref)


def test_compress_without_codebook_end_to_end(cuda, imgc_golden):
    """compress(image, 256, seed) with the GPU trainer: SPEC acceptance on the
    512^2 fixture (ratio <= 0.13, PSNR >= 25 dB, deterministic), and quality
    within 0.5 dB of the reference's own bitstream."""
    from paper_1203_4938_b200.apps import imgc
    image = imgc_golden["fix512_cb256_s0_image"]
    ci = imgc.compress(image, 256, seed=0)
    blob = ci.to_bytes()
    assert len(blob) / image.nbytes <= 0.13
    q = imgc.psnr(image, imgc.decompress(ci))
    ref = imgc.CompressedImage.from_bytes(imgc_golden["fix512_cb256_s0_blob"].tobytes())
    q_ref = imgc.psnr(image, imgc.decompress(ref))
    assert q >= 25.0 and q >= q_ref - 0.5, (q, q_ref)
    assert imgc.compress(image, 256, seed=0).to_bytes() == blob
    # uniform gray and single block (test_imgc.py:156-172)
    gray = np.full((32, 32, 3), 77, np.uint8)
    ci = imgc.compress(gray, 8, seed=3)
    assert int(ci.sigma_idx.max()) == 0 and np.array_equal(imgc.decompress(ci), gray)
    assert len(imgc.compress(io.synthetic_image(4, 4, seed=3), 1, seed=2).means) == 1
