"""The CPU oracle is pinned to the reference's own outputs before it judges anything.

Goldens come from running the reference itself (tests/golden/make_golden.py);
known-answer tests are the reference's (pkg/tests/test_fft.py, test_imgc.py).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import fft_oracle as fo
from oracle import imgc_oracle as io


# -- numpy reduction order self-check ------------------------------

@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_numpy_pairwise_order_is_the_one_the_kernels_implement(dtype):
    rng = np.random.default_rng(0)
    a = (rng.standard_normal((50000, 16)) * rng.uniform(1e-3, 1e3, (50000, 1))).astype(dtype)
    r = a[:, :8] + a[:, 8:]
    pw = ((r[:, 0] + r[:, 1]) + (r[:, 2] + r[:, 3])) + ((r[:, 4] + r[:, 5]) + (r[:, 6] + r[:, 7]))
    assert np.array_equal(pw, a.sum(axis=1))
    assert np.array_equal(pw / 16, a.mean(axis=1))
    m = a.mean(axis=1)
    d = (a - m[:, None]) ** 2
    r = d[:, :8] + d[:, 8:]
    pw = ((r[:, 0] + r[:, 1]) + (r[:, 2] + r[:, 3])) + ((r[:, 4] + r[:, 5]) + (r[:, 6] + r[:, 7]))
    assert np.array_equal(np.sqrt(pw / 16), a.std(axis=1))


# -- FFT oracle -------------------------------------------------------------------

def test_naive_dft_known_answers():  # test_fft.py:18-36
    assert np.allclose(fo.naive_dft(np.array([1, 0, 0, 0], np.complex64)), np.ones(4), atol=1e-6)
    assert np.allclose(fo.naive_dft(np.array([1, 2, 3, 4], np.complex64)),
                       [10, -2 + 2j, -2, -2 - 2j], atol=1e-5)
    out = fo.naive_dft(np.full(8, 2.5, np.complex64))
    assert abs(out[0] - 20) < 1e-5 and np.abs(out[1:]).max() < 1e-5
    assert fo.naive_dft(np.array([3 + 4j], np.complex64))[0] == np.complex64(3 + 4j)


def test_bit_reverse_known_answer():  # test_fft.py:41-42
    assert list(fo.bit_reverse_indices(8)) == [0, 4, 2, 6, 1, 5, 3, 7]


def test_leaf_known_answers():  # test_fft.py:45-52
    assert np.array_equal(fo.leaf_eval(1, np.array([1, 0, 1, 0], np.float32)).ravel(), [2, 0, 0, 0])
    assert np.allclose(fo.leaf_eval(1, np.array([3, 1, 5, -1], np.float32)).ravel(), [8, 0, -2, 2])


@pytest.mark.parametrize("k", [1, 2, 3])
def test_leaf_eval_bit_exact_vs_reference_engine(leaf_golden, k):
    got = fo.leaf_eval(k, leaf_golden[f"x_k{k}"]).ravel()
    assert np.array_equal(got, leaf_golden[f"y_k{k}"])


def test_fft_bit_exact_vs_reference_ladder(fft_golden):
    for m in range(3, 13):
        n = 1 << m
        for k in (1, 2, 3):
            assert np.array_equal(fo.fft(fft_golden[f"x_{n}"], n, k), fft_golden[f"y_{n}_k{k}"]), (n, k)


def test_fft_bit_exact_c1_and_16k(fft_golden):
    assert np.array_equal(fo.fft(fft_golden["c1_x"], 1024, 3), fft_golden["c1_y"])
    assert np.array_equal(fo.fft(fft_golden["x_16384"], 16384, 3), fft_golden["y_16384_k3"])


def test_fft_rows_matches_per_row_calls(fft_golden):
    x = np.stack([fft_golden[f"x_{256}"], fft_golden[f"x_{256}"][::-1].copy()])
    rows = fo.fft_rows(x)
    assert np.array_equal(rows[0], fo.fft(x[0]))
    assert np.array_equal(rows[1], fo.fft(x[1]))


def test_fft_oracle_vs_naive(fft_golden):  # test_acceptance.py:170-205 criterion
    for m in range(3, 11):
        n = 1 << m
        ref = fft_golden[f"naive_{n}"]
        got = fo.fft(fft_golden[f"x_{n}"], n, 3)
        assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-4


def test_fft2_composition_vs_numpy():
    rng = np.random.default_rng(1)
    x = (rng.standard_normal((32, 64)) + 1j * rng.standard_normal((32, 64))).astype(np.complex64)
    ref = np.fft.fft2(x.astype(np.complex128))
    assert np.linalg.norm(fo.fft2(x) - ref) / np.linalg.norm(ref) < 1e-6


# -- codec oracle ---------------------------------------------------------------------

def _cases(imgc_golden):
    return sorted(k[:-5] for k in imgc_golden.files if k.endswith("_blob"))


def test_codec_bitstreams_bit_exact_vs_reference(imgc_golden):
    for name in _cases(imgc_golden):
        if name.startswith("fix512"):
            continue  # covered below (slow-ish)
        ncb, seed = imgc_golden[f"{name}_meta"]
        blob = io.compress(imgc_golden[f"{name}_image"], int(ncb), int(seed))
        assert blob == imgc_golden[f"{name}_blob"].tobytes(), name


def test_codec_512_fixture_bit_exact(imgc_golden):
    blob = io.compress(imgc_golden["fix512_cb256_s0_image"], 256, 0)
    assert blob == imgc_golden["fix512_cb256_s0_blob"].tobytes()
    # SPEC acceptance: ratio <= 0.13, PSNR >= 25 dB (test_acceptance.py:266-279)
    img = imgc_golden["fix512_cb256_s0_image"]
    assert len(blob) / img.nbytes <= 0.13
    assert io.psnr(img, io.decode(io.from_bytes(blob))) >= 25.0


def test_decode_bit_exact_vs_reference(imgc_golden):
    for name in _cases(imgc_golden):
        dec = io.decode(io.from_bytes(imgc_golden[f"{name}_blob"].tobytes()))
        assert np.array_equal(dec, imgc_golden[f"{name}_decoded"]), name


def test_node_level_outputs_bit_exact(imgc_golden):
    y, cb, cr = io.ycbcr(imgc_golden["ycbcr_in"][:, :3])
    assert np.array_equal(y, imgc_golden["ycbcr_yl"])
    assert np.array_equal(cb, imgc_golden["ycbcr_cb"])
    assert np.array_equal(cr, imgc_golden["ycbcr_cr"])
    blk = imgc_golden["box_in"]
    acc = blk[:, 0].copy()
    for m in range(1, 16):
        acc = acc + blk[:, m]
    assert np.array_equal(acc * np.float32(0.0625), imgc_golden["box_out"])
    assert np.array_equal(io.vq_nearest(imgc_golden["vq_blocks"], imgc_golden["vq_cents"]),
                          imgc_golden["vq_idx"])


def test_container_size_formula():  # test_imgc.py:222-229
    img = io.synthetic_image(64, 64, seed=12)
    f = io.encode(img, None, 256, 0)
    blob = io.to_bytes(f)
    assert len(blob) == 18 + len(f["codebook"]) * 64 + 3 * 256 + 2 * 256


def test_uniform_gray_exact_round_trip():  # test_imgc.py:156-160
    gray = np.full((32, 32, 3), 77, np.uint8)
    f = io.encode(gray, None, 8, 3)
    assert int(f["sigma_idx"].max()) == 0
    assert np.array_equal(io.decode(f), gray)


def test_kmeans_properties():  # test_imgc.py:90-128
    rng = np.random.default_rng(6)
    pts = rng.standard_normal((400, 16))
    trace: list[float] = []
    io.kmeans(pts, 16, seed=2, trace=trace)
    assert all(b <= a + 1e-9 for a, b in zip(trace, trace[1:]))
    pts = rng.standard_normal((256, 16))
    assert io.kmeans(pts, 32, 9).tobytes() == io.kmeans(pts, 32, 9).tobytes()
    with pytest.raises(ValueError, match="exceeds"):
        io.kmeans(np.zeros((3, 16)), 4, seed=0)
