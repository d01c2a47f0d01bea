"""Generate golden vectors by running the REFERENCE implementation itself.

Run inside the build container (the reference is importable there, not on the
GPU box):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Outputs (committed):
  fft_golden.npz   reference fft() outputs: the acceptance ladder N=8..4096 x
                   k=1..3 on seed-42 signals (test_acceptance.py:170-205), the
                   C1 case N=1024 k=3 (test_fft.py:91-96), and N=16384 k=3.
  leaf_golden.npz  reference engine outputs of the dft2/4/8 leaf programs on
                   random work-items (bit-exact targets for the native leaf).
  imgc_golden.npz  reference compress() bitstreams for the test fixtures and
                   reference node outputs (ycbcr, boxdown, gradient, vq).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def main() -> None:
    from dpp import LocalBackend, StreamFile, run
    from dpp.apps import fft as rfft
    from dpp.apps import imgc as rimgc
    from dpp.types import DataType

    # -- FFT ---------------------------------------------------------------
    out = {}
    rng = np.random.default_rng(42)
    for m in range(3, 13):
        n = 1 << m
        x = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
        rng.standard_normal(n), rng.standard_normal(n)  # the acceptance test also draws y
        out[f"x_{n}"] = x
        for k in (1, 2, 3):
            out[f"y_{n}_k{k}"] = rfft.fft(x, rfft.FftPlan(n, k))
        out[f"naive_{n}"] = rfft.naive_dft(x) if n <= 1024 else np.zeros(0, np.complex64)
    r42 = np.random.default_rng(42)
    c1 = (r42.standard_normal(1024) + 1j * r42.standard_normal(1024)).astype(np.complex64)
    out["c1_x"] = c1
    out["c1_y"] = rfft.fft(c1, rfft.FftPlan(1024, 3))
    r7 = np.random.default_rng(7)
    big = (r7.standard_normal(16384) + 1j * r7.standard_normal(16384)).astype(np.complex64)
    out["x_16384"] = big
    out["y_16384_k3"] = rfft.fft(big, rfft.FftPlan(16384, 3))
    np.savez_compressed(HERE / "fft_golden.npz", **out)

    # -- leaf nodes through the reference engine -----------------------------
    leaf = {}
    r = np.random.default_rng(5)
    for k in (1, 2, 3):
        w = 2 ** (k + 1)
        vals = (r.standard_normal(300 * w) * 10).astype(np.float32)
        res = run(LocalBackend(), rfft.leaf_program(k),
                  {"0.x": StreamFile(DataType("float", w), vals)})["0.y"].values
        leaf[f"x_k{k}"] = vals
        leaf[f"y_k{k}"] = res
        leaf[f"body_k{k}"] = np.frombuffer(rfft.leaf_kernel(k).body.encode(), np.uint8)
    np.savez_compressed(HERE / "leaf_golden.npz", **leaf)

    # -- image codec ---------------------------------------------------------
    img = {}
    cases = {
        "fix64_cb32_s4": (rimgc.synthetic_image(64, 64, seed=9), 32, 4),
        "fix32_cb16_s5": (rimgc.synthetic_image(32, 32, seed=10), 16, 5),
        "fix48x32_cb16_s1": (rimgc.synthetic_image(48, 32, seed=11), 16, 1),
        "single_cb1_s2": (rimgc.synthetic_image(4, 4, seed=3), 1, 2),
        "gray77_cb8_s3": (np.full((32, 32, 3), 77, np.uint8), 8, 3),
        "fix128_cb256_s0": (rimgc.synthetic_image(128, 128, seed=12), 256, 0),
        "fix512_cb256_s0": (rimgc.synthetic_image(512, 512, seed=7), 256, 0),
    }
    g = rimgc.synthetic_image(256, 256, seed=7)[..., 1]
    cases["gray256_cb256_s0"] = (np.repeat(g[..., None], 3, 2), 256, 0)
    for name, (image, ncb, seed) in cases.items():
        blob = rimgc.compress(image, ncb, seed=seed).to_bytes()
        img[f"{name}_image"] = image
        img[f"{name}_blob"] = np.frombuffer(blob, np.uint8)
        img[f"{name}_meta"] = np.array([ncb, seed])
        dec = rimgc.decompress(rimgc.CompressedImage.from_bytes(blob))
        img[f"{name}_decoded"] = dec

    # node-level outputs
    rr = np.random.default_rng(2)
    rgba = rr.integers(0, 256, (4096, 4)).astype(np.uint8)
    rgba[:, 3] = 0
    res = run(LocalBackend(chunk_size=4096), rimgc.ycbcr_program(),
              {"0.rgb": StreamFile(DataType("uchar", 4), rgba.ravel())})
    img["ycbcr_in"] = rgba
    for p in ("yl", "cb", "cr"):
        img[f"ycbcr_{p}"] = res[f"0.{p}"].values
    gray = np.repeat(np.arange(256, dtype=np.uint8)[:, None], 4, 1)
    gray[:, 3] = 0
    res = run(LocalBackend(chunk_size=256), rimgc.ycbcr_program(),
              {"0.rgb": StreamFile(DataType("uchar", 4), gray.ravel())})
    for p in ("yl", "cb", "cr"):
        img[f"gray_{p}"] = res[f"0.{p}"].values
    blk = (rr.standard_normal((500, 16)) * 40 + 128).astype(np.float32)
    res = run(LocalBackend(chunk_size=500), rimgc.chroma_down_program(),
              {"0.blk": StreamFile(DataType("float", 16), blk.ravel())})
    img["box_in"] = blk
    img["box_out"] = res["0.avg"].values
    w, h = 24, 16
    lum = (rr.standard_normal(w * h) * 30 + 100).astype(np.float32)
    res = run(LocalBackend(chunk_size=w * h), rimgc.gradient_program(w, h),
              {"0.lum": StreamFile(DataType("float"), lum)})
    img["grad_in"] = lum
    img["grad_dx"] = res["0.dx"].values
    img["grad_dy"] = res["0.dy"].values
    blocks = rr.standard_normal((256, 16)).astype(np.float32)
    cents = rr.standard_normal((64, 16)).astype(np.float32)
    blocks[:8] = cents[[3, 3, 7, 9, 0, 63, 63, 1]]  # exact hits: distance 0
    tiled = np.tile(cents, (4, 1))
    res = run(LocalBackend(chunk_size=64), rimgc.vq_program(64),
              {"0.blk": StreamFile(DataType("float", 16), blocks.ravel()),
               "0.cbk": StreamFile(DataType("float", 16), tiled.ravel())})
    img["vq_blocks"] = blocks
    img["vq_cents"] = cents
    img["vq_idx"] = res["0.idx"].values
    # program bodies (the native registry matches them exactly)
    for name, prog in (("ycbcr", rimgc.ycbcr_program()), ("boxdown", rimgc.chroma_down_program()),
                       ("gradient_24x16", rimgc.gradient_program(24, 16)),
                       ("vq_64", rimgc.vq_program(64))):
        (node,) = prog.kernels.values()
        img[f"body_{name}"] = np.frombuffer(node.body.encode(), np.uint8)
    np.savez_compressed(HERE / "imgc_golden.npz", **img)

    # -- documents: canonical bytes + ids from the reference model, and the
    # reference's verdict on this framework's native-node bodies --------------
    import json
    sys.path.insert(0, str(HERE.parents[1]))
    from dpp import parse_program, program_id, serialize_program, validate
    from paper_1203_4938_b200 import serialize_program as our_serialize
    from paper_1203_4938_b200.apps import fft as offt
    from paper_1203_4938_b200.apps import imgc as oimgc
    docs = {}
    progs = {"leaf1": rfft.leaf_program(1), "leaf2": rfft.leaf_program(2),
             "leaf3": rfft.leaf_program(3), "ycbcr": rimgc.ycbcr_program(),
             "boxdown": rimgc.chroma_down_program(), "gradient": rimgc.gradient_program(640, 480),
             "vq256": rimgc.vq_program(256)}
    for name, prog in progs.items():
        docs[f"{name}_doc"] = np.frombuffer(serialize_program(prog), np.uint8)
        docs[f"{name}_id"] = np.frombuffer(program_id(prog).encode(), np.uint8)
    ours = {"fft8": offt.fft_program(8), "fft1024": offt.fft_program(1024),
            "fft65536": offt.fft_program(65536), "fft2d_8x16": offt.fft2d_program(8, 16),
            "encode_64x32": oimgc.encode_program(64, 32, 16)}
    for name, prog in ours.items():
        ref_prog = parse_program(our_serialize(prog))
        rep = validate(ref_prog)
        docs[f"ours_{name}_valid"] = np.array([rep.ok])
        docs[f"ours_{name}_id"] = np.frombuffer(program_id(ref_prog).encode(), np.uint8)
    # the self-describing fft node executed BY THE REFERENCE ENGINE (small n)
    rs = np.random.default_rng(3)
    xs = (rs.standard_normal(3 * 16) + 1j * rs.standard_normal(3 * 16)).astype(np.complex64)
    res = run(LocalBackend(chunk_size=16), parse_program(our_serialize(offt.fft_program(16))),
              {"0.x": StreamFile(DataType("float", 2), xs.view(np.float32))})["0.y"].values
    docs["ours_fft16_in"] = xs
    docs["ours_fft16_out_refengine"] = res.view(np.complex64)
    # the fused node must fault on the reference interpreter
    try:
        run(LocalBackend(chunk_size=128), parse_program(our_serialize(oimgc.encode_program(64, 32, 16))),
            {"0.px": StreamFile(DataType("uchar", 16), np.zeros(128 * 16, np.uint8)),
             "0.cbk": StreamFile(DataType("float", 16), np.zeros(128 * 16, np.float32))})
        docs["ours_encode_faults"] = np.array([False])
    except Exception as exc:  # noqa: BLE001
        docs["ours_encode_faults"] = np.array([True])
        docs["ours_encode_fault_msg"] = np.frombuffer(str(exc).encode(), np.uint8)
    # C5 chain adapters: reference validation + reference-engine outputs
    from paper_1203_4938_b200.apps import chain as ochain
    from paper_1203_4938_b200.model import Instance as OInst, Program as OProg
    cprog = ochain.chain_program(64, 32, 16)
    docs["ours_chain_valid"] = np.array([validate(parse_program(our_serialize(cprog))).ok])
    for name, node in (("to_complex", ochain.to_complex_kernel()), ("spectrum_u8", ochain.spectrum_u8_kernel())):
        one = parse_program(our_serialize(OProg({node.name: node}, (OInst(0, node.name),), ())))
        docs[f"ours_{name}_valid"] = np.array([validate(one).ok])
        if name == "to_complex":
            xin = rs.integers(0, 256, 1024).astype(np.uint8)
            res = run(LocalBackend(chunk_size=1024), one, {"0.x": StreamFile(DataType("uchar"), xin)})["0.y"]
        else:
            mag = np.exp(rs.uniform(-2, 22, 4096))
            ph = rs.uniform(0, 2 * np.pi, 4096)
            xin = (mag * np.exp(1j * ph)).astype(np.complex64).view(np.float32)
            res = run(LocalBackend(chunk_size=4096), one, {"0.x": StreamFile(DataType("float", 2), xin)})["0.y"]
        docs[f"ours_{name}_in"] = xin
        docs[f"ours_{name}_out_refengine"] = res.values
    docs["table2_doc"] = np.frombuffer(json.dumps(
        json.loads(serialize_program(parse_program(json.dumps(_table2()).encode())))).encode(), np.uint8)
    np.savez_compressed(HERE / "docs_golden.npz", **docs)
    print("wrote", sorted(p.name for p in HERE.glob("*.npz")), file=sys.stderr)


def _table2() -> dict:
    sys.path.insert(0, str(HERE.parent))
    from conftest import table2_doc
    return table2_doc()


if __name__ == "__main__":
    main()
