"""Device executor: the reference engine contract, native nodes, device-resident edges."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import complex_signals, rel_l2, table2_doc
from oracle import fft_oracle as fo

pytestmark = pytest.mark.gpu


def test_leaf_program_through_run_matches_reference_engine(cuda, leaf_golden):
    from paper_1203_4938_b200 import CudaBackend, DataType, StreamFile, run
    from paper_1203_4938_b200.apps.fft import leaf_program
    for k in (1, 2, 3):
        w = 2 ** (k + 1)
        sf = StreamFile(DataType("float", w), leaf_golden[f"x_k{k}"])
        for chunk in (None, 7, 4096):  # chunking never changes per-item results
            out = run(CudaBackend(chunk_size=chunk), leaf_program(k), {"0.x": sf})["0.y"]
            assert np.array_equal(out.values, leaf_golden[f"y_k{k}"])


def test_leaf_known_answers(cuda):  # test_fft.py:45-52
    from paper_1203_4938_b200 import DataType, LocalBackend, StreamFile, run
    from paper_1203_4938_b200.apps.fft import leaf_program
    sf = StreamFile(DataType("float", 4), np.array([1, 0, 1, 0], np.float32))
    assert np.array_equal(run(LocalBackend(), leaf_program(1), {"0.x": sf})["0.y"].values, [2, 0, 0, 0])
    sf = StreamFile(DataType("float", 4), np.array([3, 1, 5, -1], np.float32))
    assert np.allclose(run(LocalBackend(), leaf_program(1), {"0.x": sf})["0.y"].values, [8, 0, -2, 2])


def test_reference_program_objects_are_accepted(cuda, docs_golden):
    """A document serialised by the reference parses and runs unchanged."""
    from paper_1203_4938_b200 import DataType, StreamFile, parse_program, run
    doc = docs_golden["leaf3_doc"].tobytes()
    prog = parse_program(doc)
    x = np.random.default_rng(0).standard_normal(16 * 10).astype(np.float32)
    out = run(None, prog, {"0.x": StreamFile(DataType("float", 16), x)})["0.y"].values
    assert np.array_equal(out, fo.leaf_eval(3, x).ravel())


def test_fft_node_chunking_and_partial_signal_fault(cuda):
    from paper_1203_4938_b200 import CudaBackend, DataType, EngineRuntimeError, StreamFile, run
    from paper_1203_4938_b200.apps.fft import fft_program
    x = complex_signals(3, (6, 256))
    sf = StreamFile(DataType("float", 2), x.reshape(-1).view(np.float32))
    for chunk in (256, 512, 1536, None):
        out = run(CudaBackend(chunk_size=chunk), fft_program(256), {"0.x": sf})["0.y"]
        got = out.values.view(np.complex64).reshape(6, 256)
        for g, r in zip(got, fo.fft_rows(x)):
            assert rel_l2(g, r) <= 8e-5
    with pytest.raises(EngineRuntimeError) as info:
        run(CudaBackend(chunk_size=384), fft_program(256), {"0.x": sf})
    assert info.value.chunk == 0 and info.value.work_item == 256


def test_device_resident_chain_fft_then_leaf(cuda):
    """Two native nodes joined by an arrow: the edge stays a device tensor."""
    import torch

    from paper_1203_4938_b200 import (Arrow, CudaBackend, DataType, DeviceStream, Instance, Program,
                                      run)
    from paper_1203_4938_b200.apps.fft import fft_kernel, leaf_kernel
    a, b = fft_kernel(64), leaf_kernel(1)
    prog = Program({a.name: a, b.name: b}, (Instance(0, a.name), Instance(1, b.name)),
                   (Arrow((0, "y"), (1, "x")),))
    x = complex_signals(9, (4, 64))
    dev = torch.from_numpy(x.reshape(-1).view(np.float32).copy()).to(cuda)
    out = run(CudaBackend(outputs="device"), prog, {"0.x": DeviceStream(DataType("float", 2), dev)})
    y = out["1.y"]
    assert isinstance(y, DeviceStream) and y.tensor.is_cuda
    mid = fo.fft_rows(x).reshape(-1).view(np.float32)
    ref = fo.leaf_eval(1, mid).ravel()
    assert np.allclose(y.tensor.cpu().numpy(), ref, rtol=1e-5, atol=1e-3)


def test_table2_graph_runs_through_the_jit(cuda):
    # bodies with no hand-written kernel are compiled for sm_100a (jit.py);
    # the reference's Table II graph: z = fan.x + rot(fan.y)
    from paper_1203_4938_b200 import DataType, PlanError, StreamFile, parse_program, plan, run
    prog = parse_program(json.dumps(table2_doc()))
    assert all(k.kind.startswith("jit:") for k in plan(prog).kernels.values())
    zin = np.random.default_rng(4).standard_normal(2 * 999).astype(np.float32)
    out = run(None, prog, {"0.z": StreamFile(DataType("float", 2), zin)})["2.z"].values
    assert np.array_equal(out, zin[0::2] + zin[1::2] * np.float32(65536.0))
    # ill-typed as printed in the paper (a shift on float points): PlanError, like the reference
    with pytest.raises(PlanError, match="shift requires integer operands"):
        plan(parse_program(json.dumps(table2_doc(rot_body="int i=get_global_id(0);\ny[i]=x[i]<<16;\n"))))


def test_client_errors(cuda):
    from paper_1203_4938_b200 import ClientError, DataType, StreamFile, run
    from paper_1203_4938_b200.apps.fft import fft_program
    with pytest.raises(ClientError, match="missing input"):
        run(None, fft_program(8), {})
    with pytest.raises(ClientError, match="carries"):
        run(None, fft_program(8), {"0.x": StreamFile(DataType("float", 4), np.zeros(8, np.float32))})
    with pytest.raises(ClientError, match="not a free input"):
        run(None, fft_program(8), {"0.x": StreamFile(DataType("float", 2), np.zeros(16, np.float32)),
                                   "0.q": StreamFile(DataType("float", 2), np.zeros(16, np.float32))})


def test_codec_program_with_broadcast_codebook(cuda, imgc_golden):
    """The fused imgc_encode node inside run(): codebook as a broadcast side input."""
    from paper_1203_4938_b200 import CudaBackend, DataType, StreamFile, run
    from paper_1203_4938_b200.apps import imgc
    blob = imgc_golden["gray256_cb256_s0_blob"].tobytes()
    ref = imgc.CompressedImage.from_bytes(blob)
    gray = np.ascontiguousarray(imgc_golden["gray256_cb256_s0_image"][..., 0])
    frames = np.concatenate([gray.ravel(), gray.ravel()])  # two frames in one chunk
    prog = imgc.encode_program(256, 256, 256)
    out = run(CudaBackend(), prog, {
        "0.px": StreamFile(DataType("uchar", 16), frames),
        "0.cbk": StreamFile(DataType("float", 16), ref.codebook.centroids.ravel())})
    nb = 64 * 64
    for f in range(2):
        sl = slice(f * nb, (f + 1) * nb)
        assert np.array_equal(out["0.mu"].values[sl], ref.means)
        assert np.array_equal(out["0.sig"].values[sl], ref.sigma_idx)
        assert np.array_equal(out["0.idx"].values[sl], ref.indices)
        assert np.array_equal(out["0.cb"].values[sl], ref.cb.ravel())
        assert np.array_equal(out["0.cr"].values[sl], ref.cr.ravel())


def test_reference_codec_nodes_through_run(cuda, imgc_golden):
    from paper_1203_4938_b200 import CudaBackend, DataType, StreamFile, run
    from paper_1203_4938_b200.apps import imgc
    rgba = imgc_golden["ycbcr_in"]
    out = run(CudaBackend(chunk_size=4096), imgc.ycbcr_program(),
              {"0.rgb": StreamFile(DataType("uchar", 4), rgba.ravel())})
    assert np.array_equal(out["0.yl"].values, imgc_golden["ycbcr_yl"])
    blocks, cents = imgc_golden["vq_blocks"], imgc_golden["vq_cents"]
    out = run(CudaBackend(chunk_size=64), imgc.vq_program(64),
              {"0.blk": StreamFile(DataType("float", 16), blocks.ravel()),
               "0.cbk": StreamFile(DataType("float", 16), np.tile(cents, (4, 1)).ravel())})
    assert np.array_equal(out["0.idx"].values, imgc_golden["vq_idx"])


def test_chunked_host_streams_pipeline(cuda):
    # chunk size set + host streams: H2D / kernels / D2H of consecutive chunks on
    # three streams (client._run_pipelined); identical to the one-slot path,
    # ragged last chunk, outputs in order
    from paper_1203_4938_b200 import CudaBackend, DataType, StreamFile, run
    from paper_1203_4938_b200.apps.fft import fft_program, leaf_program
    x = complex_signals(11, (301, 1024))
    sf = StreamFile(DataType("float", 2), x.reshape(-1).view(np.float32))
    outs = [run(CudaBackend(chunk_size=1024 * 32, max_in_flight=m), fft_program(1024), {"0.x": sf})["0.y"].values
            for m in (1, 2, 3)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    got = outs[2].view(np.complex64).reshape(301, 1024)
    for g, r in zip(got[::37], fo.fft_rows(x[::37])):
        assert rel_l2(g, r) <= 1e-5 * 10
    y = np.random.default_rng(5).standard_normal(16 * 10007).astype(np.float32)
    sf = StreamFile(DataType("float", 16), y)
    a = run(CudaBackend(chunk_size=1000, max_in_flight=3), leaf_program(3), {"0.x": sf})["0.y"].values
    assert np.array_equal(a, fo.leaf_eval(3, y).ravel())


def test_fft2d_node_without_a_native_schedule_runs_its_body(cuda):
    """fft2d_8x16 (column length < 256): the node's naive-DFT body through the
    JIT on the GPU — the document's meaning (tests/golden/docs_golden.npz)."""
    from paper_1203_4938_b200 import DataType, StreamFile, run
    from paper_1203_4938_b200.apps.fft import fft2d_program
    rng = np.random.default_rng(3)
    x = (rng.standard_normal((2, 8, 16)) + 1j * rng.standard_normal((2, 8, 16))).astype(np.complex64)
    sf = StreamFile(DataType("float", 2), x.view(np.float32).reshape(-1))
    y = run(None, fft2d_program(8, 16), {"0.x": sf})["0.y"].values.view(np.complex64).reshape(2, 8, 16)
    ref = np.fft.fft2(x.astype(np.complex128))
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) < 1e-5
