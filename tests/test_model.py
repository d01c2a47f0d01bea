"""Graph API mirror: documents, ids and rules match the reference's (CPU only)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from paper_1203_4938_b200 import (Arrow, DataType, Direction, Instance, IOPoint, Node, Program,
                                  ProgramFormatError, StreamFile, free_points, parse_program,
                                  program_id, serialize_program, topological_order, validate)
from paper_1203_4938_b200.apps import fft as afft
from paper_1203_4938_b200.apps import imgc as aimgc

from conftest import table2_doc

TABLE2_ID = "fe7c14426649a2ffca378754dca3637c587c376f6c5db57167585ce9e286bf47"  # test_model.py:182


def test_table2_id_is_the_reference_id():
    assert program_id(parse_program(json.dumps(table2_doc()).encode())) == TABLE2_ID


def test_key_order_and_whitespace_do_not_change_the_id():
    doc = table2_doc()
    a = program_id(parse_program(json.dumps(doc)))
    b = program_id(parse_program(json.dumps(doc, indent=3, sort_keys=True)))
    assert a == b == TABLE2_ID


@pytest.mark.parametrize("name,prog", [
    ("leaf1", afft.leaf_program(1)), ("leaf2", afft.leaf_program(2)), ("leaf3", afft.leaf_program(3)),
    ("ycbcr", aimgc.ycbcr_program()), ("boxdown", aimgc.chroma_down_program()),
    ("gradient", aimgc.gradient_program(640, 480)), ("vq256", aimgc.vq_program(256)),
])
def test_generated_programs_are_byte_identical_to_the_reference(docs_golden, name, prog):
    assert serialize_program(prog) == docs_golden[f"{name}_doc"].tobytes()
    assert program_id(prog) == docs_golden[f"{name}_id"].tobytes().decode()


@pytest.mark.parametrize("name", ["fft8", "fft1024", "fft65536", "fft2d_8x16", "encode_64x32"])
def test_native_node_documents_validate_on_the_reference(docs_golden, name):
    assert bool(docs_golden[f"ours_{name}_valid"][0])


def test_ids_of_native_node_documents_agree(docs_golden):
    assert program_id(afft.fft_program(1024)) == docs_golden["ours_fft1024_id"].tobytes().decode()
    assert program_id(aimgc.encode_program(64, 32, 16)) == \
        docs_golden["ours_encode_64x32_id"].tobytes().decode()


def test_fused_node_faults_on_the_reference_interpreter(docs_golden):
    assert bool(docs_golden["ours_encode_faults"][0])


def test_fft_node_body_means_the_dft_on_the_reference_engine(docs_golden):
    from oracle.fft_oracle import naive_dft
    x = docs_golden["ours_fft16_in"]
    y = docs_golden["ours_fft16_out_refengine"]
    for s in range(3):
        ref = naive_dft(x[16 * s:16 * (s + 1)])
        assert np.abs(y[16 * s:16 * (s + 1)] - ref).max() / np.abs(ref).max() < 1e-5


def test_chain_documents_validate_and_adapters_are_pinned(docs_golden):
    """C5 chain: the reference validates the whole graph and each adapter; the
    oracle adapters equal the reference engine's outputs bit for bit."""
    from oracle import chain_oracle as co
    for name in ("chain", "to_complex", "spectrum_u8"):
        assert bool(docs_golden[f"ours_{name}_valid"][0]), name
    x = docs_golden["ours_to_complex_in"]
    assert np.array_equal(co.to_complex(x).view(np.float32), docs_golden["ours_to_complex_out_refengine"])
    z = docs_golden["ours_spectrum_u8_in"].view(np.complex64)
    assert np.array_equal(co.spectrum_u8(z), docs_golden["ours_spectrum_u8_out_refengine"])


def test_parse_rejections():
    with pytest.raises(ProgramFormatError, match="missing key"):
        parse_program('{"kernels": {}, "nodes": []}')
    doc = table2_doc()
    doc["arrows"].append({"output": [0, "x"], "input": [0, "z"]})
    with pytest.raises(ProgramFormatError, match="same instance"):
        parse_program(json.dumps(doc))
    doc = table2_doc()
    doc["nodes"].append([0, {"kernel": "fan"}])
    with pytest.raises(ProgramFormatError, match="duplicate instance"):
        parse_program(json.dumps(doc))
    with pytest.raises(ProgramFormatError, match="unknown key"):
        parse_program('{"kernels": {}, "nodes": [], "arrows": [], "x": 1}')


def test_topological_order_and_free_points():
    p = parse_program(json.dumps(table2_doc()))
    assert topological_order(p) == [0, 1, 2]
    assert [fp.stream for fp in free_points(p)] == ["0.z", "2.z"]
    assert validate(p).ok


def test_validate_reports_cycles_and_type_mismatch():
    f = DataType("float")
    a = Node("a", "x", (IOPoint("i", f, Direction.INPUT), IOPoint("o", f, Direction.OUTPUT)))
    b = Node("b", "x", (IOPoint("i", DataType("int"), Direction.INPUT),
                        IOPoint("o", f, Direction.OUTPUT)))
    prog = Program({"a": a, "b": b}, (Instance(0, "a"), Instance(1, "b")),
                   (Arrow((0, "o"), (1, "i")), Arrow((1, "o"), (0, "i"))))
    kinds = {v.kind for v in validate(prog).violations}
    assert {"cycle", "arrow-type-mismatch", "no-free-input", "no-free-output"} <= kinds


def test_stream_file_round_trip():
    sf = StreamFile.from_values("float2", np.arange(8, dtype=np.float32))
    back = StreamFile.from_bytes(sf.to_bytes())
    assert back.data == sf.data and np.array_equal(back.values, sf.values) and back.count == 4


def test_fft_plan_rules():  # test_fft.py:99-105
    with pytest.raises(ValueError, match="power of two"):
        afft.FftPlan(12)
    with pytest.raises(ValueError, match="leaf size"):
        afft.FftPlan(4, 3)


def test_parse_sizes():  # test_fft.py:132-140
    sizes = afft.parse_sizes("20K..10M")
    assert sizes[0] == 20 * 1024 and sizes[-1] == 10 * 1024 * 1024
    assert afft.parse_sizes("64K, 1M") == [65536, 1048576]


def test_ppm_round_trip(tmp_path):  # test_imgc.py:17-37
    image = aimgc.synthetic_image(20, 12, seed=1)
    aimgc.write_ppm(image, tmp_path / "a.ppm")
    assert np.array_equal(aimgc.read_ppm(tmp_path / "a.ppm"), image)
    assert aimgc.read_ppm(b"P6\n# c\n2 1\n# d\n255\n" + bytes(6)).shape == (1, 2, 3)
    for blob, frag in ((b"P5\n1 1\n255\n\x00", "not a binary PPM"),
                       (b"P6\n2 2\n65535\n" + bytes(24), "maxval 255"),
                       (b"P6\n4 4\n255\n" + bytes(5), "expected 48")):
        with pytest.raises(ValueError, match=frag):
            aimgc.read_ppm(blob)


def test_container_round_trip_host(imgc_golden):
    blob = imgc_golden["fix32_cb16_s5_blob"].tobytes()
    ci = aimgc.CompressedImage.from_bytes(blob)
    assert ci.to_bytes() == blob
    assert ci.block_count == 64
