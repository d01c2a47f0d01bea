"""JIT of kernel-language nodes against the reference evaluator.

CPU: the front end accepts exactly the bodies the reference accepts (same
diagnostic text and position for the rejected ones) and every generated
kernel compiles with NVRTC for sm_100a.  GPU: outputs equal the reference
evaluator's bit for bit (transcendental builtins: a few ulp), faults name the
same message and work-item, untouched outputs stay zero.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from jit_corpus import CASES

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def jit_meta():
    return json.loads((GOLD / "jit_golden.json").read_text())


@pytest.fixture(scope="module")
def jit_arrays():
    return np.load(GOLD / "jit_golden.npz")


def _node(case):
    from paper_1203_4938_b200.model import Node
    from paper_1203_4938_b200.types import DataType, Direction, IOPoint
    io = tuple(IOPoint(p, DataType(b, w), Direction.INPUT if d == "in" else Direction.OUTPUT)
               for p, (b, w, d) in case["io"].items())
    return Node(case["name"], case["body"], io)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_front_end_matches_reference_verdict(case, jit_meta):
    from paper_1203_4938_b200.errors import KernelError
    from paper_1203_4938_b200.kernel import compile_kernel
    from paper_1203_4938_b200.kernel.codegen import generate
    node = _node(case)
    want = jit_meta[case["name"]]
    if "compile_error" in want:
        with pytest.raises(KernelError) as info:
            compile_kernel(node.body, {p.name: p for p in node.io})
        assert str(info.value) == want["compile_error"]
        return
    k = compile_kernel(node.body, {p.name: p for p in node.io})
    src, params, sites = generate(k, "k")
    assert 'extern "C" __global__' in src and len(params) == 2 * len(node.io) + 7 and sites


def test_generated_kernels_compile_with_nvrtc(jit_meta):
    import ctypes as C

    from paper_1203_4938_b200 import _lib
    from paper_1203_4938_b200.kernel import compile_kernel
    from paper_1203_4938_b200.kernel.codegen import generate
    lib = _lib.load()
    for case in CASES:
        if "compile_error" in jit_meta[case["name"]]:
            continue
        node = _node(case)
        src, _, _ = generate(compile_kernel(node.body, {p.name: p for p in node.io}), "k_" + case["name"])
        h = C.c_void_p()
        log = C.create_string_buffer(8192)
        rc = lib.dpp_jit_compile(src.encode(), ("k_" + case["name"]).encode(), C.byref(h), log, 8192)
        if rc == _lib.DPP_ENOTSUP:
            pytest.skip("NVRTC not available in this container")
        assert rc == 0, (case["name"], _lib.last_error())
        lib.dpp_jit_destroy(h)


def _ulps(a, b):
    ai = a.view(np.int32).astype(np.int64)
    bi = b.view(np.int32).astype(np.int64)
    ai = np.where(ai < 0, -(ai & 0x7FFFFFFF), ai)
    bi = np.where(bi < 0, -(bi & 0x7FFFFFFF), bi)
    return np.abs(ai - bi)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_jit_matches_reference_evaluator(cuda, case, jit_meta, jit_arrays):
    import torch

    from paper_1203_4938_b200.errors import KernelRuntimeError, PlanError
    from paper_1203_4938_b200.jit import jit_node
    from paper_1203_4938_b200.types import DataType
    want = jit_meta[case["name"]]
    node = _node(case)
    if "compile_error" in want:
        with pytest.raises(PlanError, match=want["compile_error"].split(" at ")[0]):
            jit_node(node)
        return
    jn = jit_node(node)
    items = case["items"]
    ins = {p: torch.from_numpy(jit_arrays[f"{case['name']}/in/{p}"]).to(cuda)
           for p, (b, w, d) in case["io"].items() if d == "in"}
    outs = {p: torch.full((items * w,), 7, dtype=getattr(torch, DataType(b, w).dtype.name), device=cuda)
            for p, (b, w, d) in case["io"].items() if d == "out"}
    if "fault" in want:
        with pytest.raises(KernelRuntimeError) as info:
            jn.launch(items, ins, outs, None)
        assert info.value.work_item == want["work_item"]
        assert str(info.value).startswith(want["fault"])
        return
    jn.launch(items, ins, outs, None)
    torch.cuda.synchronize()
    for p, t in outs.items():
        got = t.cpu().numpy()
        ref = jit_arrays[f"{case['name']}/out/{p}"]
        if case.get("exact", True):
            assert np.array_equal(got, ref) or (got.dtype.kind == "f" and np.array_equal(
                got.view(np.int32), ref.view(np.int32))), (p, np.flatnonzero(got != ref)[:5])
        else:
            fin = np.isfinite(ref)
            assert np.array_equal(np.isfinite(got), fin)
            assert _ulps(got[fin], ref[fin]).max() <= 4


def _app_cases():
    meta = json.loads((GOLD / "jit_golden.json").read_text())
    return [dict(name=k, body=v["body"], io={p: tuple(t) for p, t in v["io"].items()}, items=v["items"])
            for k, v in sorted(meta.items()) if v.get("app")]


@pytest.mark.gpu
@pytest.mark.parametrize("case", _app_cases(), ids=lambda c: c["name"])
def test_jit_runs_the_reference_app_nodes_bit_exact(cuda, case, jit_arrays):
    # the reference's own generated bodies (leaf dft2/4/8, ycbcr, chroma box,
    # gradient, vq) compiled by the JIT instead of the hand-written kernels
    import torch

    from paper_1203_4938_b200.jit import JitNode
    from paper_1203_4938_b200.types import DataType
    jn = JitNode(_node(case))
    items = case["items"]
    ins = {p: torch.from_numpy(jit_arrays[f"{case['name']}/in/{p}"]).to(cuda)
           for p, (b, w, d) in case["io"].items() if d == "in"}
    outs = {p: torch.empty(items * w, dtype=getattr(torch, DataType(b, w).dtype.name), device=cuda)
            for p, (b, w, d) in case["io"].items() if d == "out"}
    jn.launch(items, ins, outs, None)
    for p, t in outs.items():
        got, ref = t.cpu().numpy(), jit_arrays[f"{case['name']}/out/{p}"]
        assert got.tobytes() == ref.tobytes(), (p, np.flatnonzero(got != ref)[:5])
