"""Shared fixtures.  ``gpu`` marks tests that need a B200 (run with -m gpu)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device; run on the B200 box")


@pytest.fixture(scope="session")
def fft_golden():
    return np.load(GOLDEN / "fft_golden.npz")


@pytest.fixture(scope="session")
def leaf_golden():
    return np.load(GOLDEN / "leaf_golden.npz")


@pytest.fixture(scope="session")
def imgc_golden():
    return np.load(GOLDEN / "imgc_golden.npz")


@pytest.fixture(scope="session")
def docs_golden():
    return np.load(GOLDEN / "docs_golden.npz")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a CUDA device (the native nodes have no CPU fallback)")
    from paper_1203_4938_b200 import _lib
    _lib.load()
    return torch.device("cuda:0")


def table2_doc(rot_body: str = "int i=get_global_id(0);\ny[i]=x[i]*65536.0f;\n",
               adder_body: str = "int i = get_global_id(0);\nz[i]=x[i]+y[i];\n") -> dict:
    """The reference's Table II graph (pkg/tests/conftest.py:18-41), restated."""
    f = lambda d: {"data": d[0], "type": d[1]}  # noqa: E731
    return {
        "kernels": {
            "adder": {"body": adder_body,
                      "io": {"x": f(("float", "InputPoint")), "y": f(("float", "InputPoint")),
                             "z": f(("float", "OutputPoint"))}},
            "fan": {"body": "int i=get_global_id(0);\nx[i]=z[i].x;\ny[i]=z[i].y;\n",
                    "io": {"x": f(("float", "OutputPoint")), "y": f(("float", "OutputPoint")),
                           "z": f(("float2", "InputPoint"))}},
            "rot": {"body": rot_body,
                    "io": {"x": f(("float", "InputPoint")), "y": f(("float", "OutputPoint"))}}},
        "nodes": [[0, {"kernel": "fan"}], [1, {"kernel": "rot"}], [2, {"kernel": "adder"}]],
        "arrows": [{"output": [0, "x"], "input": [2, "x"]},
                   {"output": [1, "y"], "input": [2, "y"]},
                   {"output": [0, "y"], "input": [1, "x"]}],
    }


def complex_signals(seed: int, shape) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64)


def rel_l2(got, ref) -> float:
    got = np.asarray(got, np.complex128)
    ref = np.asarray(ref, np.complex128)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
