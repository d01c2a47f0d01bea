"""The C-ABI library loads and exports every symbol include/dpp_b200.h declares (CPU only)."""

from __future__ import annotations

import ctypes
import re

import pytest
from pathlib import Path

from paper_1203_4938_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "dpp_b200.h"


def declared_symbols() -> set[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return set(re.findall(r"\b(dpp_[a-z0-9_]+)\s*\(", text))


def test_header_and_binding_agree():
    assert declared_symbols() == set(_lib.SIGNATURES)


def declared_arity() -> dict[str, int]:
    """Parameter count of every prototype in the header."""
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    out = {}
    for name, params in re.findall(r"\b(dpp_[a-z0-9_]+)\s*\(([^;{]*?)\)\s*;", text, flags=re.S):
        params = params.strip()
        out[name] = 0 if params in ("", "void") else params.count(",") + 1
    return out


def test_binding_arity_matches_the_header():
    """ctypes argtypes have exactly as many entries as the C prototypes
    (a missing or extra argument would shift every pointer after it)."""
    arity = declared_arity()
    assert set(arity) == set(_lib.SIGNATURES)
    for name, (_, argtypes) in _lib.SIGNATURES.items():
        assert len(argtypes) == arity[name], (name, len(argtypes), arity[name])


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr), name
    assert lib.dpp_abi_version() == _lib.ABI_VERSION


def test_error_path_without_a_gpu():
    lib = _lib.load()
    rc = lib.dpp_imgc_encode(None, 2, 8, 8, 16, 128, 1, None, 16, 0, 0.25, None, None, None, None, None,
                             None)
    assert rc == _lib.DPP_EINVAL
    assert "channels" in _lib.last_error()
    assert lib.dpp_fft_leaf(5, None, None, 0, None) == _lib.DPP_EINVAL


def test_plan_shape_query_without_a_gpu():
    """dpp_fft_plan_supported is pure shape rules: it answers on a CPU-only host."""
    lib = _lib.load()
    assert lib.dpp_fft_plan_supported(1, 1 << 16, 1) == 1
    assert lib.dpp_fft_plan_supported(1, 1 << 30, 1) == 1
    assert lib.dpp_fft_plan_supported(1, 3, 1) == 0
    assert lib.dpp_fft_plan_supported(1, 1 << 31, 1) == 0
    assert lib.dpp_fft_plan_supported(2, 16384, 16384) == 1
    assert lib.dpp_fft_plan_supported(2, 32768, 32) == 1
    assert lib.dpp_fft_plan_supported(2, 32768, 8) == 0     # 16-column tiles
    assert lib.dpp_fft_plan_supported(2, 8192, 8) == 1      # 8-column tiles
    assert lib.dpp_fft_plan_supported(2, 128, 256) == 0     # columns < 256 rows: JIT body
    assert lib.dpp_fft_plan_supported(3, 16, 16) == 0
    from paper_1203_4938_b200.nodes import match_fft
    from paper_1203_4938_b200.apps.fft import fft2d_kernel
    assert match_fft(fft2d_kernel(4096, 256)) is not None
    assert match_fft(fft2d_kernel(128, 256)) is None


def _sass_by_function() -> dict[str, list[str]]:
    import subprocess
    out = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    funcs: dict[str, list[str]] = {}
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur and re.match(r"\s+/\*[0-9a-f]{4}\*/", line):
            funcs[cur].append(line)
    return funcs


def test_bit_exact_kernels_contain_no_fused_binary32_multiply_add():
    """The codec and leaf kernels must keep every binary32 product and sum
    separately rounded (the reference evaluates them with numpy, no FMA).
    FFMA2 fusion would silently break the byte-exact bitstream (ptxas fuses
    FMUL2 -> FADD2 even for explicit .rn PTX), so the SASS is checked here.
    The only FFMA allowed is the `FFMA R, RZ, x, y` range probe inside the
    correctly-rounded binary64 division routine."""
    import shutil
    if not shutil.which("cuobjdump"):
        import pytest
        pytest.skip("cuobjdump not available")
    exact = ("encode_kernel", "vqnearest_kernel", "ycbcr_kernel", "boxdown_kernel", "gradient_kernel",
             "leaf_dft_kernel", "decode_kernel", "kpp_update")
    checked = 0
    for name, lines in _sass_by_function().items():
        if not any(k in name for k in exact if k != "kpp_update"):
            continue
        checked += 1
        for ln in lines:
            assert "FFMA2" not in ln, (name, ln)
            if re.search(r"\bFFMA\b", ln):
                assert re.search(r"FFMA R\d+, RZ,", ln), (name, ln)
    assert checked >= 10


def test_library_is_sm100a():
    blob = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in blob


@pytest.mark.gpu
def test_plain_c_consumer(tmp_path):
    """tests/c/abi_smoke.c: the C ABI from a C program (gcc, cudart, the
    in-tree library) — no Python or torch between the caller and the kernels."""
    import subprocess
    root = Path(__file__).resolve().parents[1]
    lib_dir = root / "paper_1203_4938_b200"
    exe = tmp_path / "abi_smoke"
    cuda = Path("/usr/local/cuda")
    subprocess.run(["gcc", "-O1", "-o", str(exe), str(root / "tests" / "c" / "abi_smoke.c"),
                    f"-I{root / 'include'}", f"-I{cuda / 'include'}", f"-L{lib_dir}", "-ldpp_b200",
                    f"-L{cuda / 'lib64'}", "-lcudart", "-lm", f"-Wl,-rpath,{lib_dir}",
                    f"-Wl,-rpath,{cuda / 'lib64'}"], check=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stderr
    assert "abi smoke ok" in res.stdout


def test_header_is_plain_c(tmp_path):
    """The header and the C consumer compile as C11 (no C++ or torch types)."""
    import subprocess
    root = Path(__file__).resolve().parents[1]
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-c", "-o", str(tmp_path / "abi_smoke.o"),
                    str(root / "tests" / "c" / "abi_smoke.c"), f"-I{root / 'include'}",
                    "-I/usr/local/cuda/include"], check=True)
