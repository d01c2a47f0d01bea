"""Build libdpp_b200.so from the csrc/ of a git ref into alt/<name>.so (A/B timing).

    python profiles/micro/build_ref.py HEAD alt/head.so
    DPP_LIB_PATH=alt/head.so python profiles/micro/time_fft.py
"""
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_1203_4938_b200 import _build  # noqa: E402

ref, out = sys.argv[1], ROOT / sys.argv[2]
with tempfile.TemporaryDirectory() as d:
    d = Path(d)
    tar = subprocess.run(["git", "-C", str(ROOT), "archive", ref, "paper_1203_4938_b200/csrc", "include"],
                         capture_output=True, check=True).stdout
    subprocess.run(["tar", "-x", "-C", str(d)], input=tar, check=True)
    srcs = sorted((d / "paper_1203_4938_b200/csrc").glob("*.cu"))
    flags = [f if f != str(ROOT / "include") else str(d / "include") for f in _build.FLAGS]
    procs = [subprocess.Popen([_build.nvcc(), *_build.ARCH, *flags, "-c", str(s), "-o", str(s.with_suffix(".o"))])
             for s in srcs]
    assert all(p.wait() == 0 for p in procs)
    out.parent.mkdir(parents=True, exist_ok=True)
    subprocess.run([_build.nvcc(), *_build.ARCH, "-shared", "-o", str(out), *[str(s.with_suffix(".o")) for s in srcs],
                    "-lcuda", "-ldl"], check=True)
print(out)
