"""Link an A/B variant library: one replaced source (any path, extra -D flags)
plus the working tree's other objects -> alt/NAME.so (git-ignored, travels to
the GPU box).  Usage: python profiles/micro/build_variant.py NAME SRC.cu [-DFOO=1 ...]"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_1203_4938_b200 import _build as b  # noqa: E402

name, src, *defs = sys.argv[1:]
b.build()
src = Path(src).resolve()
obj = Path("/tmp") / f"variant_{name}.o"
inc = ["-I", str(b.CSRC)]
subprocess.run([b.nvcc(), *b.ARCH, *b.FLAGS, *inc, *defs, "-c", str(src), "-o", str(obj)], check=True)
objs = [str(o) for o in sorted(b.BUILD.glob("*.o")) if o.stem != src.stem] + [str(obj)]
(ROOT / "alt").mkdir(exist_ok=True)
out = ROOT / "alt" / f"{name}.so"
subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", str(out), *objs, "-lcuda", "-ldl"], check=True)
print(out)
