"""Summarise registers/spills per kernel from `cuobjdump -res-usage` of the built library."""

import re
import subprocess
import sys
from pathlib import Path

lib = Path(__file__).resolve().parents[1] / "paper_1203_4938_b200" / "libdpp_b200.so"
out = subprocess.run(["cuobjdump", "-res-usage", str(lib)], capture_output=True, text=True).stdout
name = None
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for line in out.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        name = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", line)
    if m and name and pat in name:
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dem = re.sub(r"\(.*", "", dem).replace("dpp::", "")
        print(f"{dem:55s} regs={m.group(1):>3} stack={m.group(2)} local={m.group(4)}")
