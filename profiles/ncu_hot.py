"""Top SASS lines and opcode share of warp-stall samples from an ncu report."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kfilter:
    cmd += ["-k", f"regex:{kfilter}"]
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
hdr = rows[1]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = [(int(r[iss] or 0), r[ia], r[isrc]) for r in rows[2:] if len(r) > iss and r[iss].isdigit()]
tot = sum(d[0] for d in data) or 1
c = Counter()
for s, _, src in data:
    toks = src.split()
    op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
    c[op.split(".")[0]] += s
print("samples", tot, "| by opcode:", ", ".join(f"{op} {100 * s / tot:.1f}%" for op, s in c.most_common(12)))
for s, a, src in sorted(data, reverse=True)[:int(sys.argv[3]) if len(sys.argv) > 3 else 16]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  {a[-5:]}  {src[:80]}")
