"""Shared-memory instructions with excessive wavefronts (bank conflicts) from an ncu source page."""
import csv
import subprocess
import sys

rows = list(csv.reader(subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                                       "sass"], capture_output=True, text=True).stdout.splitlines()))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iex, iw = hdr.index("L1 Wavefronts Shared Excessive"), hdr.index("L1 Wavefronts Shared")
out = []
for r in rows[2:]:
    try:
        ex, w = float(r[iex] or 0), float(r[iw] or 0)
    except (ValueError, IndexError):
        continue
    if ex > 0:
        out.append((ex, w, r[ia][-5:], r[isrc][:70]))
tot = sum(o[0] for o in out)
print(f"excessive wavefronts total {tot:.3g}")
for ex, w, a, s in sorted(out, reverse=True)[:12]:
    print(f"{ex:12.4g} of {w:12.4g}  {a}  {s}")
