"""Summarise an ncu --metrics gpu__time_duration.sum CSV: time share per kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
d = defaultdict(list)
for r in rows[h + 1:]:
    if len(r) > iv and r[im] == "gpu__time_duration.sum":
        d[r[ik].split("(")[0][:70]].append(float(r[iv].replace(",", "")))
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{k:70s} n={len(v):4d} total={sum(v) / 1e6:9.3f} ms avg={sum(v) / len(v) / 1e3:9.1f} us share={100 * sum(v) / tot:5.1f}%")
