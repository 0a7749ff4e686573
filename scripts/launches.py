"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: median per kernel+grid."""
import collections
import csv
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
mi = hdr.index("Metric Name") if "Metric Name" in hdr else None
d = collections.OrderedDict()
for r in rows[1:]:
    if len(r) > vi and "trail" in r[ki] and (mi is None or r[mi] == "gpu__time_duration.sum"):
        d.setdefault((r[ki].split("(")[0][:60], r[gi]), []).append(float(r[vi].replace(",", "")))
for (k, g), v in d.items():
    v.sort()
    print(f"{len(v):4d} {v[len(v) // 2] / 1e3:8.2f} us  {g:>14}  {k}")
