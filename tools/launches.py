"""Summarise an ncu launch list CSV by kernel: python tools/launches.py gpurun_out/launches_TAG.csv"""
import csv
import re
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = OrderedDict()
tot = 0.0
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) / 1e3
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
    a = agg.setdefault(name, [0.0, 0])
    a[0] += v
    a[1] += 1
    tot += v
for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{t/1e3:9.3f} ms {100*t/tot:5.1f}%  {c:4d} launches  {k}")
print(f"total {tot/1e3:.3f} ms, {sum(c for _, c in agg.values())} launches")
