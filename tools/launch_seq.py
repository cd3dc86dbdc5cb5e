"""Print an ncu launch list CSV in launch order: python tools/launch_seq.py gpurun_out/launches_TAG.csv"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
gi = h.index("Grid Size") if "Grid Size" in h else None
tot = 0.0
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) / 1e6
    tot += v
    name = r[ki].replace("void ", "").replace("pcwd::", "").replace("(anonymous namespace)::", "")
    name = re.sub(r"\(const .*", "", name)
    print(f"{v:8.3f} ms  {name[:110]}  {r[gi] if gi is not None else ''}")
print(f"total {tot:.3f} ms")
