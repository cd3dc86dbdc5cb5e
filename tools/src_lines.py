"""Per-source-line instruction and stall shares from `ncu -i X --page source --csv --print-source cuda,sass`.
python tools/src_lines.py file.csv [file_filter] [top]"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
filt = sys.argv[2] if len(sys.argv) > 2 else "fine.cu"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur = None
agg = {}
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not cur or filt not in cur or len(r) < len(hdr):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    ii = hdr.index("Instructions Executed")
    wi = hdr.index("Warp Stall Sampling (All Samples)")
    a = agg.setdefault(ln, [0.0, 0.0, r[1][:90]])
    num = lambda x: float(x) if re.match(r"^[0-9.eE+-]+$", x or "") and x not in ("-", "+") else 0.0
    a[0] += num(r[ii])
    a[1] += num(r[wi])
ti = sum(v[0] for v in agg.values()) or 1
tw = sum(v[1] for v in agg.values()) or 1
print(f"total instructions {ti:.4g}, stall samples {tw:.4g}")
for ln, (i, w, s) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"L{ln:5d} inst {100 * i / ti:5.1f}%  stall {100 * w / tw:5.1f}%  {s.strip()}")
