"""Decomposition time of every BASELINE config on one GPU (CUDA events, median of 5 after 2 warm-ups; c2 in both
precisions): python tools/configs_bench.py > out.json"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from synth import configs as C  # noqa: E402

rows = []
for name in ("c1", "c2", "c3", "c4", "c5"):
    p = C.get(name)
    for dtype in p.dtypes:
        dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(),
                                 dtype=dtype, retain=p.retain, tau_rel=p.tau_rel, band_L=p.band_L))
        for _ in range(2):
            dec.decompose()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            dec.decompose()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        nnz = dec.info().nnz
        ms = statistics.median(ts)
        rows.append({"config": name, "dtype": dtype, "retain": p.retain, "n": p.n, "d": p.d, "J": p.J, "m": p.m,
                     "nnz": int(nnz), "ms": ms, "entries_per_s": nnz / (ms * 1e-3)})
        dec.close()
        print(json.dumps(rows[-1]), flush=True)
