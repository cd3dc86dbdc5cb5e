"""Decomposition throughput vs torus size (band L = 128, DB4, m = 10, seeded random operator with a 37² filter
support, fp32): python tools/size_sweep.py > out.jsonl"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from synth import configs as C  # noqa: E402

for n, J in ((128, 5), (256, 6), (512, 7), (1024, 8), (2048, 9), (4096, 10)):   # the paper's range
    p = C.micro(n, 2, 4, J, 10, 18, 60 + n, retain="band", band_L=128)
    dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(np.ascontiguousarray(p.u)).cuda(),
                             torch.from_numpy(np.ascontiguousarray(p.v)).cuda(), dtype="f32", retain="band",
                             band_L=128))
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
    ms = statistics.median(ts)
    nnz = dec.info().nnz
    print(json.dumps({"n": n, "J": J, "units": p.N, "nnz": int(nnz), "ms": ms, "entries_per_s": nnz / (ms * 1e-3)}),
          flush=True)
    dec.close()
