"""d = 3 variant (pcwd_rows3d) timed on one GPU: rows/s and the correlation's fp64 FMA rate at 32³ and 64³
(CUDA events around the synchronous call, median of 5 after 2 warm-ups).  python tools/volume_bench.py > out.jsonl"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2005_09870_b200 import pcwd  # noqa: E402
from synth.filters import daubechies  # noqa: E402
from synth.volume import volume_problem  # noqa: E402

for n, J, M, m, R, count in ((32, 3, 4, 4, 2, 1184), (32, 3, 4, 4, 2, 18944), (64, 4, 4, 4, 2, 592), (64, 4, 4, 4, 2, 4736)):
    h = daubechies(M)
    u, v = volume_problem(n, m, R, 7)
    ud, vd = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
    units = np.random.default_rng(1).integers(0, n ** 3, count)
    ts = []
    for it in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = pcwd.rows3d(n, J, h, ud, vd, units)
        b.record()
        b.synchronize()
        if it >= 2:
            ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    N = n ** 3
    fma_corr = count * N * m * (2 * R + 1) ** 3                      # step 2, the dominant term
    fma_casc = count * 2 * sum(3 * (n >> (l - 1)) ** 3 * len(h) for l in range(1, J + 1))   # steps 1 and 3 (≤, parity-masked)
    print(json.dumps({"n": n, "J": J, "taps": len(h), "m": m, "R": R, "units": count, "ms": ms,
                      "rows_per_s": count / ms * 1e3, "entries_per_s": count * N / ms * 1e3,
                      "dense_equiv_fp64_tflops": 2 * (fma_corr + fma_casc) / ms * 1e-9,   # before the zero-line skip of step 2
                      "out_GBps": count * N * 8 / ms * 1e-6}), flush=True)
