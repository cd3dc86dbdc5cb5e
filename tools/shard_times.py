"""Per-shard decomposition time on ONE GPU: the handle of rank r of world W, timed alone (CUDA events,
median of reps).  max_r t_r predicts the W-GPU step time of bench.py (no collective on the band path).
python tools/shard_times.py [config] [W ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from synth import configs as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
worlds = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
p = C.get(name)
u = torch.from_numpy(p.u).cuda()
v = torch.from_numpy(p.v).cuda()
out = {}
for W in worlds:
    ts = []
    for r in range(W):
        dec = Decomposition(Spec(p.d, p.n, p.J, p.h, u, v, dtype="f32", retain=p.retain, tau_rel=p.tau_rel,
                                 band_L=p.band_L, rank=r, world=W))
        for _ in range(2):
            dec.decompose()
        torch.cuda.synchronize()
        times = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dec.decompose()
            b.record()
            b.synchronize()
            times.append(a.elapsed_time(b))
        times.sort()
        info = dec.info()
        ts.append((info.row0, info.row1, round(times[len(times) // 2], 3)))
        dec.close()
    out[W] = {"shards": ts, "max_ms": max(t[2] for t in ts), "sum_ms": round(sum(t[2] for t in ts), 3)}
    print(W, json.dumps(out[W]), flush=True)
