"""Per-kernel durations of one decomposition with the launches serialised (pcwd_profile(h, 2)): each unit-kernel
launch timed alone with CUDA events, plus the step time of the normal (overlapped) schedule.
Usage: python tools/launch_profile.py CONFIG [DTYPE]  -> one JSON line"""
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from paper_2005_09870_b200 import pcwd as P  # noqa: E402
from synth import configs as C  # noqa: E402

name = sys.argv[1]
dtype = sys.argv[2] if len(sys.argv) > 2 else "f32"
if name.startswith("n"):   # the size sweep's operators: n<side> (tools/size_sweep.py)
    import numpy as np
    side = int(name[1:])
    p = C.micro(side, 2, 4, side.bit_length() - 3, 10, 18, 60 + side, retain="band", band_L=128)
    p.u, p.v = np.ascontiguousarray(p.u), np.ascontiguousarray(p.v)
else:
    p = C.get(name)
dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(), dtype=dtype,
                         retain=p.retain, tau_rel=p.tau_rel, band_L=p.band_L))


def step_ms(k=5):
    ts = []
    for _ in range(k):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        dec.decompose()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


dec.decompose()
overlapped = step_ms()
P._check(P.lib().pcwd_profile(dec._h, 2), "profile")
dec.decompose()
serial = step_ms()
torch.cuda.synchronize()
lp = dec.launch_profile()
print(json.dumps({"config": name, "dtype": dtype, "step_ms": overlapped, "step_ms_serialised": serial,
                  "launches": [{"kind": k, "level": lv, "ms": round(ms, 4), "fma": f,
                                "tflops": round(2 * f / (ms * 1e-3) / 1e12, 2) if ms > 0 else None}
                               for (ms, f, k, lv) in lp]}))
