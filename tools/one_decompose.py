"""Run config decompositions (for ncu launch lists / captures): python tools/one_decompose.py c5 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from synth import configs as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dtype = sys.argv[3] if len(sys.argv) > 3 else "f32"
p = C.get(name)
dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(), dtype=dtype,
                         retain=p.retain, tau_rel=p.tau_rel, band_L=p.band_L))
for _ in range(reps):
    dec.decompose()
torch.cuda.synchronize()
print("ok", dec.info().nnz)
