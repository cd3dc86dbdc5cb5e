"""Print the unit-kernel launches (kind, level) a config uses: python tools/kinds.py c3 [f32]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from synth import configs as C  # noqa: E402

name = sys.argv[1]
dtype = sys.argv[2] if len(sys.argv) > 2 else "f32"
p = C.get(name) if name.startswith("c") else C.micro(*eval(name))
dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(np.ascontiguousarray(p.u)).cuda(),
                         torch.from_numpy(np.ascontiguousarray(p.v)).cuda(), dtype=dtype, retain=p.retain,
                         tau_rel=p.tau_rel, band_L=p.band_L))
dec.decompose()   # warm-up (module load, smem attributes, TMA descriptors)
dec.profile(True)
dec.decompose()
torch.cuda.synchronize()
for ms, fma, kind, lev in dec.launch_profile():
    print(f"{kind:8s} level {lev}  {ms:8.3f} ms  {2 * fma / (ms * 1e-3) / 1e12:6.2f} TFLOP/s")
