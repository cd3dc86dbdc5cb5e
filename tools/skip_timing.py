import sys, os, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_2005_09870_b200 import Decomposition, Spec
from synth import configs as C
p = C.get(sys.argv[1] if len(sys.argv) > 1 else "c4")
dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(), dtype="f32",
                         retain=p.retain, tau_rel=p.tau_rel, band_L=p.band_L))
for _ in range(2): dec.decompose()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record(); dec.decompose(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(os.environ.get("PCWD_SKIP_LEVELS", "0"), round(statistics.median(ts), 2))
