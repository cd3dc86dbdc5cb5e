import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2005_09870_b200 import Decomposition, Spec
from synth import configs as C
p = C.get("c4")
dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(), dtype="f32", retain=p.retain, tau_rel=p.tau_rel))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    dec.decompose()
torch.cuda.synchronize(); print("ok", dec.info().nnz)
