for kb in ${KBS:-72 48 100}; do echo "== $kb"; PCWD_GENERIC_SMEM_KB=$kb timeout 300 python - <<'PY'
import sys, torch, statistics
sys.path.insert(0, '.')
from paper_2005_09870_b200 import Decomposition, Spec
from synth import configs as C
p = C.get("c4")
dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(), dtype="f32", retain=p.retain, tau_rel=p.tau_rel))
dec.decompose(); dec.decompose()
ts=[]
for _ in range(3):
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record(); dec.decompose(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
print("c4 ms", statistics.median(ts))
PY
done
