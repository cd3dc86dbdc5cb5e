"""Time the parts of the end-to-end call sequence (create with host inputs, decompose, CSR D2H)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from paper_2005_09870_b200 import pcwd as P  # noqa: E402
from synth import configs as C  # noqa: E402

p = C.get(sys.argv[1] if len(sys.argv) > 1 else "c5")
u_h = torch.from_numpy(p.u).pin_memory()
v_h = torch.from_numpy(p.v).pin_memory()
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = Decomposition(Spec(p.d, p.n, p.J, p.h, u_h.numpy(), v_h.numpy(), dtype="f32", retain=p.retain,
                           tau_rel=p.tau_rel, band_L=p.band_L))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    d.decompose()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    meta = d.csr_meta()
    if it == 0:
        rp = torch.empty(meta.n_rows + 1, dtype=torch.int64).pin_memory()
        col = torch.empty(meta.nnz, dtype=torch.int32).pin_memory()
        val = torch.empty(meta.nnz, dtype=torch.float32).pin_memory()
    P._check(P.lib().pcwd_copy_csr(d._h, rp.data_ptr(), col.data_ptr(), val.data_ptr(), ctypes.c_void_p(0)), "copy")
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    d.close()
    print(f"create {1e3*(t1-t0):.1f} ms  decompose {1e3*(t2-t1):.1f} ms  d2h {1e3*(t3-t2):.1f} ms "
          f"({(rp.numel()*8+col.numel()*4+val.numel()*4)/(t3-t2)/1e9:.1f} GB/s)", flush=True)
