"""η sweep of Algorithm 1 on the GPU at N = 256² (the setting of the paper's Fig. 3): for each η,
pcwd_approx's time (CUDA events around the call, which synchronises), the nonzeros of Θ̃, the truncation index S_k of
every term and the measured ‖Θ − Θ̃‖₂ (power iteration, Θ applied as Ψ* H Ψ through the library's transforms and
operator).  Operator: config 3's inputs (256², DB4, J = 6, m = 8) in fp64.
Usage: python tools/approx_sweep.py [eta ...]  -> JSON lines"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from synth import configs as C  # noqa: E402


def spectral_error(dec, N, iters=40):
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(N, dtype=torch.float64, device="cuda", generator=g)
    x /= x.norm()
    lam = 0.0
    for _ in range(iters):
        r = dec.wavelet_transform(dec.operator_apply(dec.wavelet_transform(x, inverse=True))) - dec.apply(x)
        z = dec.wavelet_transform(dec.operator_apply(dec.wavelet_transform(r, inverse=True), adjoint=True)) \
            - dec.apply(r, transpose=True)
        lam = float(z.norm())
        if lam == 0.0:
            return 0.0
        x = z / lam
    return lam ** 0.5


rules = [a for a in sys.argv[1:] if a in ("index", "magnitude")] or ["magnitude", "index"]
etas = [float(a) for a in sys.argv[1:] if a not in ("index", "magnitude")] or [30.0, 10.0, 3.0, 1.0, 0.3]
p = C.get("c3")
dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(), dtype="f64",
                         retain="band", band_L=64))
dec.approx(etas[0])   # warm-up
for rule, eta in [(r, e) for r in rules for e in etas]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    info = dec.approx(eta, rule)
    t = time.perf_counter() - t0
    err = spectral_error(dec, p.N) if info["nnz"] <= 1.2e9 else None   # Θ̃ᵀ too large for the power iteration
    print(json.dumps({"config": "c3 operator (256^2, DB4, J=6, m=8), fp64", "rule": rule, "eta": eta, "seconds": t,
                      "nnz": info["nnz"], "nnz_per_row": info["nnz"] / p.N, "S": info["S"],
                      "schur_bound": info["bound"], "spectral_error": err, "error_le_eta": None if err is None else err <= eta}), flush=True)
dec.close()
