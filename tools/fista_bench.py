"""FISTA-W / FISTA-WP in the wavelet domain at c5 scale (N = 1024², Θ_L with L = 128 per row, fp32 and fp64),
the paper's deblurring use of the decomposition (its GPU timing, P:1092/P:1105:
FISTA-WP 0.087 s for 38 iterations, GTX Titan X, fp64 — context, a different Θ_L).  Prints one JSON line:
python tools/fista_bench.py [iters]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from synth import configs as C  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 38
p = C.get("c5")
out = {"workload": "c5 operator (1024², DB4, J=8, m=10), Θ_L band L=128, synthetic image", "iters": iters}
for dtype in ("f32", "f64"):
    tdt = torch.float32 if dtype == "f32" else torch.float64
    dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(),
                             dtype=dtype, retain=p.retain, band_L=p.band_L))
    dec.decompose()
    # synthetic piecewise-smooth image f (seeded), observed through Θ_L in the wavelet domain with noise
    rng = np.random.default_rng(0)
    yy, xx = np.mgrid[0:p.n, 0:p.n] / p.n
    f = (np.sin(6 * xx) * np.cos(4 * yy) + (((xx - 0.5) ** 2 + (yy - 0.4) ** 2) < 0.05)).ravel()
    zf = dec.wavelet_transform(torch.from_numpy(f).to(tdt).cuda())
    z0 = dec.apply(zf) + torch.from_numpy(1e-3 * rng.standard_normal(p.N)).to(tdt).cuda()
    lev = np.concatenate([np.full((p.n >> l) ** 2 * (3 if k else 1), l) for l, k in
                          [(p.J, 0)] + [(l, 1) for l in range(p.J, 0, -1)]])
    w = torch.from_numpy(2e-3 * (1.0 + lev)).to(tdt).cuda()
    res = {}
    for name, pre in (("fista_w", False), ("fista_wp", True)):
        _, tau = dec.fista(z0, w, 1, precond=pre)   # warm-up, τ by power iteration
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        ev[0].record()
        _, tau2 = dec.fista(z0, w, 1, precond=pre)   # the power iteration alone (1 iteration after it)
        ev[1].record()
        ev[2].record()
        z, _ = dec.fista(z0, w, iters, precond=pre, tau=tau)
        ev[3].record()
        torch.cuda.synchronize()
        rec = dec.wavelet_transform(z, inverse=True)
        err = float(torch.linalg.norm(rec.double().cpu() - torch.from_numpy(f)) / np.linalg.norm(f))
        res[name] = {"iters_s": ev[2].elapsed_time(ev[3]) * 1e-3, "ms_per_iter": ev[2].elapsed_time(ev[3]) / iters,
                     "power_iteration_s": ev[0].elapsed_time(ev[1]) * 1e-3, "tau": tau,
                     "rel_image_error": err}
    out[dtype] = res
    dec.close()
print(json.dumps(out))
