"""GPU tests of the consumer entry points: the periodic wavelet transform Ψ* / Ψ
(pcwd_wavelet_transform) and FISTA-W / FISTA-WP on the decomposed Θ_L (pcwd_fista),
against the oracle (oracle/basis.py, oracle/fista.py) on the same seeded inputs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import basis, fista as OF, operator as op, retention as ret  # noqa: E402
from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from synth import configs as C  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = {"f32": 1e-5, "f64": 1e-12}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_09870_b200 import _build
    _build.build()


def _handle(p, dtype):
    dec = Decomposition(Spec(p.d, p.n, p.J, p.h, p.u, p.v, dtype=dtype, retain=p.retain, tau_rel=p.tau_rel,
                             band_L=p.band_L))
    return dec


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


TRANSFORMS = [(2, 32, 3, 4), (2, 64, 5, 4), (2, 16, 4, 1), (2, 8, 3, 6), (1, 64, 6, 4), (1, 32, 5, 1), (2, 1024, 8, 4)]


@pytest.mark.parametrize("case", TRANSFORMS, ids=[f"d{c[0]}n{c[1]}J{c[2]}M{c[3]}" for c in TRANSFORMS])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_wavelet_transform_matches_oracle(case, dtype):
    d, n, J, M = case
    p = C.micro(n, d, M, J, 1, 1, 50, retain="band", band_L=1)
    rng = np.random.default_rng(7)
    f = rng.standard_normal(p.N)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    dec = _handle(p, dtype)
    c = dec.wavelet_transform(torch.from_numpy(f).to(tdt).cuda())
    ref = basis.forward(f, d, n, J, p.h)
    assert _rel(c.double().cpu().numpy(), ref) <= TOL[dtype]
    back = dec.wavelet_transform(torch.from_numpy(ref).to(tdt).cuda(), inverse=True)
    assert _rel(back.double().cpu().numpy(), basis.inverse(ref, d, n, J, p.h)) <= TOL[dtype]
    assert _rel(back.double().cpu().numpy(), f) <= TOL[dtype] * 10
    dec.close()


def _theta_band_dense(p):
    """Θ_L from the oracle: the dense Θ with the band rule's retained set (others zero)."""
    T = op.theta_dense(p)
    pat = ret.band_pattern_dense(p, p.band_L)
    TL = np.zeros_like(T)
    for mu, cols in pat.items():
        TL[mu, cols] = T[mu, cols]
    return TL


@pytest.mark.parametrize("precond", [False, True])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_fista_matches_oracle(precond, dtype):
    p = C.micro(32, 2, 4, 3, 3, 3, 51, retain="band", band_L=64)
    TL = _theta_band_dense(p)
    rng = np.random.default_rng(9)
    # a sparse-ish true coefficient vector, observed through Θ_L with noise
    z_true = rng.standard_normal(p.N) * (rng.uniform(size=p.N) < 0.2)
    z0 = TL @ z_true + 1e-3 * rng.standard_normal(p.N)
    lev, _, _, _ = basis.index_of(p.d, p.n, p.J)
    w = 2e-3 * (1.0 + lev)                         # weights growing with the scale index (R-F2)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    dec = _handle(p, dtype)
    dec.decompose()
    zg, tau = dec.fista(torch.from_numpy(z0).to(tdt).cuda(), torch.from_numpy(w).to(tdt).cuda(), 40, precond=precond)
    sigma = OF.jacobi_sigma(TL) if precond else None
    tau_ref = OF.step_size(TL, sigma)
    # power iteration vs the exact 2-norm: close, and the step stays below the convergence bound 1 / ‖·‖²
    assert abs(tau / tau_ref - 1.0) < 5e-3 and tau / tau_ref * 0.99 < 1.0
    zr = OF.fista(TL, z0, w, 40, sigma=sigma, tau=tau)
    err40 = _rel(zg.double().cpu().numpy(), zr)
    from conftest import record_parity
    record_parity(f"fista{'wp' if precond else 'w'}_40it", dtype, err40, p.N)
    assert err40 <= (1e-5 if dtype == "f32" else 1e-10)   # measured r02: 0.9e-6 (W) / 2.1e-6 (WP) in fp32
    # a few iterations: rounding has had little time to accumulate
    z5, _ = dec.fista(torch.from_numpy(z0).to(tdt).cuda(), torch.from_numpy(w).to(tdt).cuda(), 5, precond=precond,
                      tau=tau)
    err5 = _rel(z5.double().cpu().numpy(), OF.fista(TL, z0, w, 5, sigma=sigma, tau=tau))
    record_parity(f"fista{'wp' if precond else 'w'}_5it", dtype, err5, p.N)
    assert err5 <= (1e-5 if dtype == "f32" else 1e-12)
    # more iterations decrease the objective towards the minimiser's
    z200, _ = dec.fista(torch.from_numpy(z0).to(tdt).cuda(), torch.from_numpy(w).to(tdt).cuda(), 200,
                        precond=precond, tau=tau)
    assert OF.objective(TL, z0, w, z200.double().cpu().numpy()) <= OF.objective(TL, z0, w, zr) * (1 + 1e-6)
    dec.close()


def test_fista_needs_decompose_and_one_shard():
    p = C.micro(16, 2, 4, 2, 2, 1, 52, retain="band", band_L=16)
    dec = _handle(p, "f32")
    z = torch.zeros(p.N, device="cuda")
    from paper_2005_09870_b200 import PcwdError
    with pytest.raises(PcwdError):
        dec.fista(z, z, 5)
    dec.close()
    d2 = Decomposition(Spec(p.d, p.n, p.J, p.h, p.u, p.v, dtype="f32", retain="band", band_L=16, rank=0, world=2))
    d2.decompose()
    with pytest.raises(PcwdError):
        d2.fista(z, z, 5)
    d2.close()
