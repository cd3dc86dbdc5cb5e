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


def _fista_problem(dtype):
    p = C.micro(32, 2, 4, 3, 3, 3, 51, retain="band", band_L=64)
    TL = _theta_band_dense(p)
    rng = np.random.default_rng(9)
    z_true = rng.standard_normal(p.N) * (rng.uniform(size=p.N) < 0.2)
    z0 = TL @ z_true + 1e-3 * rng.standard_normal(p.N)
    lev, _, _, _ = basis.index_of(p.d, p.n, p.J)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    return p, TL, torch.from_numpy(z0).to(tdt).cuda(), torch.from_numpy(2e-3 * (1.0 + lev)).to(tdt).cuda()


@pytest.mark.parametrize("precond", [False, True])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_fista_sharded_world1_is_fista(precond, dtype):
    """pcwd_fista_sharded on the whole Θ with a one-rank reduce (nothing to add) = pcwd_fista, bit for bit."""
    p, _, z0, w = _fista_problem(dtype)
    dec = _handle(p, dtype)
    dec.decompose()
    za, ta = dec.fista(z0, w, 25, precond=precond)
    calls = []
    zb, tb = dec.fista_sharded(z0, w, 25, lambda which, buf: calls.append(which), precond=precond)
    assert ta == tb and torch.equal(za, zb)
    assert calls.count(0) >= 25 + 8 and calls.count(1) == (1 if precond else 0)
    dec.close()


@pytest.mark.parametrize("precond", [False, True])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_fista_two_shards_match_whole(precond, dtype):
    """Θ_L split over two handles (rank 0 / 1 of world 2), each running pcwd_fista_sharded in its own thread and
    stream; the reduce sums the two partial gradients (a two-party all-reduce on the host threads).  The iterates
    equal the one-handle FISTA up to the summation order of Θᵀr, and both ranks return the same z and τ."""
    import threading
    p, TL, z0, w = _fista_problem(dtype)
    whole = _handle(p, dtype)
    whole.decompose()
    zr, tr = whole.fista(z0, w, 40, precond=precond)
    whole.close()
    decs = [Decomposition(Spec(p.d, p.n, p.J, p.h, p.u, p.v, dtype=dtype, retain="band", band_L=p.band_L, rank=r,
                               world=2)) for r in range(2)]
    for d in decs:
        d.decompose()
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    bar = threading.Barrier(2, timeout=120)   # a failing rank breaks the barrier instead of hanging the test
    bufs = [None, None]
    out = [None, None]

    def reduce_for(r):
        def reduce(_which, buf):
            streams[r].synchronize()
            bufs[r] = buf
            bar.wait()
            if r == 0:
                s = bufs[0] + bufs[1]
                bufs[0].copy_(s)
                bufs[1].copy_(s)
                torch.cuda.synchronize()
            bar.wait()
        return reduce

    def run(r):
        with torch.cuda.stream(streams[r]):
            out[r] = decs[r].fista_sharded(z0, w, 40, reduce_for(r), precond=precond,
                                           stream=streams[r].cuda_stream)
        streams[r].synchronize()

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert out[0] is not None and out[1] is not None
    (z_a, t_a), (z_b, t_b) = out
    assert t_a == t_b and torch.equal(z_a, z_b)
    assert abs(t_a / tr - 1.0) < (1e-5 if dtype == "f32" else 1e-10)
    err = _rel(z_a.double().cpu().numpy(), zr.double().cpu().numpy())
    from conftest import record_parity
    record_parity(f"fista{'wp' if precond else 'w'}_2shards_vs_whole", dtype, err, p.N)
    assert err <= (1e-5 if dtype == "f32" else 1e-10)
    # and against the oracle's FISTA at the same step
    sigma = OF.jacobi_sigma(TL) if precond else None
    ref = OF.fista(TL, z0.double().cpu().numpy(), w.double().cpu().numpy(), 40, sigma=sigma, tau=t_a)
    assert _rel(z_a.double().cpu().numpy(), ref) <= (1e-5 if dtype == "f32" else 1e-10)
    for d in decs:
        d.close()


def test_fista_distributed_nccl_world1(tmp_path):
    """fista_distributed through a real NCCL process group (world 1, one process): same z as pcwd_fista."""
    import os
    import subprocess
    import sys
    code = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from paper_2005_09870_b200 import Decomposition, Spec, pcwd as PW
from synth import configs as C
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
p = C.micro(32, 2, 4, 3, 3, 3, 51, retain="band", band_L=64)
dec = Decomposition(Spec(p.d, p.n, p.J, p.h, p.u, p.v, dtype="f64", retain="band", band_L=64))
dec.decompose()
rng = np.random.default_rng(3)
z0 = torch.from_numpy(rng.standard_normal(p.N)).cuda()
w = torch.full((p.N,), 1e-3, dtype=torch.float64, device="cuda")
za, ta = dec.fista(z0, w, 20, precond=True)
zb, tb = PW.fista_distributed(dec, z0, w, 20, precond=True)
torch.cuda.synchronize()
assert ta == tb and torch.equal(za, zb), (ta, tb)
dist.destroy_process_group()
print("NCCL-FISTA-OK")
'''
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29500 + os.getpid() % 1000))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert "NCCL-FISTA-OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
