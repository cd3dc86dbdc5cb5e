"""GPU Algorithm 1 (pcwd_approx, the η-approximation Θ̃ = Σ_k Ã_k B_k) against the literal dense
oracle (oracle/approx.py): the truncation index S_k of every term (an integer, exactly), the Schur bounds, the
support of Θ̃ (its nonzeros, bit-exact) and its values (fp64 bar); plus the accuracy lemma ‖Θ − Θ̃‖₂ ≤ η
 measured on the GPU by power iteration with Θ applied through the operator (Ψ* H Ψ)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import approx as AP, basis  # noqa: E402
from paper_2005_09870_b200 import Decomposition, PcwdError, Spec  # noqa: E402
from synth import configs as C  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_09870_b200 import _build
    _build.build()


def _smooth_micro(n, d, M, J, m, seed):
    """Gaussian-like u_k (taps jittered so that no symmetry makes entries cancel exactly) and smooth positive v_k
    (the shape of the paper's blurs) on a small torus."""
    p = C.micro(n, d, M, J, m, 2, seed)
    rng = np.random.default_rng(seed)
    r = np.arange(-2, 3)
    if d == 2:
        g = np.exp(-(r[:, None] ** 2 + r[None, :] ** 2) / 2.0)
        u = np.zeros((m, n, n))
        for k in range(m):
            w = g ** (1 + k) * (1 + 0.5 * rng.uniform(size=g.shape))
            w /= w.sum()
            for i, a in enumerate(r):
                for j, b in enumerate(r):
                    u[k, a % n, b % n] = w[i, j]
        y = np.arange(n) / n
        v = np.stack([1.0 + 0.3 * (k + 1) * np.cos(2 * np.pi * (y[:, None] + 2 * k * y[None, :])) for k in range(m)])
    else:
        g = np.exp(-(r ** 2) / 2.0)
        u = np.zeros((m, n))
        for k in range(m):
            w = g ** (1 + k) * (1 + 0.5 * rng.uniform(size=g.shape))
            u[k, r % n] = w / w.sum()
        y = np.arange(n) / n
        v = np.stack([1.0 + 0.3 * (k + 1) * np.cos(2 * np.pi * (k + 1) * y) for k in range(m)])
    p.u = u.reshape(m, -1)
    p.v = v.reshape(m, -1)
    return p


CASES = [  # (n, d, M, J, m, seed, eta values)
    (16, 2, 2, 3, 3, 1, (10.0, 1.0, 1e-2, 1e-300)),
    (32, 2, 2, 4, 2, 2, (3.0, 0.5, 1e-3)),
    (64, 1, 4, 5, 3, 3, (2.0, 0.3, 1e-4)),
    (32, 2, 1, 5, 2, 4, (1.0, 0.1)),          # Haar, full depth
]


@pytest.mark.parametrize("rule", ["index", "magnitude"])
@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}d{c[1]}M{c[2]}J{c[3]}" for c in CASES])
def test_approx_matches_dense_algorithm1(case, rule):
    n, d, M, J, m, seed, etas = case
    p = _smooth_micro(n, d, M, J, m, seed)
    W = basis.analysis_matrix(p.d, p.n, p.J, p.h)
    dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(),
                             dtype="f64", retain="full"))
    for eta in etas:
        T_ref, info_ref, sup = AP.theta_tilde(p, eta, W, rule)
        got = dec.approx(eta, rule)
        assert got["S"] == [i["S"] for i in info_ref], (eta, got["S"], [i["S"] for i in info_ref])
        for b, i in zip(got["bound"], info_ref):
            assert abs(b - i["bound"]) <= 1e-10 * max(i["bound"], 1e-300)
        rp, col, val = (t.numpy() for t in dec.csr(device="cpu"))
        assert got["nnz"] == np.count_nonzero(sup) == len(col)
        dense = np.zeros((p.N, p.N))
        for r in range(p.N):
            assert np.array_equal(col[rp[r]:rp[r + 1]], np.nonzero(sup[r])[0]), (eta, r)
            dense[r, col[rp[r]:rp[r + 1]]] = val[rp[r]:rp[r + 1]]
        if np.any(T_ref):
            assert np.linalg.norm(dense - T_ref) <= 1e-12 * np.linalg.norm(T_ref), eta
    dec.close()


def _spectral_error(dec, N, iters=60, seed=0):
    """‖Θ − Θ̃‖₂ by power iteration on (Θ − Θ̃)ᵀ(Θ − Θ̃): Θx = Ψ*HΨx and Θᵀy = Ψ*H*Ψy through the library's
    transforms and operator, Θ̃ x / Θ̃ᵀ y through pcwd_apply."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(N, dtype=torch.float64, device="cuda", generator=g)
    x /= x.norm()
    lam = 0.0
    for _ in range(iters):
        th = dec.wavelet_transform(dec.operator_apply(dec.wavelet_transform(x, inverse=True)))
        r = th - dec.apply(x)
        tht = dec.wavelet_transform(dec.operator_apply(dec.wavelet_transform(r, inverse=True), adjoint=True))
        z = tht - dec.apply(r, transpose=True)
        lam = float(z.norm())
        if lam == 0.0:
            return 0.0
        x = z / lam
    return lam ** 0.5


def test_operator_apply_matches_oracle():
    from oracle import operator as op
    p = C.micro(16, 2, 4, 3, 3, 2, 11)
    dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(),
                             dtype="f64", retain="full"))
    f = np.random.default_rng(1).standard_normal(p.N)
    y = dec.operator_apply(torch.from_numpy(f).cuda()).cpu().numpy()
    ya = dec.operator_apply(torch.from_numpy(f).cuda(), adjoint=True).cpu().numpy()
    assert np.max(np.abs(y - op.apply_fft(p, f))) <= 1e-12 * np.max(np.abs(y))
    assert np.max(np.abs(ya - op.adjoint_apply_fft(p, f))) <= 1e-12 * np.max(np.abs(ya))
    dec.close()


def _blur128():
    """A 128² space-varying blur (N = 16,384, DB4, J = 5, m = 4, 9 × 9 taps) in the shape of the paper's operators."""
    p = C.micro(128, 2, 4, 5, 4, 4, 91)
    rng = np.random.default_rng(91)
    r = np.arange(-4, 5)
    g = np.exp(-(r[:, None] ** 2 + r[None, :] ** 2) / 4.0)
    u = np.zeros((4, 128, 128))
    for k in range(4):
        w = g ** (1 + k) * (1 + 0.5 * rng.uniform(size=g.shape))
        w /= w.sum()
        for i, a in enumerate(r):
            for j, b in enumerate(r):
                u[k, a % 128, b % 128] = w[i, j]
    y = np.arange(128) / 128
    p.u = u.reshape(4, -1)
    p.v = np.stack([1.0 + 0.3 * (k + 1) * np.cos(2 * np.pi * (y[:, None] + k * y[None, :])) for k in range(4)]).reshape(4, -1)
    return p


@pytest.mark.parametrize("rule", ["index", "magnitude"])
@pytest.mark.parametrize("eta", [3.0, 0.3, 0.03])
def test_accuracy_lemma_128(eta, rule):
    """‖Θ − Θ̃‖₂ ≤ η measured on the GPU by power iteration (128², fp64)."""
    p = _blur128()
    dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(),
                             dtype="f64", retain="band", band_L=64))
    try:
        info = dec.approx(eta, rule)
        err = _spectral_error(dec, p.N)
        assert err <= eta, (eta, err, info["S"])
    finally:
        dec.close()


def test_approx_argument_checks():
    p = C.micro(16, 2, 2, 3, 2, 2, 12)
    dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(),
                             dtype="f32", retain="full"))
    with pytest.raises(PcwdError) as e:
        dec.approx(1.0)
    assert e.value.code == 7
    dec.close()
    dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(),
                             dtype="f64", retain="full"))
    with pytest.raises(PcwdError) as e:
        dec.approx(0.0)
    assert e.value.code == 3
    with pytest.raises(KeyError):
        dec.approx(1.0, "other")
    dec.close()
