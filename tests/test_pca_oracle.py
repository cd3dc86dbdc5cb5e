"""Pins of the PC-expansion oracle (oracle/pca.py, §3.3) that do not come from the oracle itself: the
identity operator's SVIR has rank 1, a shift-invariant convolution gives one exact term, an exact rank-r
family is recovered exactly, and the interpolation reproduces the samples at the cell centres and averages halfway."""
import numpy as np

from oracle import pca as PC


def test_identity_operator_has_rank_one_svir():
    """"the identity operator ... has an SVIR of rank 1": every response is δ_0."""
    n, R = 16, 2
    W = (2 * R + 1) ** 2
    svir = np.zeros((n * n, W))
    svir[:, W // 2] = 1.0
    u, v, sig = PC.pc_from_svir(svir, 2, n, R, 1)
    e = np.zeros(n * n)
    e[0] = 1.0
    assert np.max(np.abs(u[0] - e)) < 1e-14 and np.max(np.abs(v[0] - 1.0)) < 1e-13
    assert abs(sig[0] - n) < 1e-12                                   # sqrt(N) for N unit rows


def test_shift_invariant_convolution_is_one_term():
    n, R, g = 32, 3, 4
    rng = np.random.default_rng(0)
    kappa = rng.uniform(0.1, 1.0, size=(2 * R + 1) ** 2)
    irs = np.tile(kappa, (g * g, 1))
    u, v, sig = PC.pc_from_samples(irs, 2, n, R, g, 1)
    nk = np.linalg.norm(kappa)
    assert abs(sig[0] - g * nk) < 1e-12 * g * nk
    assert np.max(np.abs(v[0] - nk)) < 1e-12 * nk                   # constant coefficient map ‖κ‖
    assert abs(u[0].sum() - kappa.sum() / nk) < 1e-12               # u = κ/‖κ‖ (positive entries)


def test_exact_rank_r_family_recovered():
    """Responses Σ_j a_j(y) K_j with orthonormal K_j: σ_{r+1..} = 0 and span(u_1..u_r) = span(K_j)."""
    n, R, r = 16, 2, 3
    W = (2 * R + 1) ** 2
    rng = np.random.default_rng(1)
    K, _ = np.linalg.qr(rng.standard_normal((W, r)))
    a = rng.standard_normal((n * n, r)) * np.array([3.0, 1.0, 0.2])
    svir = a @ K.T
    u, v, sig = PC.pc_from_svir(svir, 2, n, R, r + 1)
    assert sig[r] < 1e-12 * sig[0]
    U = PC.leading_components(svir, r)[0]
    assert np.linalg.norm(K - U @ (U.T @ K)) < 1e-12
    recon = np.zeros_like(svir)
    for k in range(r):
        recon += np.outer(v[k], U[:, k])
    assert np.max(np.abs(recon - svir)) < 1e-12 * np.max(np.abs(svir))


def test_bilinear_reproduces_samples_and_midpoints():
    n, g = 32, 4                                       # centres at 4, 12, 20, 28
    rng = np.random.default_rng(2)
    c = rng.standard_normal((g * g, 2))
    v = PC.bilinear(c, 2, n, g)
    for i0 in range(g):
        for i1 in range(g):
            y = (8 * i0 + 4) * n + (8 * i1 + 4)
            assert np.allclose(v[:, y], c[i0 * g + i1], rtol=0, atol=1e-15)
    y = (4) * n + 8                                    # halfway between centres (4,4) and (4,12)
    assert np.allclose(v[:, y], 0.5 * (c[0] + c[1]), atol=1e-15)
    y = (0) * n + 0                                    # wraps: halfway between (28,28),(28,4),(4,28),(4,4)
    assert np.allclose(v[:, y], 0.25 * (c[15] + c[12] + c[3] + c[0]), atol=1e-15)
