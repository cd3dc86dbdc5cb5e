"""Pins of the d = 3 oracle (oracle/volume.py) against what the paper and the mathematics fix:
the tensor-product identity against the pinned 1-D transform, orthogonality, the dense brute-force Θ = W K Wᵀ on 4³
built from the definition of ⋆ by loops, H = identity and H = a shift."""
import numpy as np
import pytest

from oracle import basis, volume
from synth.filters import daubechies, haar
from synth.volume import volume_problem


def _coeffs_1d(x, n, lev, h):
    """Level-`lev` approximation and detail of a line, from the pinned 1-D cascade of depth `lev`."""
    c = basis.forward(x, 1, n, lev, h)
    nl = n >> lev
    return c[:nl], c[nl:2 * nl]          # coarse block, then the level-`lev` details (Λ layout, d = 1)


@pytest.mark.parametrize("M,n,J", [(1, 8, 3), (2, 8, 2), (3, 16, 3), (2, 4, 2)])
def test_tensor_product_identity(M, n, J):
    """(a ⊗ b ⊗ c) has sub-band (ℓ, e) = c_a^{ℓ,e0} ⊗ c_b^{ℓ,e1} ⊗ c_c^{ℓ,e2}: a wrong axis order, a
    swapped orientation code or a wrong sub-band offset fails (a, b, c are distinct random lines)."""
    h = haar() if M == 1 else daubechies(M)
    rng = np.random.default_rng(5)
    a, b, c = rng.standard_normal((3, n))
    f = np.einsum("i,j,k->ijk", a, b, c)
    got = volume.forward3(f, n, J, h)
    for (lev, e, off, nl) in volume.subbands3(n, J):
        e0, e1, e2 = (e >> 2) & 1, (e >> 1) & 1, e & 1
        ca, cb, cc = (_coeffs_1d(x, n, lev, h)[bit] for x, bit in ((a, e0), (b, e1), (c, e2)))
        want = np.einsum("i,j,k->ijk", ca, cb, cc).ravel()
        assert np.allclose(got[off:off + nl ** 3], want, atol=1e-12), (lev, e)


@pytest.mark.parametrize("M,n,J", [(2, 8, 3), (3, 8, 2)])
def test_orthogonal(M, n, J):
    h = daubechies(M)
    x = np.random.default_rng(1).standard_normal(n ** 3)
    c = volume.forward3(x, n, J, h)
    assert abs(np.linalg.norm(c) - np.linalg.norm(x)) < 1e-12
    assert np.allclose(volume.inverse3(c, n, J, h), x, atol=1e-12)
    y = np.random.default_rng(2).standard_normal(n ** 3)          # inverse3 is the adjoint of forward3
    assert abs(np.dot(volume.forward3(x, n, J, h), y) - np.dot(x, volume.inverse3(y, n, J, h))) < 1e-11


def test_theta_dense_bruteforce_4cubed():
    """Θ[μ][λ] = <Hψ_λ, ψ_μ> with K[x][y] = Σ_k u_k((x − y) mod n) v_k(y) built by loops from P:29-32 (R9) and
    W's rows = ψ_μ: Θ = W K Wᵀ.  A transposed operand (H for H*), a dropped v_k or a wrong row fails."""
    n, J, m = 4, 2, 2
    h = daubechies(2)
    u, v = volume_problem(n, m, 1, seed=3)
    N = n ** 3
    K = np.zeros((N, N))
    for x in range(N):
        x0, x1, x2 = x // (n * n), (x // n) % n, x % n
        for y in range(N):
            y0, y1, y2 = y // (n * n), (y // n) % n, y % n
            z = (((x0 - y0) % n) * n + (x1 - y1) % n) * n + (x2 - y2) % n
            K[x, y] = sum(u[k, z] * v[k, y] for k in range(m))
    assert not np.allclose(K, K.T)                                   # the case can tell H from H*
    W = np.stack([volume.forward3(np.eye(N)[i], n, J, h) for i in range(N)], axis=1)   # W[:, i] = Ψ* e_i
    theta = W @ K @ W.T
    for mu in (0, 1, 9, 30, 63):
        assert np.allclose(volume.theta_row3(n, J, h, u, v, mu), theta[mu], atol=1e-12), mu


def test_identity_and_shift():
    """m = 1, v = 1: u = δ gives Θ = I; u = δ_s (a shift by s) gives Θ = W S Wᵀ with (S f)(x) = f(x − s)."""
    n, J = 8, 2
    h = daubechies(2)
    N = n ** 3
    v = np.ones((1, N))
    u = np.zeros((1, N))
    u[0, 0] = 1.0
    for mu in (0, 70, 511):
        row = volume.theta_row3(n, J, h, u, v, mu)
        want = np.zeros(N)
        want[mu] = 1.0
        assert np.allclose(row, want, atol=1e-12)
    s = (2, 0, 4)                                                    # even shifts ≥ 2^ℓ map level-ℓ wavelets to wavelets
    u = np.zeros((1, n, n, n))
    u[0][s] = 1.0
    lev, e, off, nl = volume.subbands3(n, J)[-1]                     # a level-1 sub-band: shift by s/2 positions
    pos = (1, 2, 3)
    mu = off + (pos[0] * nl + pos[1]) * nl + pos[2]
    row = volume.theta_row3(n, J, h, u.reshape(1, -1), v, mu)
    # <Hψ_λ, ψ_μ> = <ψ_λ(· − s), ψ_μ> = 1 iff λ = μ shifted back by s/2
    q = tuple((p - si // 2) % nl for p, si in zip(pos, s))
    want = np.zeros(N)
    want[off + (q[0] * nl + q[1]) * nl + q[2]] = 1.0
    assert np.allclose(row, want, atol=1e-12)
