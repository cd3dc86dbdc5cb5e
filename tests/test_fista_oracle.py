"""Pins of the FISTA oracle (oracle/fista.py) against closed forms and optimality conditions."""
import numpy as np
import pytest

from oracle import fista as F


def test_identity_operator_one_step_is_the_prox():
    """Θ = I, Σ = I, τ = 1: z^(1) = soft(z0, w) (the closed-form minimiser), and it is a fixed point."""
    rng = np.random.default_rng(0)
    z0 = rng.standard_normal(50)
    w = rng.uniform(0.1, 1.0, 50)
    z1 = F.fista(np.eye(50), z0, w, 1, tau=1.0)
    assert np.array_equal(z1, np.sign(z0) * np.maximum(np.abs(z0) - w, 0.0))
    assert np.allclose(F.fista(np.eye(50), z0, w, 7, tau=1.0), z1, atol=0, rtol=0)


@pytest.mark.parametrize("precond", [False, True])
def test_diagonal_operator_converges_to_closed_form(precond):
    """Θ = diag(d): argmin ½(d z − b)² + w|z| = soft(d b, w) / d² per coordinate."""
    rng = np.random.default_rng(1)
    d = rng.uniform(0.3, 2.0, 40)
    b = rng.standard_normal(40)
    w = rng.uniform(0.0, 0.5, 40)
    theta = np.diag(d)
    sigma = F.jacobi_sigma(theta) if precond else None
    z = F.fista(theta, b, w, 3000, sigma=sigma)
    z_star = np.sign(d * b) * np.maximum(np.abs(d * b) - w, 0.0) / d ** 2
    assert np.max(np.abs(z - z_star)) < 1e-9


@pytest.mark.parametrize("precond", [False, True])
def test_kkt_at_convergence(precond):
    """Random sparse-ish Θ: at the minimiser, g = Θᵀ(Θz − z0) has g_λ = −w_λ sign(z_λ) on the support and
    |g_λ| ≤ w_λ off it (the ℓ1 subdifferential)."""
    rng = np.random.default_rng(2)
    N = 60
    theta = rng.standard_normal((N, N)) * (rng.uniform(size=(N, N)) < 0.15) + 3 * np.eye(N)
    z0 = rng.standard_normal(N)
    w = rng.uniform(0.05, 0.5, N)
    sigma = F.jacobi_sigma(theta) if precond else None
    z = F.fista(theta, z0, w, 4000, sigma=sigma)
    g = theta.T @ (theta @ z - z0)
    on = z != 0
    assert np.max(np.abs(g[on] + w[on] * np.sign(z[on]))) < 1e-7
    assert np.all(np.abs(g[~on]) <= w[~on] + 1e-7)


def test_jacobi_sigma_and_step_size_definitions():
    """σ = 1 / column sums of squares; τ·‖ΘΣ^½‖² = 0.99 (checked against an independent power iteration)."""
    rng = np.random.default_rng(3)
    theta = rng.standard_normal((30, 30))
    s = F.jacobi_sigma(theta)
    assert np.allclose(s * np.einsum("ij,ij->j", theta, theta), 1.0)
    m = theta * np.sqrt(s)[None, :]
    v = np.ones(30)
    for _ in range(2000):
        v = m.T @ (m @ v)
        v /= np.linalg.norm(v)
    lam = np.linalg.norm(m.T @ (m @ v))
    assert abs(F.step_size(theta, s) * lam - 0.99) < 1e-8
