"""ORACLE (test infrastructure) — FISTA-W / FISTA-WP in the wavelet domain, written out plainly.

Follows PAPER.md Appendix for problem
    argmin_z ½‖Θ_L z − z0‖² + ‖z‖_{1,w},   z0 = Ψ* f0:
    z^(0) = y^(1) = 0;  for i ≥ 1:
        z^(i)   = Prox^Σ_{‖·‖_{1,w}}( y^(i) − τ Σ Θ_Lᵀ(Θ_L y^(i) − z0) )
        y^(i+1) = z^(i) + (i−1)/(i+2) (z^(i) − z^(i−1))
with Σ = I (FISTA-W) or the Jacobi preconditioner Σ = diag(Θ_LᵀΘ_L)⁻¹ (FISTA-WP; reading R-F1 of
DESIGN.md: "equal to the Jacobi preconditioner diag(Θ_L*Θ_L)" read as its inverse, the usual Jacobi
scaling), Prox^Σ = the soft threshold at τ Σ_λλ w[λ] (the weighted ℓ1 prox in the Σ⁻¹ metric), and
τ = 0.99 / ‖Σ^½ Θ_LᵀΘ_L Σ^½‖₂ (the paper: τ ≤ ‖·‖⁻²), here from the exact 2-norm (numpy SVD).
Dense fp64 numpy; nothing is blocked or fused.
"""
from __future__ import annotations

import numpy as np


def soft(x: np.ndarray, t: np.ndarray) -> np.ndarray:
    """Soft threshold (the prox of t·|·|, componentwise)."""
    return np.sign(x) * np.maximum(np.abs(x) - t, 0.0)


def jacobi_sigma(theta: np.ndarray) -> np.ndarray:
    """Σ = diag(ΘᵀΘ)⁻¹ (0 where the column is empty)."""
    d = np.sum(theta * theta, axis=0)
    return np.where(d > 0, 1.0 / np.where(d > 0, d, 1.0), 0.0)


def step_size(theta: np.ndarray, sigma: np.ndarray | None = None) -> float:
    """τ = 0.99 / ‖Σ^½ ΘᵀΘ Σ^½‖₂ = 0.99 / ‖Θ Σ^½‖₂²."""
    m = theta if sigma is None else theta * np.sqrt(sigma)[None, :]
    s = np.linalg.norm(m, 2)
    return 0.99 / (s * s) if s > 0 else 1.0


def fista(theta: np.ndarray, z0: np.ndarray, w: np.ndarray, iters: int, sigma: np.ndarray | None = None,
          tau: float | None = None) -> np.ndarray:
    """z^(iters) of the iteration above (Σ = I when sigma is None)."""
    N = theta.shape[1]
    s = np.ones(N) if sigma is None else sigma
    if tau is None:
        tau = step_size(theta, sigma)
    y = np.zeros(N)
    z_prev = np.zeros(N)
    z = z_prev
    for i in range(1, iters + 1):
        grad = theta.T @ (theta @ y - z0)
        z = soft(y - tau * s * grad, tau * s * w)
        y = z + (i - 1) / (i + 2) * (z - z_prev)
        z_prev = z
    return z


def objective(theta: np.ndarray, z0: np.ndarray, w: np.ndarray, z: np.ndarray) -> float:
    r = theta @ z - z0
    return 0.5 * float(r @ r) + float(np.sum(w * np.abs(z)))
