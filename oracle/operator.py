"""ORACLE (test infrastructure) — the product-convolution operator and Θ by brute force.

  * P:25-32 (Eq. 1-2): H f = Σ_k u_k ⋆ (v_k ⊙ f) with the periodic convolution
    (u ⋆ f)(x) = Σ_y u((x-y) mod n) f(y) (reading R9; ⋆ is not defined in the paper),
    so the kernel is K[x][y] = Σ_k u_k((x-y) mod n) v_k(y).
  * H can be applied through FFTs in O(mN log N)  (apply_fft — a pin for K).
  * θ[λ,μ] = <H ψ_λ, ψ_μ>, Θ = Ψ* H Ψ.  Matrix entry Θ[μ][λ] := θ[λ,μ]
    (reading R1): Θ = W K Wᵀ with W = Ψ* (rows ψ_μ).
  * Adjoint: H* g = Σ_k v_k ⊙ (ũ_k ⋆ g), ũ(z) = u(-z); so row μ of Θ is
    Θ[μ][·] = (Ψ* H* ψ_μ)ᵀ because <H ψ_λ, ψ_μ> = <ψ_λ, H* ψ_μ>.
"""
from __future__ import annotations

import numpy as np

from . import basis


def _shape(p):
    return (p.n,) * p.d


def kernel_matrix(p) -> np.ndarray:
    """Dense K[x][y] = Σ_k u_k((x - y) mod n) v_k(y)  (Eq. 1-2).  N ≤ 4096 only."""
    N, n, d = p.N, p.n, p.d
    assert N <= 4096
    idx = np.arange(N)
    if d == 1:
        diff = (idx[:, None] - idx[None, :]) % n
    else:
        r, c = idx // n, idx % n
        diff = ((r[:, None] - r[None, :]) % n) * n + ((c[:, None] - c[None, :]) % n)
    K = np.zeros((N, N))
    for k in range(p.m):
        K += p.u[k][diff] * p.v[k][None, :]
    return K


def apply_direct(p, f: np.ndarray) -> np.ndarray:
    """H f by the definition: Σ_k Σ_y u_k(x-y) v_k(y) f(y), looping over the nonzeros of u_k."""
    shp = _shape(p)
    out = np.zeros(shp)
    for k in range(p.m):
        w = (p.v[k] * f).reshape(shp)
        uk = p.u[k].reshape(shp)
        for z in zip(*np.nonzero(uk)):
            out += uk[z] * np.roll(w, shift=z, axis=tuple(range(p.d)))
    return out.ravel()


def apply_fft(p, f: np.ndarray) -> np.ndarray:
    """H f = Σ_k IDFT(DFT(u_k) · DFT(v_k ⊙ f))."""
    shp = _shape(p)
    ax = tuple(range(p.d))
    acc = np.zeros(shp, dtype=np.complex128)
    for k in range(p.m):
        acc += np.fft.fftn(p.u[k].reshape(shp), axes=ax) * np.fft.fftn((p.v[k] * f).reshape(shp), axes=ax)
    return np.real(np.fft.ifftn(acc, axes=ax)).ravel()


def adjoint_apply_fft(p, g: np.ndarray) -> np.ndarray:
    """H* g = Σ_k v_k ⊙ (ũ_k ⋆ g) with ũ_k ⋆ g = IDFT(conj(DFT(u_k)) · DFT(g)) (u real)."""
    shp = _shape(p)
    ax = tuple(range(p.d))
    G = np.fft.fftn(g.reshape(shp), axes=ax)
    out = np.zeros(p.N)
    for k in range(p.m):
        c = np.real(np.fft.ifftn(np.conj(np.fft.fftn(p.u[k].reshape(shp), axes=ax)) * G, axes=ax))
        out += p.v[k] * c.ravel()
    return out


def theta_dense(p, W: np.ndarray | None = None) -> np.ndarray:
    """Θ = W K Wᵀ (entry [μ][λ] = <H ψ_λ, ψ_μ>)  — plain matrix products, N ≤ 4096."""
    if W is None:
        W = basis.analysis_matrix(p.d, p.n, p.J, p.h)
    K = kernel_matrix(p)
    return W @ K @ W.T


def theta_row_fft(p, mu: int) -> np.ndarray:
    """Θ[μ][·] = Ψ*(H* ψ_μ) with ψ_μ = Ψ e_μ, H* through FFTs (any N; slow but plain)."""
    e = np.zeros(p.N)
    e[mu] = 1.0
    psi = basis.inverse(e, p.d, p.n, p.J, p.h)
    return basis.forward(adjoint_apply_fft(p, psi), p.d, p.n, p.J, p.h)
