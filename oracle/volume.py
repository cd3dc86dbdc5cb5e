"""ORACLE (test infrastructure) — d = 3: the wavelet representation of a product-convolution operator on the
periodic n × n × n grid, written out plainly in fp64.  Only tests/ and __graft_entry__.smoke() may import this.

Follows PAPER.md:
  * P:22, P:63-65   the grid is N_1 × … × N_d (here d = 3, N_1 = N_2 = N_3 = n = 2^p), periodic.
  * P:29-32         H f = Σ_k u_k ⋆ (v_k ⊙ f), (u ⋆ f)(x) = Σ_y u((x − y) mod n) f(y) (reading R9).
  * P:110-119       isotropic separable basis: one step filters axis 0, then axis 1, then axis 2 with (h, g)
                    (reading R6 carried to three axes); sub-band e = (e0, e1, e2) ∈ {0,1}^3, e = 0 feeds the next
                    step.  The 1-D step itself is oracle.basis.analysis_step (R5), used as is.
  * P:121-125, R2   Λ layout: the coarse scaling block, then levels J, J−1, …, 1, within a level the orientations
                    e_code = 4 e0 + 2 e1 + e2 = 1 … 7, positions row-major (l0, l1, l2).
  * P:43, R1 Θ[μ][λ] = <H ψ_λ, ψ_μ>, Θ = Ψ* H Ψ; row μ of Θ is Ψ*(H* ψ_μ) with
                    H* g = Σ_k v_k ⊙ (ũ_k ⋆ g), ũ(z) = u(−z).

No blocking, windowing or reordering: every step filters the whole periodic array.  Pinned by
tests/test_volume_oracle.py (tensor-product identity against the pinned 1-D transform, orthogonality, the dense
brute-force W K Wᵀ on 4³, H = I, H = a shift).
"""
from __future__ import annotations

import numpy as np

from . import basis

ORIENTS = (1, 2, 3, 4, 5, 6, 7)


def _bits(e: int) -> tuple[int, int, int]:
    return (e >> 2) & 1, (e >> 1) & 1, e & 1


def subbands3(n: int, J: int):
    """Λ layout for d = 3: list of (level ℓ, e_code, offset, side n_ℓ) in storage order."""
    out = []
    nJ = n >> J
    off = 0
    out.append((J, 0, off, nJ))
    off += nJ ** 3
    for lev in range(J, 0, -1):
        nl = n >> lev
        for e in ORIENTS:
            out.append((lev, e, off, nl))
            off += nl ** 3
    assert off == n ** 3
    return out


def forward3(f: np.ndarray, n: int, J: int, h: np.ndarray) -> np.ndarray:
    """Ψ* f on the n³ torus, output in Λ layout."""
    cur = np.asarray(f, dtype=np.float64).reshape(n, n, n)
    details = {}
    for lev in range(1, J + 1):
        parts = {0: cur}
        for axis in (0, 1, 2):                      # axis 0 first (e0), then e1, then e2
            nxt = {}
            for code, x in parts.items():
                a, d = basis.analysis_step(x, h, axis)
                nxt[2 * code] = a
                nxt[2 * code + 1] = d
            parts = nxt
        details[lev] = {e: parts[e] for e in ORIENTS}
        cur = parts[0]
    out = [cur.ravel()]
    for lev in range(J, 0, -1):
        for e in ORIENTS:
            out.append(details[lev][e].ravel())
    return np.concatenate(out)


def inverse3(c: np.ndarray, n: int, J: int, h: np.ndarray) -> np.ndarray:
    """Ψ c: the adjoint (= inverse) of forward3.  Returns a flat length-n³ signal."""
    c = np.asarray(c, dtype=np.float64)
    blocks = {}
    for (lev, e, off, nl) in subbands3(n, J):
        blocks[(lev, e)] = c[off:off + nl ** 3].reshape(nl, nl, nl)
    cur = blocks[(J, 0)]
    for lev in range(J, 0, -1):
        parts = {0: cur}
        for e in ORIENTS:
            parts[e] = blocks[(lev, e)]
        for axis in (2, 1, 0):                      # undo axis 2 first
            nxt = {}
            for code in range(len(parts) // 2):
                nxt[code] = basis.synthesis_step(parts[2 * code], parts[2 * code + 1], h, axis)
            parts = nxt
        cur = parts[0]
    return cur.ravel()


def adjoint_apply3(n: int, u: np.ndarray, v: np.ndarray, g: np.ndarray) -> np.ndarray:
    """H* g = Σ_k v_k ⊙ (ũ_k ⋆ g), (ũ_k ⋆ g)(y) = Σ_x u_k((x − y) mod n) g(x), by the circular-correlation theorem."""
    shp = (n, n, n)
    G = np.fft.fftn(np.asarray(g, dtype=np.float64).reshape(shp))
    out = np.zeros(shp)
    for k in range(u.shape[0]):
        U = np.fft.fftn(u[k].reshape(shp))
        out += v[k].reshape(shp) * np.real(np.fft.ifftn(np.conj(U) * G))
    return out.ravel()


def theta_row3(n: int, J: int, h: np.ndarray, u: np.ndarray, v: np.ndarray, mu: int) -> np.ndarray:
    """Row μ of Θ = Ψ* H Ψ: Θ[μ][·] = Ψ*(H* ψ_μ), ψ_μ = Ψ e_μ."""
    e = np.zeros(n ** 3)
    e[mu] = 1.0
    psi = inverse3(e, n, J, h)
    return forward3(adjoint_apply3(n, u, v, psi), n, J, h)
