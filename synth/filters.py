"""Orthonormal wavelet low-pass filters h (an INPUT of the method, not its arithmetic).

PAPER.md P:93-100 assumes a compactly supported orthogonal filter bank (h, g) with
supp h = [0, 2δ-1] and δ = M vanishing moments for Daubechies wavelets, but prints no
coefficient table.  This module derives the extremal-phase (minimum-phase,
front-loaded) Daubechies filters by spectral factorisation in fp64 (DESIGN.md reading
R4).  The oracle and the CUDA path both receive the taps produced here as an input
array, so neither recomputes them.

Pinned in tests/test_filters.py against the DB2 closed form
h = ((1+√3),(3+√3),(3-√3),(1-√3)) / (4√2) and the orthonormality / vanishing-moment
identities.
"""
from __future__ import annotations

import math

import numpy as np


def daubechies(M: int) -> np.ndarray:
    """Extremal-phase Daubechies low-pass filter with M vanishing moments (2M taps).

    |m0(ω)|² = cos^{2M}(ω/2) · P(sin²(ω/2)),  P(y) = Σ_{k<M} C(M-1+k, k) y^k.
    Each root y_r of P gives the pair z, 1/z of z² - (2-4y_r) z + 1 = 0; keeping the
    root inside the unit circle gives the minimum-phase factor.  h is normalised to
    Σ h = √2 (so ‖h‖₂ = 1).
    """
    if M < 1:
        raise ValueError("M must be >= 1")
    if M == 1:
        return np.array([1.0, 1.0]) / math.sqrt(2.0)
    coeffs = [math.comb(M - 1 + k, k) for k in range(M)]  # ascending powers of y
    yroots = np.roots(coeffs[::-1])
    zroots = []
    for yr in yroots:
        b = 2.0 - 4.0 * yr
        disc = np.sqrt(b * b - 4.0 + 0j)
        z1 = (b + disc) / 2.0
        z2 = (b - disc) / 2.0
        zroots.append(z1 if abs(z1) < 1.0 else z2)
    # H(z) (polynomial in z^{-1}) = (1 + z^{-1})^M · Π (1 - z_r z^{-1})
    poly = np.array([1.0 + 0j])
    for _ in range(M):
        poly = np.convolve(poly, [1.0, 1.0])
    for zr in zroots:
        poly = np.convolve(poly, [1.0, -zr])
    h = np.real(poly)
    h = h * (math.sqrt(2.0) / h.sum())
    return h


def _phase_nonlinearity(h: np.ndarray, grid: int = 512) -> float:
    """Mean squared deviation of the unwrapped phase of H(e^{iω}) = Σ h[n] e^{-iωn} from its best linear fit on
    ω ∈ (0, π) (the least-asymmetric criterion)."""
    w = np.linspace(1e-3, math.pi - 1e-3, grid)
    H = np.exp(-1j * np.outer(w, np.arange(len(h)))) @ h
    ph = np.unwrap(np.angle(H))
    A = np.stack([w, np.ones_like(w)], axis=1)
    coef, *_ = np.linalg.lstsq(A, ph, rcond=None)
    return float(np.mean((ph - A @ coef) ** 2))


def symlet(M: int) -> np.ndarray:
    """Least-asymmetric Daubechies ("Symmlet") low-pass filter with M vanishing moments (2M taps) — the paper's
    basis is the Symmlet of order 6.

    Same spectral factorisation as `daubechies` (so |m0(ω)| is identical), but instead of taking every root inside
    the unit circle, one root of each reciprocal pair {z, 1/z} is chosen so that the phase of m0 is closest to
    linear (reading R4b).  Conjugate y-roots are chosen together (h stays real).  Of the two mirror-image
    optima (h and its reversal) the one with the later energy centre Σ n h[n]² is returned.
    """
    if M < 1:
        raise ValueError("M must be >= 1")
    if M == 1:
        return daubechies(1)
    coeffs = [math.comb(M - 1 + k, k) for k in range(M)]
    yroots = np.roots(coeffs[::-1])
    groups, used = [], [False] * len(yroots)
    for i, yr in enumerate(yroots):
        if used[i]:
            continue
        used[i] = True
        g = [i]
        if abs(yr.imag) > 1e-12:
            j = min((j for j in range(len(yroots)) if not used[j]), key=lambda j: abs(yroots[j] - np.conj(yr)))
            used[j] = True
            g.append(j)
        groups.append(g)

    def zpair(yr):
        b = 2.0 - 4.0 * yr
        disc = np.sqrt(b * b - 4.0 + 0j)
        z1, z2 = (b + disc) / 2.0, (b - disc) / 2.0
        return (z1, z2) if abs(z1) < 1.0 else (z2, z1)   # (inside, outside)

    best = None
    for mask in range(1 << len(groups)):
        poly = np.array([1.0 + 0j])
        for _ in range(M):
            poly = np.convolve(poly, [1.0, 1.0])
        for gi, g in enumerate(groups):
            for i in g:
                z = zpair(yroots[i])[(mask >> gi) & 1]
                poly = np.convolve(poly, [1.0, -z])
        h = np.real(poly)
        h = h * (math.sqrt(2.0) / h.sum())          # any factor of |m0|² with m0(0) = √2 has ‖h‖₂ = 1
        score = _phase_nonlinearity(h)
        if best is None or score < best[0] - 1e-12:
            best = (score, h)
    h = best[1]
    n = np.arange(len(h))
    if np.dot(n, h ** 2) < np.dot(n, h[::-1] ** 2):
        h = h[::-1].copy()
    return h


def haar() -> np.ndarray:
    return daubechies(1)


def qmf_highpass(h: np.ndarray) -> dict:
    """g[i] = (-1)^{1-i} h[1-i] for i in [2-2δ, 1].  Returned as {i: g[i]}."""
    L = len(h)
    return {i: ((-1) ** (1 - i)) * h[1 - i] for i in range(2 - L, 2)}
