"""ORACLE (test infrastructure) — which (μ, λ) pairs of Θ are retained, by brute force.

BASELINE.json names three retention rules; the paper only motivates them (Theorem 2 and
its Remark: keep entries close in scale and position, or "simply threshold
A").  Readings (R14-R16):

  full       every pair (μ, λ) ∈ Λ×Λ, exact zeros included.
  threshold  keep iff |Θ[μ][λ]| ≥ τ_rel · M, M = max over all entries of |Θ| (closed
             inequality), decided on fp64 values.
  pattern    the caller's CSR over units (any Θ_L of Eq. 7; the A_L of the Remark).
  band (L)   for each unit μ keep exactly the L partners λ that come first in the total
             order of `band_key` (scale proximity Δ = |ℓ-ℓ'|, then position proximity ρ
             measured on the coarser of the two grids — the (i)/(ii) quantities of the
             Remark, ranked instead of cut; ties broken by sub-band and offset).

Everything here ranks ALL N partners of a unit with plain numpy; nothing is tabulated.
"""
from __future__ import annotations

import numpy as np

from . import basis


def _canon(raw: np.ndarray, nl: np.ndarray) -> np.ndarray:
    """Canonical periodic offset in [-nl/2, nl/2)  (nl = 1 -> 0)."""
    half = nl // 2
    return np.mod(raw + half, nl) - half


def _pdist(q: np.ndarray, nc: np.ndarray) -> np.ndarray:
    r = np.mod(q, nc)
    return np.minimum(r, nc - r)


def band_key(p, mu: int):
    """Key components for every λ ∈ Λ relative to unit μ (reading R16).

    Returns a tuple of int arrays (Δ+ρ, Δ, ρ, ℓ, e, Σo², o0, o1) over all λ.
    """
    lev, ec, l0, l1 = basis.index_of(p.d, p.n, p.J)
    Lm, l0m, l1m = lev[mu], l0[mu], l1[mu]
    delta = np.abs(lev - Lm)
    nl = p.n >> lev                       # side of λ's grid
    lc = np.maximum(lev, Lm)
    nc = p.n >> lc                        # side of the coarser grid
    same = lev == Lm
    finer = lev < Lm
    coarser = lev > Lm
    keys_o = []
    keys_rho = []
    comps = [(l0, l0m), (l1, l1m)] if p.d == 2 else [(l1, l1m)]
    for (l, lm) in comps:
        base = np.where(same, lm, np.where(finer, lm << np.maximum(Lm - lev, 0),
                                            lm >> np.maximum(lev - Lm, 0)))
        o = _canon(l - base, nl)
        # ρ on the coarser grid: λ finer -> floor(o / 2^Δ); otherwise o itself
        q = np.where(finer, np.floor_divide(o, 1 << delta), o)
        rho = _pdist(q, nc)
        keys_o.append(o)
        keys_rho.append(rho)
    rho = np.max(np.stack(keys_rho), axis=0)
    o2 = np.sum(np.stack(keys_o) ** 2, axis=0)
    if p.d == 2:
        o0, o1 = keys_o
    else:
        o0, o1 = np.zeros_like(keys_o[0]), keys_o[0]
    return (delta + rho, delta, rho, lev, ec, o2, o0, o1)


def band_partners(p, mu: int, L: int) -> np.ndarray:
    """The L partners of μ first in band_key order, returned sorted by λ (CSR column order)."""
    k = band_key(p, mu)
    order = np.lexsort(tuple(reversed(k)))          # primary key = k[0]
    return np.sort(order[:L])


def band_pattern_dense(p, L: int):
    """{μ: sorted λ array} for all units (small N only)."""
    return {mu: band_partners(p, mu, L) for mu in range(p.N)}


def threshold_keep(row: np.ndarray, tau: float) -> np.ndarray:
    """Retained λ of a row: |θ| ≥ τ (closed inequality)."""
    return np.nonzero(np.abs(row) >= tau)[0]


def retained_row(p, mu: int, row: np.ndarray, M: float | None = None):
    """(cols, vals) retained for unit μ given its full fp64 row Θ[μ][·]."""
    if p.retain == "full":
        cols = np.arange(p.N)
    elif p.retain == "band":
        cols = band_partners(p, mu, p.band_L)
    elif p.retain == "threshold":
        assert M is not None
        cols = threshold_keep(row, p.tau_rel * M)
    elif p.retain == "pattern":     # the caller's retained set, taken as given (index-defined: zeros kept, R14)
        cols = np.asarray(p.pat_col[p.pat_rowptr[mu]:p.pat_rowptr[mu + 1]], dtype=np.int64)
    else:
        raise ValueError(p.retain)
    return cols, row[cols]
