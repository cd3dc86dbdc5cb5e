"""ORACLE (test infrastructure) — the periodic orthogonal wavelet basis, written out plainly.

Follows PAPER.md §2:
  * P:94-96  φ_{j,l} = Σ_n h[n-2l] φ_{j+1,n},  ψ_{j,l} = Σ_n g[n-2l] φ_{j+1,n}; with
    φ_{J,n} = 1_{n} the finest scaling functions are Diracs, so one analysis step on a
    periodic line x of even length n' is
        a[l] = Σ_t h[t] x[(2l+t) mod n'],
        d[l] = Σ_i g[i] x[(2l+i) mod n']   with g[i] = (-1)^{1-i} h[1-i],
    for l < n'/2; taps that wrap more than once accumulate (the filter folds; reading R5).
  * P:110-119 isotropic separable d-D basis: filter axis 0 with (h, g), then axis 1,
    giving sub-bands e = (e0, e1); e = (0,0) feeds the next step (reading R6).
  * P:121-125 with the garbled Λ of P:117 read as: one coarse scaling block (level J,
    e = 0) followed by the detail sub-bands of levels J, J-1, ..., 1, orientations
    (0,1), (1,0), (1,1) (d=2) or 1 (d=1), positions row-major (readings R2, R3).
  * P:127  Ψ* = forward transform, Ψ = its inverse (= adjoint, the basis is orthogonal).

Level ℓ ∈ {1..J} counts analysis steps (ℓ = 1 finest); a level-ℓ sub-band has n >> ℓ
positions per axis.  No blocking or windowing: every step filters the whole periodic
array.
"""
from __future__ import annotations

import numpy as np


def highpass(h: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """g as (taps, offsets): g[i] = (-1)^{1-i} h[1-i], i ∈ [2-2δ, 1]."""
    L = len(h)
    offs = np.arange(2 - L, 2)
    taps = np.array([((-1.0) ** (1 - i)) * h[1 - i] for i in offs])
    return taps, offs


def analysis_step(x: np.ndarray, h: np.ndarray, axis: int) -> tuple[np.ndarray, np.ndarray]:
    """One periodic analysis step along `axis`: returns (approx a, detail d)."""
    x = np.moveaxis(x, axis, -1)
    n2 = x.shape[-1]
    half = n2 // 2
    l2 = 2 * np.arange(half)
    a = np.zeros(x.shape[:-1] + (half,))
    d = np.zeros(x.shape[:-1] + (half,))
    for t in range(len(h)):                       # a[l] = Σ_t h[t] x[2l+t]
        a += h[t] * x[..., (l2 + t) % n2]
    gt, go = highpass(h)
    for c, i in zip(gt, go):                      # d[l] = Σ_i g[i] x[2l+i]
        d += c * x[..., (l2 + i) % n2]
    return np.moveaxis(a, -1, axis), np.moveaxis(d, -1, axis)


def synthesis_step(a: np.ndarray, d: np.ndarray, h: np.ndarray, axis: int) -> np.ndarray:
    """Adjoint of analysis_step (= its inverse, the step is orthogonal)."""
    a = np.moveaxis(a, axis, -1)
    d = np.moveaxis(d, axis, -1)
    half = a.shape[-1]
    n2 = 2 * half
    x = np.zeros(a.shape[:-1] + (n2,))
    l2 = 2 * np.arange(half)
    for t in range(len(h)):
        np.add.at(x, (..., (l2 + t) % n2), h[t] * a)
    gt, go = highpass(h)
    for c, i in zip(gt, go):
        np.add.at(x, (..., (l2 + i) % n2), c * d)
    return np.moveaxis(x, -1, axis)


def subbands(d: int, n: int, J: int):
    """Λ layout: list of (level ℓ, e_code, offset, side n_ℓ) in storage order.

    e_code: 0 = coarse scaling block (ℓ = J); d=2: 1=(0,1), 2=(1,0), 3=(1,1); d=1: 1.
    """
    out = []
    nJ = n >> J
    off = 0
    out.append((J, 0, off, nJ))
    off += nJ ** d
    for lev in range(J, 0, -1):
        nl = n >> lev
        for e in ((1, 2, 3) if d == 2 else (1,)):
            out.append((lev, e, off, nl))
            off += nl ** d
    assert off == n ** d
    return out


def forward(f: np.ndarray, d: int, n: int, J: int, h: np.ndarray) -> np.ndarray:
    """Ψ* f : the plain periodic cascade, output in Λ layout (length N)."""
    cur = np.asarray(f, dtype=np.float64).reshape((n,) * d)
    details = {}
    for lev in range(1, J + 1):
        if d == 1:
            a, dd = analysis_step(cur, h, 0)
            details[lev] = {1: dd}
            cur = a
        else:
            a0, d0 = analysis_step(cur, h, 0)          # axis 0 first (e0)
            a0a, a0d = analysis_step(a0, h, 1)         # then axis 1 (e1)
            d0a, d0d = analysis_step(d0, h, 1)
            details[lev] = {1: a0d, 2: d0a, 3: d0d}
            cur = a0a
    parts = [cur.ravel()]
    for lev in range(J, 0, -1):
        for e in ((1, 2, 3) if d == 2 else (1,)):
            parts.append(details[lev][e].ravel())
    return np.concatenate(parts)


def inverse(c: np.ndarray, d: int, n: int, J: int, h: np.ndarray) -> np.ndarray:
    """Ψ c : inverse of `forward` (its adjoint).  Returns a flat length-N signal."""
    c = np.asarray(c, dtype=np.float64)
    sb = subbands(d, n, J)
    blocks = {}
    for (lev, e, off, nl) in sb:
        blocks[(lev, e)] = c[off:off + nl ** d].reshape((nl,) * d)
    cur = blocks[(J, 0)]
    for lev in range(J, 0, -1):
        if d == 1:
            cur = synthesis_step(cur, blocks[(lev, 1)], h, 0)
        else:
            a0 = synthesis_step(cur, blocks[(lev, 1)], h, 1)
            d0 = synthesis_step(blocks[(lev, 2)], blocks[(lev, 3)], h, 1)
            cur = synthesis_step(a0, d0, h, 0)
    return cur.ravel()


def analysis_matrix(d: int, n: int, J: int, h: np.ndarray) -> np.ndarray:
    """W = Ψ* as a dense N×N matrix: row μ is ψ_μ (W[μ][i] = <e_i, ψ_μ> = ψ_μ(i))."""
    N = n ** d
    W = np.zeros((N, N))
    for i in range(N):
        e = np.zeros(N)
        e[i] = 1.0
        W[:, i] = forward(e, d, n, J, h)
    return W


def index_of(d: int, n: int, J: int):
    """Per Λ index: arrays (level, e_code, l0, l1) — l0 = 0 for d = 1."""
    N = n ** d
    lev = np.zeros(N, dtype=np.int64)
    ec = np.zeros(N, dtype=np.int64)
    l0 = np.zeros(N, dtype=np.int64)
    l1 = np.zeros(N, dtype=np.int64)
    for (L, e, off, nl) in subbands(d, n, J):
        cnt = nl ** d
        idx = np.arange(cnt)
        lev[off:off + cnt] = L
        ec[off:off + cnt] = e
        if d == 2:
            l0[off:off + cnt] = idx // nl
            l1[off:off + cnt] = idx % nl
        else:
            l1[off:off + cnt] = idx
    return lev, ec, l0, l1
