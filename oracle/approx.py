"""ORACLE (test infrastructure) — Algorithm 1 of the paper, the η-approximation Θ̃, written out literally.

PAPER.md P:180-195 (Algorithm 1), on dense matrices (N ≤ 4096):
    ε_k = η / (m ‖v_k‖∞)
    A_k = Ψ* U_k Ψ        (wavelet representation of the convolution by u_k)
    Ã_k = A_k thresholded to an ε_k-approximation
    B_k = Ψ* V_k Ψ,  V_k = diag(v_k)
    C_k = Ã_k B_k,   Θ̃ = Σ_k C_k
with the guarantee ‖Θ − Θ̃‖₂ ≤ η (Lemma "accuracy", which uses ‖B_k‖₂ = ‖v_k‖∞).

"Threshold A_k to get an ε_k approximation" is read (DESIGN.md R-A1..R-A3) as the truncation of Theorem 2's
Remark: zero every entry with (i) ||λ| − |μ|| > S or (ii) ϑ(λ,μ) > 2^S, where
    ϑ(λ,μ) = 1 + 2^{min(|λ|,|μ|)} dist(supp ψ_λ, supp ψ_μ)     (Definition 1)
— on the grid: dist = Euclidean distance in pixels between the periodic support boxes, 2^{min|λ|,|μ|} = 1/2^{ℓ_c}
with ℓ_c the coarser of the two levels, so (ii) is dist ≤ (2^S − 1)·2^{ℓ_c} — and S = S_k is the smallest
integer (S = −1: Ã_k = 0) for which the dropped part E = A_k − Ã_k satisfies
    sqrt(‖E‖_1 ‖E‖_∞) ≤ ε_k        (Schur's bound, ≥ ‖E‖₂, so ‖A_k − Ã_k‖₂ ≤ ε_k holds).
The index rule makes the kept pattern exact (no floating-point threshold decisions).

Support of ψ_(ℓ,e,l) per axis a (P:103-104 with reading R7): [2^ℓ l_a + s_a, 2^ℓ l_a + s_a + L_ℓ − 1] mod n,
L_ℓ = (2^ℓ − 1)(2δ − 1) + 1, s_a = 2^{ℓ−1}(2 − 2δ) if the axis carries the wavelet (e_a = 1), else 0
(the scaling function); the whole line when L_ℓ ≥ n.  The coarse block is level J with e = 0.
"""
from __future__ import annotations

import numpy as np

from . import basis


def _ebits(d: int, e: int):
    if d == 1:
        return (0, 1 if e else 0)
    return {0: (0, 0), 1: (0, 1), 2: (1, 0), 3: (1, 1)}[e]


def support_boxes(p):
    """Per Λ index and axis: (start, length) of supp ψ_λ on the periodic line (length n = whole line)."""
    lev, ec, l0, l1 = basis.index_of(p.d, p.n, p.J)
    delta = len(p.h) // 2
    L = (2 ** lev - 1) * (2 * delta - 1) + 1
    starts, lens = [], []
    for a, pos in ((0, l0), (1, l1)):
        bits = np.array([_ebits(p.d, int(e))[a] for e in ec])
        s = (2 ** lev) * pos + np.where(bits == 1, (2 ** (lev - 1)) * (2 - 2 * delta), 0)
        ln = np.minimum(L, p.n)
        if p.d == 1 and a == 0:
            s, ln = np.zeros_like(s), np.ones_like(ln)
        starts.append(np.where(ln >= p.n, 0, np.mod(s, p.n)))
        lens.append(ln)
    return lev, starts, lens


def _axis_gap(s1, L1, s2, L2, n):
    """Distance in pixels between the periodic integer intervals [s1, s1+L1−1] and [s2, s2+L2−1] mod n."""
    d = np.mod(s2 - s1, n)
    overlap = (d <= L1 - 1) | (n - d <= L2 - 1) | (L1 >= n) | (L2 >= n)
    gap = np.minimum(d - (L1 - 1), (n - d) - (L2 - 1))
    return np.where(overlap, 0, gap)


def dist2_matrix(p) -> np.ndarray:
    """Squared Euclidean pixel distance between the periodic support boxes of every pair (ψ_μ, ψ_ν)."""
    lev, st, ln = support_boxes(p)
    N = p.N
    dist2 = np.zeros((N, N), dtype=np.int64)
    for a in ((0, 1) if p.d == 2 else (1,)):
        g = _axis_gap(st[a][:, None], ln[a][:, None], st[a][None, :], ln[a][None, :], p.n).astype(np.int64)
        dist2 += g * g
    return dist2


def s_keep_matrix(p) -> np.ndarray:
    """S_keep[μ][ν] = smallest S ≥ 0 with (i) |ℓ_μ − ℓ_ν| ≤ S and (ii) dist ≤ (2^S − 1)·2^{ℓ_c}."""
    lev, st, ln = support_boxes(p)
    dist2 = dist2_matrix(p)
    delta = np.abs(lev[:, None] - lev[None, :])
    lc = np.maximum(lev[:, None], lev[None, :])
    S = delta.copy()
    for _ in range(64):                       # raise S until (ii) holds (plain loop, integer arithmetic)
        reach = ((2 ** S) - 1) * (2 ** lc)
        bad = reach * reach < dist2
        if not bad.any():
            break
        S = np.where(bad, S + 1, S)
    return S


def conv_rep(p, k: int, W: np.ndarray) -> np.ndarray:
    """A_k = Ψ* U_k Ψ = W U_k Wᵀ, U_k[x][y] = u_k((x − y) mod n)."""
    N, n = p.N, p.n
    idx = np.arange(N)
    if p.d == 1:
        diff = (idx[:, None] - idx[None, :]) % n
    else:
        r, c = idx // n, idx % n
        diff = ((r[:, None] - r[None, :]) % n) * n + ((c[:, None] - c[None, :]) % n)
    return W @ p.u[k][diff] @ W.T


def mult_rep(p, k: int, W: np.ndarray) -> np.ndarray:
    """B_k = Ψ* V_k Ψ = W diag(v_k) Wᵀ."""
    return (W * p.v[k][None, :]) @ W.T


def schur_bound(E: np.ndarray) -> float:
    """sqrt(max column abs sum × max row abs sum) ≥ ‖E‖₂."""
    a = np.abs(E)
    return float(np.sqrt(a.sum(axis=0).max() * a.sum(axis=1).max())) if E.size else 0.0


def choose_S(A: np.ndarray, Sk: np.ndarray, eps: float):
    """Smallest S ∈ {−1, 0, 1, …} whose dropped part has Schur bound ≤ eps; returns (S, bound)."""
    smax = int(Sk[A != 0].max()) if np.any(A != 0) else -1
    for S in range(-1, smax + 1):
        E = np.where(Sk > S, A, 0.0)
        b = schur_bound(E)
        if b <= eps:
            return S, b
    return smax, 0.0


def magnitude_bins(A: np.ndarray) -> np.ndarray:
    """The magnitude rule's index ("simply threshold A"; reading R-A4): b with |a| ∈ [2^{-b-1}, 2^{-b}), from
    the binary exponent, clamped to [0, 62]; index S keeps b ≤ S, i.e. |a| ≥ 2^{-(S+1)}."""
    _, e = np.frexp(np.abs(A))
    return np.clip(-e, 0, 62)


def theta_tilde(p, eta: float, W: np.ndarray | None = None, rule: str = "index"):
    """Θ̃ of Algorithm 1, its bookkeeping {eps, S, bound} per k, and its predicted support (Lemma 9,
    P:1452): 𝒮 = supp(F·I) with F[μ][ν] = [Ã_k[μ][ν] ≠ 0 for some k] and I[ν][λ] = [supp ψ_ν ∩ supp ψ_λ ≠ ∅]
    (the set ℐ of P:1187, which contains supp B_k)."""
    if W is None:
        W = basis.analysis_matrix(p.d, p.n, p.J, p.h)
    Sidx = s_keep_matrix(p) if rule == "index" else None
    T = np.zeros((p.N, p.N))
    F = np.zeros((p.N, p.N), dtype=bool)
    info = []
    for k in range(p.m):
        vinf = float(np.abs(p.v[k]).max())
        eps = eta / (p.m * vinf) if vinf > 0 else np.inf
        A = conv_rep(p, k, W)
        Sk = Sidx if rule == "index" else magnitude_bins(A)
        S, b = choose_S(A, Sk, eps)
        At = np.where(Sk <= S, A, 0.0)
        T += At @ mult_rep(p, k, W)
        F |= At != 0
        info.append({"eps": eps, "S": S, "bound": b})
    I = dist2_matrix(p) == 0
    support = (F.astype(np.float64) @ I.astype(np.float64)) > 0
    return T, info, support
