"""Pins of the Algorithm-1 oracle (oracle/approx.py) that do not come from the oracle itself:
the accuracy lemma ‖Θ − Θ̃‖₂ ≤ η and ‖A_k − Ã_k‖₂ ≤ ε_k (true 2-norms by SVD), ‖B_k‖₂ = ‖v_k‖∞
(P:1483), the limits η → 0 (Θ̃ = Θ of the exact oracle) and η → ∞ (Θ̃ = 0), and hand-derived truncation
indices S_keep on a 1-D Haar grid (Definition 1, Remark P:1178)."""
import numpy as np
import pytest

from oracle import approx as AP, basis, operator as op
from synth import configs as C


def _haar8():
    u = np.zeros((1, 8))
    u[0, 0] = 1.0
    return C.Problem("haar8", 1, 8, 3, C.daubechies(1), u, u, "full")


def test_support_boxes_haar_hand_derived():
    """Haar (δ = 1), n = 8, J = 3: level 1 ψ_l on [2l, 2l+1], level 2 on [4l, 4l+3], level 3 (and the coarse
    block) the whole line.  Λ: coarse 0, level 3 → 1, level 2 → 2..3, level 1 → 4..7."""
    lev, st, ln = AP.support_boxes(_haar8())
    assert list(lev) == [3, 3, 2, 2, 1, 1, 1, 1]
    assert list(st[1]) == [0, 0, 0, 4, 0, 2, 4, 6]
    assert list(ln[1]) == [8, 8, 4, 4, 2, 2, 2, 2]


def test_s_keep_haar_hand_derived():
    """S_keep = smallest S with |ℓ−ℓ'| ≤ S and dist ≤ (2^S − 1)·2^{ℓ_c}:
    (4,6): [0,1] vs [4,5], dist 3, ℓ_c = 1 → (2^S−1)·2 ≥ 3 → S = 2;   (4,5): dist 1 → S = 1;
    (4,7): [0,1] vs [6,7] wraps, dist 5−... = 8−6−1 = 1 → S = 1;      (4,4): 0;
    (4,3): [0,1] vs [4,7], dist min(3, 1) = 1, Δ = 1, ℓ_c = 2 → S = 1;  (4,2): overlap, Δ = 1 → 1;
    (4,0) / (4,1): the whole line, Δ = 2 → 2;  (2,3): [0,3] vs [4,7], dist 1, ℓ_c = 2 → S = 1."""
    Sk = AP.s_keep_matrix(_haar8())
    want = {(4, 6): 2, (4, 5): 1, (4, 7): 1, (4, 4): 0, (4, 3): 1, (4, 2): 1, (4, 0): 2, (4, 1): 2, (2, 3): 1,
            (5, 7): 2, (0, 1): 0}
    for (a, b), s in want.items():
        assert Sk[a, b] == s and Sk[b, a] == s, (a, b, Sk[a, b])


def _gauss_micro(n=16, J=3, m=3, seed=5):
    """A small space-varying blur (the paper's operator shape): Gaussian u_k, smooth v_k."""
    p = C.micro(n, 2, 2, J, m, 2, seed)
    r = np.arange(-2, 3)
    g = np.exp(-(r[:, None] ** 2 + r[None, :] ** 2) / 2.0)
    u = np.zeros((m, n, n))
    for k in range(m):
        w = g ** (1 + k) / (g ** (1 + k)).sum()
        for i, a in enumerate(r):
            for j, b in enumerate(r):
                u[k, a % n, b % n] = w[i, j]
    p.u = u.reshape(m, -1)
    y = np.arange(n) / n
    p.v = np.stack([1.0 + 0.3 * (k + 1) * np.cos(2 * np.pi * (y[:, None] + 2 * k * y[None, :])) for k in range(m)]).reshape(m, -1)
    return p


@pytest.mark.parametrize("rule", ["index", "magnitude"])
@pytest.mark.parametrize("eta", [1.0, 1e-1, 1e-2, 1e-3, 1e-5])
def test_accuracy_lemma(eta, rule):
    p = _gauss_micro()
    W = basis.analysis_matrix(p.d, p.n, p.J, p.h)
    T = op.theta_dense(p, W)
    Tt, info, sup = AP.theta_tilde(p, eta, W, rule)
    assert np.linalg.norm(T - Tt, 2) <= eta * (1 + 1e-12)
    assert not np.any(Tt[~sup])                                            # supp Θ̃ ⊆ 𝒮 (Lemma 9)
    for k, inf in enumerate(info):
        A = AP.conv_rep(p, k, W)
        Sk = AP.s_keep_matrix(p) if rule == "index" else AP.magnitude_bins(A)
        E = np.where(Sk > inf["S"], A, 0.0)
        assert np.linalg.norm(E, 2) <= inf["eps"] * (1 + 1e-12)          # ‖A_k − Ã_k‖₂ ≤ ε_k
        assert abs(inf["eps"] - eta / (p.m * np.abs(p.v[k]).max())) <= 1e-15 * inf["eps"]


def test_sparsity_grows_as_eta_shrinks():
    p = _gauss_micro()
    W = basis.analysis_matrix(p.d, p.n, p.J, p.h)
    nnz = [np.count_nonzero(AP.theta_tilde(p, eta, W)[2]) for eta in (10.0, 2.0, 1e-4)]
    assert nnz[0] <= nnz[1] <= nnz[2] and nnz[0] < nnz[2]


def test_multiplier_norm():
    """‖B_k‖₂ = ‖V_k‖₂ = ‖v_k‖∞ (Ψ orthogonal)."""
    p = C.micro(16, 2, 4, 3, 2, 2, 7)
    W = basis.analysis_matrix(p.d, p.n, p.J, p.h)
    for k in range(p.m):
        assert abs(np.linalg.norm(AP.mult_rep(p, k, W), 2) - np.abs(p.v[k]).max()) <= 1e-12


def test_eta_to_zero_is_exact_theta():
    p = C.micro(16, 2, 4, 3, 2, 2, 8)
    W = basis.analysis_matrix(p.d, p.n, p.J, p.h)
    T = op.theta_dense(p, W)
    Tt, info, _ = AP.theta_tilde(p, 1e-300, W)
    assert np.max(np.abs(T - Tt)) <= 1e-13 * np.max(np.abs(T))
    assert all(i["bound"] == 0.0 for i in info)


def test_eta_huge_is_zero():
    p = C.micro(16, 2, 4, 3, 2, 2, 9)
    Tt, info, sup = AP.theta_tilde(p, 1e6)
    assert all(i["S"] == -1 for i in info) and not np.any(Tt) and not np.any(sup)


def test_zero_multiplier_term_contributes_nothing():
    """‖v_k‖∞ = 0 ⇒ ε_k = ∞, Ã_k = 0."""
    p = C.micro(16, 2, 4, 3, 2, 2, 10)
    p.v[1] = 0.0
    Tt, info, _ = AP.theta_tilde(p, 1e-3)
    assert info[1]["S"] == -1
    q = C.micro(16, 2, 4, 3, 2, 2, 10)
    q.u, q.v = q.u[:1], q.v[:1]
    T1, _, _ = AP.theta_tilde(q, 1e-3 / 2)          # same ε_0 = η/(m ‖v_0‖∞) with m = 1
    assert np.max(np.abs(Tt - T1)) <= 1e-14


def test_magnitude_bins_hand_values():
    """|a| ∈ [2^{-b-1}, 2^{-b}) → b (0.5 ∈ [½, 1) → 0, 2^-10 ∈ [2^-10, 2^-9) → 9); ≥ 1 → 0; tiny → 62; exact zeros
    (which contribute nothing either way) → 0."""
    a = np.array([1.5, 1.0, 0.75, 0.5, 0.4999, 0.25, -0.3, 2.0 ** -10, 1e-30, 0.0])
    assert AP.magnitude_bins(a).tolist() == [0, 0, 0, 0, 1, 1, 1, 9, 62, 0]


def test_magnitude_rule_is_sparser_for_the_same_eta():
    p = _gauss_micro()
    W = basis.analysis_matrix(p.d, p.n, p.J, p.h)
    a = np.count_nonzero(AP.theta_tilde(p, 1.0, W, "index")[2])
    b = np.count_nonzero(AP.theta_tilde(p, 1.0, W, "magnitude")[2])
    assert b < a
