"""Pins of the ORACLE against what the paper and the mathematics fix (no GPU).

Each test names the passage or identity it checks.  A plausible mistake anywhere in the
oracle (a dropped term, a wrong sign, an index off by one, a transposed operand, a wrong
shift direction) fails at least one of these.
"""
import math
import os

import numpy as np
import pytest

from oracle import basis, operator as op, retention as ret, rows as R
from synth import configs as C
from synth.filters import daubechies

HERE = os.path.dirname(os.path.abspath(__file__))


def _load_golden(name):
    rows = []
    for line in open(os.path.join(HERE, "golden", name)):
        if line.startswith("#") or not line.strip():
            continue
        rows.append([float(x) for x in line.split()])
    return np.array(rows)


# ----------------------------------------------------------------------------- basis

def test_golden_haar_n4():
    W = basis.analysis_matrix(1, 4, 2, daubechies(1))
    assert np.max(np.abs(2 * W - _load_golden("haar_W_n4_J2.txt"))) < 1e-15


def test_golden_db2_folded_n4():
    h = daubechies(2)
    code = _load_golden("db2_W_n4_J1_folded.txt").astype(int)
    ref = np.sign(code) * h[np.abs(code) - 1]
    W = basis.analysis_matrix(1, 4, 1, h)
    assert np.max(np.abs(W - ref)) < 1e-15


@pytest.mark.parametrize("d,n,M,J", [(1, 4, 4, 1), (1, 8, 4, 3), (1, 16, 6, 4), (1, 16, 1, 4),
                                     (2, 4, 2, 2), (2, 8, 4, 3), (2, 16, 6, 4), (2, 8, 1, 3),
                                     (2, 16, 2, 2)])
def test_orthogonality(d, n, M, J):
    """W Wᵀ = I (orthogonal basis), including folded coarse levels."""
    W = basis.analysis_matrix(d, n, J, daubechies(M))
    assert np.max(np.abs(W @ W.T - np.eye(n ** d))) < 1e-13


def test_inverse_and_parseval():
    rng = np.random.default_rng(0)
    for (d, n, M, J) in [(1, 64, 4, 5), (2, 32, 4, 4), (2, 32, 6, 3)]:
        h = daubechies(M)
        f = rng.standard_normal(n ** d)
        c = basis.forward(f, d, n, J, h)
        assert abs(np.linalg.norm(c) - np.linalg.norm(f)) < 1e-12 * np.linalg.norm(f)
        assert np.max(np.abs(basis.inverse(c, d, n, J, h) - f)) < 1e-12


def test_constant_signal_has_no_details():
    # Σ g = 0: constant input -> all detail coefficients vanish
    c = basis.forward(np.ones(32 * 32), 2, 32, 3, daubechies(4))
    assert np.max(np.abs(c[16:])) < 1e-12


def test_haar_2d_closed_form():
    """2-D Haar wavelets are ±2^{-ℓ} on 2^ℓ×2^ℓ boxes; g[0] = -1/√2, g[1] = +1/√2."""
    n, J = 8, 3
    W = basis.analysis_matrix(2, n, J, daubechies(1))
    lev, ec, l0, l1 = basis.index_of(2, n, J)
    for mu in range(n * n):
        L = lev[mu]
        s = 1 << L
        e0, e1 = {0: (0, 0), 1: (0, 1), 2: (1, 0), 3: (1, 1)}[ec[mu]]
        ref = np.zeros((n, n))
        for a in range(s):
            for b in range(s):
                fa = 1.0 if e0 == 0 else (-1.0 if a < s // 2 else 1.0)
                fb = 1.0 if e1 == 0 else (-1.0 if b < s // 2 else 1.0)
                ref[l0[mu] * s + a, l1[mu] * s + b] = fa * fb / s
        assert np.max(np.abs(W[mu].reshape(n, n) - ref)) < 1e-15


def test_shift_law():
    """ψ_{(ℓ,e,l)} = τ_{2^ℓ l} ψ_{(ℓ,e,0)} exactly on the torus (consequence of P:96)."""
    n, J, h = 16, 3, daubechies(4)
    W = basis.analysis_matrix(2, n, J, h)
    for (L, e, off, nl) in basis.subbands(2, n, J):
        base = W[off].reshape(n, n)
        for idx in range(nl * nl):
            r, c = divmod(idx, nl)
            sh = np.roll(base, (r << L, c << L), axis=(0, 1))
            assert np.max(np.abs(W[off + idx].reshape(n, n) - sh)) < 1e-14


@pytest.mark.parametrize("M", [2, 4])
def test_wavelet_support(M):
    """supp φ_{ℓ,0} = [0, (2^ℓ-1)(2δ-1)]; ψ_{ℓ,0} has the same length (2^ℓ-1)(2δ-1)+1
    and, from the recursion P:96, starts at 2^{ℓ-1}(2-2δ) (reading R7: P:104's offset is a slip)."""
    n, J, h = 512, 4, daubechies(M)
    for (L, e, off, nl) in basis.subbands(1, n, J):
        ec = np.zeros(n)
        ec[off] = 1.0
        w = basis.inverse(ec, 1, n, J, h)
        nz = np.nonzero(np.abs(w) > 1e-13)[0]
        nz = np.where(nz > n // 2, nz - n, nz)
        length = (2 ** L - 1) * (2 * M - 1) + 1
        lo = 0 if e == 0 else (2 ** (L - 1)) * (2 - 2 * M)
        assert nz.min() >= lo and nz.max() <= lo + length - 1
        assert nz.min() == lo and nz.max() == lo + length - 1


def test_lemma6_support_count():
    """Lemma 6: a κ-box signal has #supp c_{j,e} ≤ 2^d(2^{d(j-J)}κ^d + (2δ)^d)."""
    rng = np.random.default_rng(3)
    n, Jf, M = 64, 6, 2
    h = daubechies(M)
    for kappa in (1, 3, 8):
        f = np.zeros((n, n))
        f[10:10 + kappa, 20:20 + kappa] = rng.standard_normal((kappa, kappa))
        c = basis.forward(f.ravel(), 2, n, Jf, h)
        for (L, e, off, nl) in basis.subbands(2, n, Jf):
            if e == 0:
                continue
            j = Jf - L                          # paper's scale index
            cnt = np.count_nonzero(np.abs(c[off:off + nl * nl]) > 1e-15)
            assert cnt <= 4 * (2 ** (2 * (j - Jf)) * kappa ** 2 + (2 * M) ** 2)


# ----------------------------------------------------------------------------- operator

def test_kernel_vs_fft_and_direct():
    """K f (Eq. 1) = H f through FFTs = the convolution sum of Eq. 2."""
    rng = np.random.default_rng(1)
    for p in (C.micro(16, 2, 4, 3, 3, 2, 5), C.micro(32, 1, 2, 3, 2, -1, 6), C.micro(8, 2, 2, 2, 2, 1, 7)):
        f = rng.standard_normal(p.N)
        Kf = op.kernel_matrix(p) @ f
        assert np.max(np.abs(Kf - op.apply_fft(p, f))) < 1e-12
        assert np.max(np.abs(Kf - op.apply_direct(p, f))) < 1e-12


def test_adjoint():
    """<Hf, g> = <f, H*g>: the FFT adjoint is Kᵀ."""
    rng = np.random.default_rng(2)
    p = C.micro(16, 2, 4, 3, 3, 3, 8)
    K = op.kernel_matrix(p)
    g = rng.standard_normal(p.N)
    assert np.max(np.abs(K.T @ g - op.adjoint_apply_fft(p, g))) < 1e-12


def test_identity_operator():
    """u = δ₀, v ≡ 1 ⇒ H = I ⇒ Θ = I."""
    p = C.micro(16, 2, 4, 3, 1, 0, 0, u_kind="delta", v_kind="ones")
    T = op.theta_dense(p)
    assert np.max(np.abs(T - np.eye(p.N))) < 1e-13
    r = R.rows(p, [0, 7, 100, 255])
    assert np.max(np.abs(r - np.eye(p.N)[[0, 7, 100, 255]])) < 1e-13


def _blocks(p, T):
    for sa in basis.subbands(p.d, p.n, p.J):
        for sb in basis.subbands(p.d, p.n, p.J):
            yield sa, sb, T[sa[2]:sa[2] + sa[3] ** p.d, sb[2]:sb[2] + sb[3] ** p.d]


@pytest.mark.parametrize("M", [1, 2, 4])
def test_convolution_case_circulant(M):
    """m = 1, v ≡ 1: every sub-band of Θ is rectangular-circulant (Definition P:1148-1154,
    Lemma 1), rows keyed by the coarser index."""
    p = C.micro(16, 2, M, 3, 1, 2, 11, v_kind="ones")
    p.h = daubechies(M)
    T = op.theta_dense(p)
    for sa, sb, B in _blocks(p, T):
        na, nb = sa[3], sb[3]
        B4 = B.reshape(na, na, nb, nb)
        if na <= nb:      # μ (rows) coarser: row shift by 1 ⇔ column shift by nb/na
            s = nb // na
            for r0 in range(na):
                for r1 in range(na):
                    ref = np.roll(B4[0, 0], (r0 * s, r1 * s), axis=(0, 1))
                    assert np.max(np.abs(B4[r0, r1] - ref)) < 1e-13
        else:
            s = na // nb
            for c0 in range(nb):
                for c1 in range(nb):
                    ref = np.roll(B4[:, :, 0, 0], (c0 * s, c1 * s), axis=(0, 1))
                    assert np.max(np.abs(B4[:, :, c0, c1] - ref)) < 1e-13


def test_convolution_case_symmetric_for_even_u():
    rng = np.random.default_rng(4)
    p = C.micro(16, 2, 4, 3, 1, 2, 12, v_kind="ones")
    w = rng.standard_normal((5, 5))
    w = 0.5 * (w + w[::-1, ::-1])                   # u(-z) = u(z)
    p.u = C._embed_window(w.reshape(1, 25), 2, 16, 2)
    T = op.theta_dense(p)
    assert np.max(np.abs(T - T.T)) < 1e-13


def _supports(p):
    W = basis.analysis_matrix(p.d, p.n, p.J, p.h)
    return W, (np.abs(W) > 1e-14)


def test_multiplier_case():
    """u = δ₀: Θ = Ψ* diag(Σ_k v_k) Ψ; supp Θ ⊆ ℐ; ‖Θ‖₂ = ‖Σ v_k‖∞;
    per-row count ≤ (2δ)^d((2^d-1)j + 2^{d(J-j)}) (Lemma 2) at full depth."""
    p = C.micro(16, 2, 2, 4, 2, 0, 13, u_kind="delta")
    T = op.theta_dense(p)
    W, S = _supports(p)
    vs = p.v.sum(axis=0)
    assert np.max(np.abs(T - W @ np.diag(vs) @ W.T)) < 1e-13
    inter = (S.astype(np.int64) @ S.T.astype(np.int64)) > 0
    assert np.all(T[~inter] == 0.0) or np.max(np.abs(T[~inter])) < 1e-15
    assert abs(np.linalg.norm(T, 2) - np.max(np.abs(vs))) < 1e-12
    lev, _, _, _ = basis.index_of(2, 16, 4)
    delta = 2
    for mu in range(p.N):
        j = 4 - lev[mu]
        assert inter[mu].sum() <= (2 * delta) ** 2 * (3 * j + 2 ** (2 * (4 - j)))


def test_frobenius_trace_parseval_linearity():
    """‖Θ‖_F = ‖K‖_F and tr Θ = tr K = Σ_k u_k(0) Σ_y v_k(y) (W orthogonal); per-unit
    Parseval Σ_λ Θ[μ][λ]² = ‖H*ψ_μ‖²; Θ is linear in the (u_k, v_k) pairs."""
    p = C.micro(16, 2, 4, 3, 3, 2, 14)
    T = op.theta_dense(p)
    K = op.kernel_matrix(p)
    assert abs(np.linalg.norm(T) - np.linalg.norm(K)) < 1e-12 * np.linalg.norm(K)
    assert abs(np.trace(T) - sum(p.u[k][0] * p.v[k].sum() for k in range(p.m))) < 1e-12
    for mu in (0, 17, 200):
        e = np.zeros(p.N)
        e[mu] = 1.0
        psi = basis.inverse(e, 2, 16, 3, p.h)
        assert abs(np.sum(T[mu] ** 2) - np.sum(op.adjoint_apply_fft(p, psi) ** 2)) < 1e-12
    import copy
    p1, p2 = copy.copy(p), copy.copy(p)
    p1.u, p1.v = p.u[:1], p.v[:1]
    p2.u, p2.v = p.u[1:], p.v[1:]
    assert np.max(np.abs(op.theta_dense(p1) + op.theta_dense(p2) - T)) < 1e-13


def test_translation_covariance():
    """Shifting every v_k and u-frame by t = 2^J·s maps Θ[μ][λ] to Θ[μ⊕t][λ⊕t] exactly."""
    p = C.micro(16, 2, 2, 2, 2, 1, 15)
    import copy
    q = copy.copy(p)
    t = (4, 8)                                  # multiples of 2^J = 4
    q.v = np.stack([np.roll(v.reshape(16, 16), t, axis=(0, 1)).ravel() for v in p.v])
    T, Tq = op.theta_dense(p), op.theta_dense(q)
    lev, ec, l0, l1 = basis.index_of(2, 16, 2)
    sbs = {(L, e): (off, nl) for (L, e, off, nl) in basis.subbands(2, 16, 2)}
    perm = np.zeros(p.N, dtype=np.int64)
    for i in range(p.N):
        off, nl = sbs[(lev[i], ec[i])]
        perm[i] = off + ((l0[i] + (t[0] >> lev[i])) % nl) * nl + (l1[i] + (t[1] >> lev[i])) % nl
    assert np.max(np.abs(Tq[np.ix_(perm, perm)] - T)) < 1e-13


# ----------------------------------------------------------------------------- C rows oracle

@pytest.mark.parametrize("args", [(8, 2, 2, 2, 2, 1, 0), (16, 2, 4, 3, 3, 2, 1), (16, 1, 4, 4, 2, -1, 2),
                                  (8, 2, 4, 3, 2, 2, 3), (8, 2, 6, 3, 3, -1, 4), (16, 2, 1, 4, 2, 3, 5),
                                  (4, 2, 4, 2, 1, 1, 6), (32, 1, 6, 5, 3, 4, 7)])
def test_rows_equal_dense(args):
    """oracle/rows.c (H*ψ_μ then Ψ*) equals the dense definition W K Wᵀ, element by element."""
    p = C.micro(*args)
    T = op.theta_dense(p)
    r = R.rows(p, np.arange(p.N))
    assert np.max(np.abs(r - T)) < 1e-13 * max(1.0, np.abs(T).max())
    assert np.max(np.abs(R.rowmax(p, np.arange(p.N)) - np.abs(T).max(axis=1))) < 1e-13


def test_rows_equal_fft_route_large():
    """Two independent large-N routes agree: C direct sums vs numpy FFT adjoint (c3 units)."""
    p = C.get("c3")
    units = [0, 16, 5000, 60000, p.N - 1]
    r = R.rows(p, units)
    for i, mu in enumerate(units):
        ref = op.theta_row_fft(p, mu)
        assert np.max(np.abs(r[i] - ref)) < 1e-13 * max(1.0, np.abs(ref).max())


def test_c1_c2_dense_vs_rows():
    for name, units in (("c1", np.arange(256)), ("c2", [0, 3, 777, 4095])):
        p = C.get(name)
        T = op.theta_dense(p)
        r = R.rows(p, units)
        assert np.max(np.abs(r - T[units])) < 1e-13


def test_parseval_bound_pruning():
    """rowmax(bound) returns -‖row‖₂ only when ‖row‖₂ < bound, else the true max."""
    p = C.micro(16, 2, 4, 3, 3, 2, 1)
    T = op.theta_dense(p)
    rm = R.rowmax(p, np.arange(p.N), bound=0.5)
    for mu in range(p.N):
        if rm[mu] < 0:
            assert abs(-rm[mu] - np.linalg.norm(T[mu])) < 1e-12 and np.linalg.norm(T[mu]) < 0.5
        else:
            assert abs(rm[mu] - np.abs(T[mu]).max()) < 1e-13


# ----------------------------------------------------------------------------- retention (R14-R16)

def test_band_rule_exactly_L_total_order():
    p = C.micro(16, 2, 4, 3, 1, 1, 0, retain="band", band_L=40)
    for mu in (0, 5, 70, 255):
        k = ret.band_key(p, mu)
        keys = set(zip(*[a.tolist() for a in k]))
        assert len(keys) == p.N                            # a total order: no ties
        cols = ret.band_partners(p, mu, 40)
        assert len(cols) == 40 and np.all(np.diff(cols) > 0)
        assert mu in cols                                  # Δ = ρ = 0 comes first


def test_band_rule_is_a_stencil():
    """Partners of μ and of μ shifted by one position are translates (the rule uses only
    relative quantities), which is what lets the library tabulate it once per sub-band."""
    n, J = 32, 4
    p = C.micro(n, 2, 4, J, 1, 1, 0, retain="band", band_L=64)
    lev, ec, l0, l1 = basis.index_of(2, n, J)
    sbs = {(L, e): (off, nl) for (L, e, off, nl) in basis.subbands(2, n, J)}
    for (L, e, off, nl) in basis.subbands(2, n, J):
        mu = off + (nl // 2) * nl + nl // 2
        if nl < 2:
            continue
        mu2 = off + (nl // 2) * nl + (nl // 2 + 1) % nl   # shift by one along axis 1 (finest: 2 px)
        A = ret.band_partners(p, mu, 64)
        B = ret.band_partners(p, mu2, 64)
        # shift of A by τ = 2^L pixels along axis 1
        def shift(i):
            off2, nl2 = sbs[(lev[i], ec[i])]
            s = (1 << L) >> lev[i] if L >= lev[i] else None
            return None if s is None else off2 + l0[i] * nl2 + (l1[i] + s) % nl2
        shifted = [shift(i) for i in A if lev[i] <= L]
        assert set(shifted) <= set(B.tolist())


def test_threshold_closed_inequality():
    row = np.array([0.5, -1.0, 1e-4, -1e-4, 9.99e-5, 0.0])
    assert ret.threshold_keep(row, 1e-4).tolist() == [0, 1, 2, 3]
