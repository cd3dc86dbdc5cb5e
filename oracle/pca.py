"""ORACLE (test infrastructure) — constructing a product-convolution expansion (§3.3), written out plainly.

  * §3.3.2: impulse responses S(·; y_i) sampled at the cell centres y_i = (n/g)(i + ½) (reading R11);
    the u_k are their principal components — the leading m left singular vectors of the W × s matrix whose columns
    are the responses on the window [−R, R]^d (uncentred, reading R10; sign: the largest-|entry| positive); the
    coefficient maps v_k interpolate the projections c_k(y_i) = <S(·; y_i), u_k> periodically and bilinearly between
    the cell centres (reading R12); with one response per pixel (g = n) v_k(y) = c_k(y).
  * §3.3.3: with the SVIR S given at every pixel, the truncated SVD of that W × N matrix is the
    Frobenius-optimal expansion for fixed m; v_k(y) = <S(·, y), u_k>.
numpy's SVD is the one library step; the sign rule, projections, interpolation and embedding are plain loops.
"""
from __future__ import annotations

import numpy as np


def leading_components(X: np.ndarray, m: int):
    """X: (s, W) responses as rows -> (U (W, m) sign-fixed, sigma (m,))."""
    U, s, _ = np.linalg.svd(X.T, full_matrices=False)
    U = U[:, :m].copy()
    for k in range(m):
        i = int(np.argmax(np.abs(U[:, k])))
        if U[i, k] < 0:
            U[:, k] = -U[:, k]
    return U, s[:m]


def embed(U: np.ndarray, d: int, n: int, R: int) -> np.ndarray:
    """u_k(z mod n) = U[w][k] for the window offset z of w (taps that wrap add up) -> (m, N)."""
    side = 2 * R + 1
    m = U.shape[1]
    N = n ** d
    u = np.zeros((m, N))
    for w in range(U.shape[0]):
        a, b = (divmod(w, side) if d == 2 else (0, w))
        z0, z1 = (a - R) % n, (b - R) % n
        idx = z0 * n + z1 if d == 2 else z1
        u[:, idx] += U[w, :]
    return u


def bilinear(c: np.ndarray, d: int, n: int, g: int) -> np.ndarray:
    """c: (s, m) values at the cell centres -> v (m, N), periodic (bi)linear interpolation; g = n: v = c."""
    m = c.shape[1]
    N = n ** d
    if g == n:
        return c.T.copy()
    sp = n / g
    v = np.zeros((m, N))
    for y in range(N):
        y0, y1 = (divmod(y, n) if d == 2 else (0, y))

        def axis(yy):
            t = yy / sp - 0.5
            i = int(np.floor(t))
            return i % g, (i + 1) % g, t - np.floor(t)
        b0, b1, fb = axis(y1)
        if d == 2:
            a0, a1, fa = axis(y0)
            r0 = c[a0 * g + b0] * (1 - fa) + c[a1 * g + b0] * fa
            r1 = c[a0 * g + b1] * (1 - fa) + c[a1 * g + b1] * fa
            v[:, y] = r0 * (1 - fb) + r1 * fb
        else:
            v[:, y] = c[b0] * (1 - fb) + c[b1] * fb
    return v


def pc_from_samples(irs: np.ndarray, d: int, n: int, R: int, g: int, m: int):
    """§3.3.2: (u (m, N), v (m, N), sigma (m,)) from the g^d sampled responses irs (g^d, W)."""
    U, sig = leading_components(irs, m)
    c = irs @ U
    return embed(U, d, n, R), bilinear(c, d, n, g), sig


def pc_from_svir(svir: np.ndarray, d: int, n: int, R: int, m: int):
    """§3.3.3: the truncated SVD of the SVIR given at every pixel (svir (N, W))."""
    return pc_from_samples(svir, d, n, R, n, m)
