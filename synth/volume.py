"""Seeded synthetic inputs for the d = 3 variant: a space-varying anisotropic Gaussian
blur on the n³ torus in product-convolution form.  INPUTS only — none of the decomposition's arithmetic.

u_k: m Gaussian impulse responses of widths σ_k (per axis, seeded) on the window [−R, R]³, unit sum, stored at index
z mod n (taps that wrap accumulate); v_k: smooth positive partition-like weights (seeded low-order cosines,
normalised to Σ_k v_k = 1).  Shapes (m, n³), fp64, row-major (z0, z1, z2).
"""
from __future__ import annotations

import numpy as np


def volume_problem(n: int, m: int, R: int, seed: int):
    rng = np.random.default_rng(seed)
    z = np.arange(-R, R + 1)
    u = np.zeros((m, n, n, n))
    for k in range(m):
        sig = 0.6 + 1.2 * rng.random(3)
        w = np.exp(-0.5 * ((z[:, None, None] / sig[0]) ** 2 + (z[None, :, None] / sig[1]) ** 2
                           + (z[None, None, :] / sig[2]) ** 2))
        w /= w.sum()
        for a, za in enumerate(z):
            for b, zb in enumerate(z):
                for c, zc in enumerate(z):
                    u[k, za % n, zb % n, zc % n] += w[a, b, c]
    t = 2.0 * np.pi * np.arange(n) / n
    v = np.zeros((m, n, n, n))
    for k in range(m):
        ph = 2.0 * np.pi * rng.random(3)
        v[k] = (1.5 + np.cos(t[:, None, None] + ph[0]) * np.cos(t[None, :, None] + ph[1])
                + 0.4 * np.sin(2 * t[None, None, :] + ph[2]))
    v /= v.sum(axis=0, keepdims=True)
    return u.reshape(m, -1), v.reshape(m, -1)
