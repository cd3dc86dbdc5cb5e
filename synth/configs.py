"""Seeded synthetic inputs for the five BASELINE.json configs and the micro cases.

This module produces INPUTS only (filters h, convolution filters u_k, multipliers v_k,
the retention rule); it contains none of the decomposition's arithmetic.  It is the
one module shared by the oracle-side tests and the CUDA-side tests / bench.

Recipes follow DESIGN.md §3 (input recipe), which settles what BASELINE.json leaves
open (SURVEY.md §8(c) ledger C10-C15):
  * grid row-major, axis 0 = y (row), axis 1 = x (column); periodic torus
  * impulse responses S(z; y) sampled on [-R, R]^d (periodised), normalised to unit sum
  * "PCA" = uncentred SVD of the IR matrix sampled at cell centres y_i = (n/g)(i + 1/2);
    u_k = leading m left singular vectors, sign so that the largest-|entry| is positive
    (§3.3.2)
  * v_k = projections <S(.;y), u_k> (exact, or periodic bilinear interpolation of the
    grid projections), or seeded smoothed random fields (config 4)
  * numpy PCG64 default_rng, seeds fixed per field.

u_k and v_k are returned as fp64 arrays of shape (m, N) (row-major flattening of the
n^d grid); u_k(z) is stored at index z mod n (so u_k is "centred" at the origin).
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

from .filters import daubechies


@dataclass
class Problem:
    name: str
    d: int
    n: int
    J: int
    h: np.ndarray
    u: np.ndarray          # (m, N) fp64
    v: np.ndarray          # (m, N) fp64
    retain: str            # "full" | "threshold" | "band"
    tau_rel: float = 0.0
    band_L: int = 0
    dtypes: tuple = ("f64",)
    meta: dict = field(default_factory=dict)
    pat_rowptr: np.ndarray | None = None   # retain == "pattern": CSR over units (int64 N+1, int32 columns)
    pat_col: np.ndarray | None = None

    def __post_init__(self):
        self.u = np.ascontiguousarray(self.u, dtype=np.float64)
        self.v = np.ascontiguousarray(self.v, dtype=np.float64)
        self.h = np.ascontiguousarray(self.h, dtype=np.float64)

    @property
    def m(self) -> int:
        return self.u.shape[0]

    @property
    def N(self) -> int:
        return self.n ** self.d

    def sha256(self) -> str:
        s = hashlib.sha256()
        for a in (self.h, self.u, self.v):
            s.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
        s.update(repr((self.d, self.n, self.J, self.retain, self.tau_rel, self.band_L)).encode())
        if self.pat_rowptr is not None:
            s.update(np.ascontiguousarray(self.pat_rowptr, dtype=np.int64).tobytes())
            s.update(np.ascontiguousarray(self.pat_col, dtype=np.int32).tobytes())
        return s.hexdigest()

    def fingerprint(self) -> list:
        """Rounding-robust summary of the inputs (sums, sums of squares, weighted sums, 16 sampled entries of h, u, v):
        the PCA and FFT steps of the recipes go through LAPACK / BLAS / pocketfft, whose last bits differ between
        CPUs, so the sha256 of the fp64 inputs is machine-dependent while these agree to ~1e-15 relative."""
        out = []
        rng = np.random.default_rng(12345)
        for a in (self.h, self.u, self.v):
            x = np.ascontiguousarray(a, dtype=np.float64).ravel()
            w = rng.uniform(-1.0, 1.0, size=x.size)
            idx = rng.integers(0, x.size, size=16)
            out += [float(x.sum()), float(np.dot(x, x)), float(np.dot(w, x))] + [float(v) for v in x[idx]]
        return out

    def fingerprint_matches(self, fp, rtol: float = 1e-10) -> bool:
        mine = self.fingerprint()
        if len(mine) != len(fp):
            return False
        scale = max(abs(v) for v in mine) or 1.0
        return all(abs(a - b) <= rtol * max(abs(a), abs(b), 1e-6 * scale) for a, b in zip(mine, fp))


# ----------------------------------------------------------------------------- helpers

def _offsets(R: int, d: int):
    r = np.arange(-R, R + 1)
    if d == 1:
        return (r,)
    dy, dx = np.meshgrid(r, r, indexing="ij")
    return dy, dx


def _normalise(ir: np.ndarray) -> np.ndarray:
    return ir / ir.sum(axis=-1, keepdims=True)


def _pca(irs: np.ndarray, m: int) -> np.ndarray:
    """irs: (#samples, W) -> (m, W) leading left singular vectors of irs.T, sign-fixed."""
    U, s, _ = np.linalg.svd(irs.T, full_matrices=False)
    U = U[:, :m].T.copy()
    for k in range(m):
        i = np.argmax(np.abs(U[k]))
        if U[k, i] < 0:
            U[k] = -U[k]
    return U


def _embed_window(win: np.ndarray, R: int, n: int, d: int) -> np.ndarray:
    """(m, (2R+1)^d) window over offsets [-R,R]^d -> (m, n^d) periodic array."""
    m = win.shape[0]
    if d == 1:
        out = np.zeros((m, n))
        z = np.arange(-R, R + 1) % n
        np.add.at(out, (slice(None), z), win)
        return out
    out = np.zeros((m, n, n))
    z = np.arange(-R, R + 1) % n
    w = win.reshape(m, 2 * R + 1, 2 * R + 1)
    for a in range(2 * R + 1):
        for b in range(2 * R + 1):
            out[:, z[a], z[b]] += w[:, a, b]
    return out.reshape(m, n * n)


def _bilinear_periodic(c: np.ndarray, g: int, n: int) -> np.ndarray:
    """c: (m, g, g) values at cell centres (n/g)(i+1/2) -> (m, n*n), periodic bilinear."""
    s = n / g
    t = np.arange(n) / s - 0.5
    i0 = np.floor(t).astype(np.int64)
    f = t - i0
    i0m = i0 % g
    i1m = (i0 + 1) % g
    cy0 = c[:, i0m, :]
    cy1 = c[:, i1m, :]
    cy = cy0 * (1 - f)[None, :, None] + cy1 * f[None, :, None]      # (m, n, g)
    cx0 = cy[:, :, i0m]
    cx1 = cy[:, :, i1m]
    out = cx0 * (1 - f)[None, None, :] + cx1 * f[None, None, :]     # (m, n, n)
    return out.reshape(c.shape[0], n * n)


def _smooth_field(n: int, corr: float, seed: int) -> np.ndarray:
    """White noise filtered by a periodic Gaussian of std corr/sqrt(2) (ledger C15)."""
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((n, n))
    s = corr / math.sqrt(2.0)
    f = np.fft.fftfreq(n)
    fy, fx = np.meshgrid(f, f, indexing="ij")
    H = np.exp(-2.0 * (math.pi ** 2) * (s ** 2) * (fx ** 2 + fy ** 2))
    return np.real(np.fft.ifft2(np.fft.fft2(w) * H))


# ----------------------------------------------------------------------------- configs

def config1() -> Problem:
    """1-D n=256, Haar, J=8, m=3; periodised Gaussian IRs σ(y)=2+3y/256 over the whole circle."""
    n, m = 256, 3
    z = np.arange(n)
    z = np.where(z < n // 2, z, z - n)          # centred offsets

    def ir(y):
        sig = 2.0 + 3.0 * y / n
        acc = np.zeros(n)
        for w in (-1, 0, 1):
            acc += np.exp(-((z + w * n) ** 2) / (2 * sig * sig))
        return acc / acc.sum()

    ys = 16 * np.arange(16) + 8
    irs = np.stack([ir(y) for y in ys])          # (16, n), indexed by z mod n
    u = _pca(irs, m)                             # (m, n)
    allir = np.stack([ir(y) for y in range(n)])  # (n, n)
    v = (allir @ u.T).T                          # v_k(y) = <S(.;y), u_k>
    return Problem("c1", 1, n, 8, daubechies(1), u, v, "full", dtypes=("f64",),
                   meta={"ir": "periodised Gaussian sigma(y)=2+3y/256"})


def config2() -> Problem:
    """64², DB4, J=5, m=5; isotropic Gaussian σ=1+2(x+y)/128, R=9; 8x8 PCA grid; bilinear v."""
    n, m, R, g = 64, 5, 9, 8
    dy, dx = _offsets(R, 2)

    def ir(y0, x0):
        sig = 1.0 + 2.0 * (x0 + y0) / 128.0
        return np.exp(-(dx ** 2 + dy ** 2) / (2 * sig * sig)).ravel()

    cs = (n // g) * np.arange(g) + (n // g) // 2
    irs = _normalise(np.stack([ir(a, b) for a in cs for b in cs]))
    uw = _pca(irs, m)
    c = (irs @ uw.T).T.reshape(m, g, g)
    v = _bilinear_periodic(c, g, n)
    u = _embed_window(uw, R, n, 2)
    return Problem("c2", 2, n, 5, daubechies(4), u, v, "threshold", tau_rel=1e-4,
                   dtypes=("f32", "f64"), meta={"R": R})


def config3() -> Problem:
    """256², DB4, J=6, m=8; anisotropic rotated Gaussian; 16x16 PCA grid; exact projections; band L=64."""
    n, m, R, g = 256, 8, 12, 16
    dy, dx = _offsets(R, 2)
    dy = dy.ravel().astype(np.float64)
    dx = dx.ravel().astype(np.float64)

    def irs_at(Y, X):
        X = np.asarray(X, dtype=np.float64)[:, None]
        Y = np.asarray(Y, dtype=np.float64)[:, None]
        sx = 1.0 + 3.0 * X / n
        sy = 1.0 + 3.0 * Y / n
        th = np.pi * X / n
        c, s = np.cos(th), np.sin(th)
        # Σ = R diag(sx², sy²) Rᵀ ; quadratic form with Σ⁻¹ = R diag(1/sx², 1/sy²) Rᵀ
        a = c * dx + s * dy
        b = -s * dx + c * dy
        q = (a / sx) ** 2 + (b / sy) ** 2
        return _normalise(np.exp(-0.5 * q))

    cs = (n // g) * np.arange(g) + (n // g) // 2
    Yg, Xg = np.meshgrid(cs, cs, indexing="ij")
    irs = irs_at(Yg.ravel(), Xg.ravel())
    uw = _pca(irs, m)
    v = np.zeros((m, n * n))
    Yall, Xall = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    Yall, Xall = Yall.ravel(), Xall.ravel()
    for s0 in range(0, n * n, 8192):
        blk = irs_at(Yall[s0:s0 + 8192], Xall[s0:s0 + 8192])
        v[:, s0:s0 + 8192] = (blk @ uw.T).T
    u = _embed_window(uw, R, n, 2)
    return Problem("c3", 2, n, 6, daubechies(4), u, v, "band", band_L=64,
                   dtypes=("f32",), meta={"R": R})


def config4() -> Problem:
    """512², DB6, J=7, m=10; Moffat β=2.5, α=max(.5, 1.5+2 sin cos); 16x16 PCA; random v; tau 1e-5."""
    n, m, R, g = 512, 10, 16, 16
    dy, dx = _offsets(R, 2)
    r2 = (dx ** 2 + dy ** 2).ravel().astype(np.float64)

    def ir(y0, x0):
        al = 1.5 + 2.0 * math.sin(2 * math.pi * x0 / n) * math.cos(2 * math.pi * y0 / n)
        al = max(al, 0.5)
        return (1.0 + r2 / (al * al)) ** (-2.5)

    cs = (n // g) * np.arange(g) + (n // g) // 2
    irs = _normalise(np.stack([ir(a, b) for a in cs for b in cs]))
    uw = _pca(irs, m)
    u = _embed_window(uw, R, n, 2)
    v = np.zeros((m, n * n))
    for k in range(m):
        f = _smooth_field(n, 64.0, 1000 + k)
        f = (f - f.mean()) / f.std()
        v[k] = f.ravel()
    return Problem("c4", 2, n, 7, daubechies(6), u, v, "threshold", tau_rel=1e-5,
                   dtypes=("f32",), meta={"R": R})


def config5() -> Problem:
    """1024², DB4, J=8, m=10; Gaussian σ∈[1,6] from a smooth field; 32x32 PCA; bilinear v; band L=128."""
    n, m, R, g = 1024, 10, 18, 32
    dy, dx = _offsets(R, 2)
    r2 = (dx ** 2 + dy ** 2).ravel().astype(np.float64)
    F = _smooth_field(n, 128.0, 2000)
    sig = 1.0 + 5.0 * (F - F.min()) / (F.max() - F.min())
    cs = (n // g) * np.arange(g) + (n // g) // 2
    irs = _normalise(np.stack([np.exp(-r2 / (2 * sig[a, b] ** 2)) for a in cs for b in cs]))
    uw = _pca(irs, m)
    c = (irs @ uw.T).T.reshape(m, g, g)
    v = _bilinear_periodic(c, g, n)
    u = _embed_window(uw, R, n, 2)
    return Problem("c5", 2, n, 8, daubechies(4), u, v, "band", band_L=128,
                   dtypes=("f32",), meta={"R": R})


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5}

_cache: dict = {}


def get(name: str) -> Problem:
    if name not in _cache:
        _cache[name] = CONFIGS[name]()
    return _cache[name]


# ----------------------------------------------------------------------------- micro cases

def micro(n: int, d: int, M: int, J: int, m: int, R: int, seed: int, retain: str = "full",
          tau_rel: float = 0.0, band_L: int = 0, u_kind: str = "random",
          v_kind: str = "random") -> Problem:
    """Small random operator: u_k supported on [-R,R]^d (R<0: dense u), v_k random."""
    rng = np.random.default_rng(seed)
    N = n ** d
    if u_kind == "delta":
        u = np.zeros((m, N))
        u[:, 0] = 1.0
    elif R < 0:
        u = rng.standard_normal((m, N))
    else:
        W = (2 * R + 1) ** d
        u = _embed_window(rng.standard_normal((m, W)), R, n, d)
    if v_kind == "ones":
        v = np.ones((m, N))
    else:
        v = rng.standard_normal((m, N))
    return Problem(f"micro_n{n}_d{d}_M{M}_J{J}_m{m}_R{R}_s{seed}_{retain}", d, n, J,
                   daubechies(M), u, v, retain, tau_rel=tau_rel, band_L=band_L,
                   dtypes=("f64", "f32"))


def c2_samples():
    """The sampled impulse responses config 2 is built from (8 × 8 cell centres, R = 9): (irs (64, 361), n, R, g, m)."""
    n, m, R, g = 64, 5, 9, 8
    dy, dx = _offsets(R, 2)

    def ir(y0, x0):
        sig = 1.0 + 2.0 * (x0 + y0) / 128.0
        return np.exp(-(dx ** 2 + dy ** 2) / (2 * sig * sig)).ravel()

    cs = (n // g) * np.arange(g) + (n // g) // 2
    return _normalise(np.stack([ir(a, b) for a in cs for b in cs])), n, R, g, m


def svir_anisotropic(n: int, R: int) -> np.ndarray:
    """The space-varying impulse response of config 3's recipe (anisotropic rotated Gaussian, σx = 1 + 3x/n,
    σy = 1 + 3y/n, angle πx/n) at EVERY pixel of an n × n torus: (N, (2R+1)²), rows normalised to unit sum."""
    dy, dx = _offsets(R, 2)
    out = np.zeros((n * n, (2 * R + 1) ** 2))
    for y0 in range(n):
        for x0 in range(n):
            sx, sy, th = 1 + 3.0 * x0 / n, 1 + 3.0 * y0 / n, math.pi * x0 / n
            c, s = math.cos(th), math.sin(th)
            a = c * dx + s * dy
            b = -s * dx + c * dy
            out[y0 * n + x0] = np.exp(-0.5 * ((a / sx) ** 2 + (b / sy) ** 2)).ravel()
    return _normalise(out)


def random_pattern(N: int, max_per_row: int, seed: int, empty_every: int = 7):
    """A seeded retained pattern for PATTERN tests: row μ keeps μ itself plus k − 1 other random units
    (k uniform in 1..max_per_row), except every `empty_every`-th row, which is empty.  Returns the CSR
    (rowptr int64 N+1, col int32, columns increasing within a row)."""
    rng = np.random.default_rng(seed)
    rp, cols = [0], []
    for mu in range(N):
        if empty_every and mu % empty_every == 3:
            c = np.zeros(0, np.int64)
        else:
            k = int(rng.integers(1, min(max_per_row, N) + 1))
            others = rng.choice(N - 1, size=k - 1, replace=False)
            others = others + (others >= mu)            # skip μ itself
            c = np.sort(np.concatenate([[mu], others]))
        cols.append(c.astype(np.int32))
        rp.append(rp[-1] + len(c))
    return np.array(rp, dtype=np.int64), np.concatenate(cols).astype(np.int32)
