"""Host-side checks of libpcwd.so (no GPU): symbols, argument validation, the band stencil
against the oracle's brute-force ranking, and the shard plan."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import basis, retention as ret
from paper_2005_09870_b200 import pcwd as P
from synth import configs as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2005_09870_b200 import _build
    _build.build()


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "pcwd.h")).read()
    declared = set(re.findall(r"\b(pcwd_[a-z_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    L = ctypes.CDLL(P.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert declared <= set(P.EXPORTS)


def _spec(**kw):
    p = C.micro(16, 2, 2, 3, 1, 1, 0)
    base = dict(d=2, n=16, levels=3, h=p.h, u=p.u, v=p.v, retain="band", band_L=8)
    base.update(kw)
    return P.Spec(**base)


@pytest.mark.parametrize("kw,code", [
    ({}, 0),
    ({"d": 3}, 1), ({"n": 48}, 1), ({"n": 1}, 1),
    ({"levels": 0}, 2), ({"levels": 5}, 2), ({"h": np.ones(3)}, 2),
    ({"retain": "threshold", "tau_rel": 0.0}, 3), ({"band_L": 0}, 3), ({"band_L": 257}, 3),
    ({"rank": 2, "world": 2}, 3), ({"world": 0}, 3),
    # not an orthogonal wavelet filter: wrong sum, wrong norm, not orthogonal to even shifts
    ({"h": np.array([1.0, 1.0]) / np.sqrt(2) * 1.001}, 2), ({"h": np.array([0.5, 0.5, 0.5, 0.5]) * np.sqrt(2) / 2}, 2),
    ({"h": np.array([0.6, 0.2, 0.3, 0.5]) * np.sqrt(2) / 1.6}, 2),
    ({"retain": "pattern"}, 3),
])
def test_validation_codes(kw, code):
    assert P.validate(_spec(**kw)) == code
    if code:
        assert P.lib().pcwd_error_string(code).decode() != "unknown status"


def test_m_zero_rejected():
    s = _spec()
    keep = []
    d = P.make_desc(s, keep)
    d.m = 0
    assert P.lib().pcwd_validate(ctypes.byref(d)) == 3


def test_create_rejects_before_touching_cuda():
    s = _spec(levels=9)
    keep = []
    d = P.make_desc(s, keep)
    h = ctypes.c_void_p()
    assert P.lib().pcwd_create(ctypes.byref(d), ctypes.byref(h)) == 2
    assert not h.value


def _stencil_partners(spec, mu):
    """λ set that the library's stencil gives unit μ (positions from its sub-band offsets)."""
    d, n, J = spec.d, spec.n, spec.levels
    sbs = basis.subbands(d, n, J)
    lev, ec, l0, l1 = basis.index_of(d, n, J)
    s_mu = next(i for i, s in enumerate(sbs) if s[2] <= mu < s[2] + s[3] ** d)
    a, o0, o1 = P.plan_stencil(spec, s_mu)
    out = []
    for sb, x0, x1 in zip(a, o0, o1):
        L_, e_, off, nl = sbs[sb]
        D = L_ - lev[mu]
        if D == 0:
            b0, b1 = l0[mu], l1[mu]
        elif D < 0:
            b0, b1 = l0[mu] << -D, l1[mu] << -D
        else:
            b0, b1 = l0[mu] >> D, l1[mu] >> D
        if d == 2:
            out.append(off + ((b0 + x0) % nl) * nl + (b1 + x1) % nl)
        else:
            out.append(off + (b1 + x1) % nl)
    return np.sort(np.array(out))


@pytest.mark.parametrize("d,n,J,L", [(2, 32, 4, 64), (2, 32, 4, 128), (2, 16, 2, 40), (1, 64, 5, 10),
                                     (2, 8, 3, 64), (1, 16, 4, 16)])
def test_stencil_matches_bruteforce_all_units(d, n, J, L):
    p = C.micro(n, d, 2, J, 1, 1, 0, retain="band", band_L=L)
    spec = P.Spec(d, n, J, p.h, p.u, p.v, retain="band", band_L=L)
    for mu in range(p.N):
        assert np.array_equal(_stencil_partners(spec, mu), ret.band_partners(p, mu, L)), mu


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_stencil_matches_bruteforce_config_geometry(name):
    n, J, L = {"c3": (256, 6, 64), "c5": (1024, 8, 128)}[name]
    N = n * n
    u = np.zeros((1, N))
    u[0, 0] = 1.0
    p = C.Problem(name, 2, n, J, C.daubechies(4), u, u, "band", band_L=L)
    spec = P.Spec(2, n, J, p.h, u, u, retain="band", band_L=L)
    rng = np.random.default_rng(0)
    for (lev, e, off, nl) in basis.subbands(2, n, J):
        for mu in {off, off + int(rng.integers(nl * nl))}:
            assert np.array_equal(_stencil_partners(spec, mu), ret.band_partners(p, mu, L)), (lev, e, mu)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_partition(world):
    p = C.get("c3")
    ranges = []
    for r in range(world):
        s = P.Spec(2, p.n, p.J, p.h, p.u, p.v, retain="band", band_L=64, rank=r, world=world)
        ranges.append(P.plan_shard(s))
    assert ranges[0][0] == 0 and ranges[-1][1] == p.N
    for a, b in zip(ranges, ranges[1:]):
        assert a[1] == b[0] and a[0] <= a[1]


@pytest.mark.parametrize("world", [2, 3, 8])
def test_c5_shard_plan_aligned_and_time_balanced(world):
    """Shards of c5 cover Λ, are contiguous, start on multiples of 16 units (whole fine-kernel rounds)
    and put the costly coarse units on the first ranks."""
    p = C.get("c5")
    rs = [P.plan_shard(P.Spec(2, p.n, p.J, p.h, p.u, p.v, retain="band", band_L=128, rank=r, world=world))
          for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == p.N
    for a, b in zip(rs, rs[1:]):
        assert a[1] == b[0] and b[0] % 16 == 0
    sizes = [b - a for a, b in rs]
    assert sizes[0] < sizes[-1]          # rank 0 holds the coarse (expensive) units


def test_corrupted_filter_rejected():
    """SPEC's fault-injection example: one tap of a valid DB4 filter perturbed by 1e-6 → E_CONFIG;
    the valid filter passes."""
    h = C.daubechies(4).copy()
    assert P.validate(_spec(h=h)) == 0
    h[3] += 1e-6
    assert P.validate(_spec(h=h)) == 2
    assert "h:" in P.lib().pcwd_last_error().decode()


@pytest.mark.parametrize("kw,code", [(dict(n=6), 1), (dict(n=512), 1), (dict(levels=0), 2), (dict(levels=4), 2),
                                     (dict(taps=3), 2), (dict(scale=1.01), 2), (dict(m=0), 3)])
def test_rows3d_rejects_before_touching_cuda(kw, code):
    """pcwd_rows3d (d = 3) validates the grid, the depth and the filter on the host (E_SHAPE / E_CONFIG / E_PARAM)
    before any CUDA call."""
    from synth.filters import daubechies
    a = dict(n=8, levels=2, taps=4, scale=1.0, m=1)
    a.update(kw)
    h = np.ascontiguousarray(daubechies(2) * a["scale"])
    dummy = np.zeros(8)
    units = np.zeros(1, dtype=np.int64)
    rc = P.lib().pcwd_rows3d(a["n"], a["levels"], ctypes.c_void_p(h.ctypes.data), a["taps"], a["m"],
                             ctypes.c_void_p(dummy.ctypes.data), ctypes.c_void_p(dummy.ctypes.data),
                             ctypes.c_void_p(units.ctypes.data), 1, ctypes.c_void_p(dummy.ctypes.data), ctypes.c_void_p(0))
    assert rc == code, P.lib().pcwd_last_error().decode()
