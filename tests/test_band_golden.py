"""Pins of the band rule (reading R16 / SURVEY C17) that do not come from the oracle itself.

1. A hand-derived partner list (tests/golden/band_16x16_J3.txt; derivation in its header) for one unit per
   level on 16², J = 3, at several L — catches a ρ measured on λ's grid instead of the coarser grid, a
   truncating instead of flooring shift of negative offsets, and the wrong half-open canonical interval.
2. The survey's independently derived rule-A maxima: the largest number of
   partners per unit with Δ + ρ ≤ S is 4 / 48 / 267 / 1,182 for S = 0..3 on 256², J = 6.
Both the oracle (`oracle.retention`) and the library's stencil (`pcwd_plan_stencil`) are checked against
the golden list.
"""
import os

import numpy as np
import pytest

from oracle import basis, retention as ret
from synth import configs as C

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden():
    out = []
    for line in open(os.path.join(HERE, "golden", "band_16x16_J3.txt")):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        head, cols = line.split(":")
        mu, L = (int(x) for x in head.split())
        out.append((mu, L, np.array([int(x) for x in cols.split()])))
    return out


GOLD = _golden()


def _problem(L):
    u = np.zeros((1, 256))
    u[0, 0] = 1.0
    return C.Problem("band16", 2, 16, 3, C.daubechies(2), u, u, "band", band_L=L)


def test_golden_file_is_well_formed():
    assert len(GOLD) == 9
    for mu, L, cols in GOLD:
        assert len(cols) == L and np.all(np.diff(cols) > 0) and mu in cols


@pytest.mark.parametrize("mu,L", [(g[0], g[1]) for g in GOLD])
def test_oracle_band_partners_match_hand_derivation(mu, L):
    want = next(c for (m, l, c) in GOLD if m == mu and l == L)
    got = ret.band_partners(_problem(L), mu, L)
    assert np.array_equal(got, want), (sorted(set(got) - set(want)), sorted(set(want) - set(got)))


@pytest.mark.parametrize("mu,L", [(g[0], g[1]) for g in GOLD])
def test_library_stencil_matches_hand_derivation(mu, L):
    from paper_2005_09870_b200 import _build, pcwd as P
    _build.build()
    from test_library_host import _stencil_partners
    p = _problem(L)
    spec = P.Spec(2, 16, 3, p.h, p.u, p.v, retain="band", band_L=L)
    want = next(c for (m, l, c) in GOLD if m == mu and l == L)
    assert np.array_equal(_stencil_partners(spec, mu), want)


def test_rule_A_maxima_256_J6():
    """max over units of #{λ : Δ+ρ ≤ S} = 4, 48, 267, 1182 for S = 0..3 (256², J = 6).
    The key is translation-invariant per sub-band, so one unit per sub-band gives the maximum; a second
    unit per sub-band (other position) must give the same counts."""
    n, J = 256, 6
    u = np.zeros((1, n * n))
    u[0, 0] = 1.0
    p = C.Problem("ruleA", 2, n, J, C.daubechies(4), u, u, "band", band_L=1)
    best = np.zeros(4, dtype=np.int64)
    rng = np.random.default_rng(0)
    for (lev, e, off, nl) in basis.subbands(2, n, J):
        counts = []
        for mu in (off, off + int(rng.integers(nl * nl))):
            s = ret.band_key(p, mu)[0]
            counts.append([int(np.sum(s <= S)) for S in range(4)])
        assert counts[0] == counts[1], (lev, e, counts)
        best = np.maximum(best, counts[0])
    assert best.tolist() == [4, 48, 267, 1182]
