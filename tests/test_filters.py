"""Pins for the filter inputs (synth/filters.py): closed forms and SPEC S:31-33 identities."""
import math

import numpy as np
import pytest

from synth.filters import daubechies, qmf_highpass


def test_db2_closed_form():
    # Daubechies' 4-tap filter in closed form (extremal phase), SPEC S:54-56 / DESIGN.md R4
    s3 = math.sqrt(3.0)
    ref = np.array([1 + s3, 3 + s3, 3 - s3, 1 - s3]) / (4 * math.sqrt(2.0))
    assert np.max(np.abs(daubechies(2) - ref)) < 1e-15


def test_haar_closed_form():
    assert np.allclose(daubechies(1), [1 / math.sqrt(2), 1 / math.sqrt(2)], atol=0, rtol=1e-16)


@pytest.mark.parametrize("M", [1, 2, 3, 4, 5, 6, 8])
def test_orthonormal_filter_identities(M):
    h = daubechies(M)
    L = len(h)
    assert L == 2 * M                                    # δ = M for Daubechies
    assert abs(np.sum(h) - math.sqrt(2)) < 1e-12
    assert abs(np.linalg.norm(h) - 1) < 1e-12
    for k in range(1, M):                                 # Σ_n h[n] h[n+2k] = 0
        assert abs(np.dot(h[:L - 2 * k], h[2 * k:])) < 1e-12
    g = qmf_highpass(h)                                   # g[i] = (-1)^{1-i} h[1-i]
    assert set(g) == set(range(2 - L, 2))                 # supp g = [-2(δ-1), 1]
    for p in range(M):                                    # M vanishing moments
        assert abs(sum(val * (i ** p) for i, val in g.items())) < 1e-8 * max(1, (L ** p))


def test_db4_front_loaded():
    # extremal phase = minimum phase: partial energy of the first taps is maximal
    h = daubechies(4)
    assert h[1] > 0.7 and abs(h[-1]) < 0.02
