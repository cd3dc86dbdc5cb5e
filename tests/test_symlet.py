"""Pins for the Symmlet filters (synth/filters.symlet; the paper's basis is the Symmlet of order 6):
the orthonormal-filter identities of SPEC S:31-33, the same magnitude response as the extremal-phase Daubechies
filter of the same order (both are spectral factors of one polynomial), and a phase closer to linear."""
import math

import numpy as np
import pytest

from synth.filters import _phase_nonlinearity, daubechies, qmf_highpass, symlet


@pytest.mark.parametrize("M", [2, 3, 4, 5, 6, 8])
def test_symlet_identities_and_magnitude(M):
    h, d = symlet(M), daubechies(M)
    L = len(h)
    assert L == 2 * M
    assert abs(np.sum(h) - math.sqrt(2)) < 1e-12 and abs(np.linalg.norm(h) - 1) < 1e-12
    for k in range(1, M):
        assert abs(np.dot(h[:L - 2 * k], h[2 * k:])) < 1e-12
    g = qmf_highpass(h)
    for p in range(M):
        assert abs(sum(val * (i ** p) for i, val in g.items())) < 1e-8 * max(1, L ** p)
    w = np.linspace(0, math.pi, 257)
    E = np.exp(-1j * np.outer(w, np.arange(L)))
    assert np.max(np.abs(np.abs(E @ h) - np.abs(E @ d))) < 1e-12
    assert _phase_nonlinearity(h) <= _phase_nonlinearity(d) + 1e-12


def test_symlet6_is_much_less_asymmetric_than_db6():
    assert _phase_nonlinearity(symlet(6)) < 0.1 * _phase_nonlinearity(daubechies(6))
    assert not np.allclose(symlet(6), daubechies(6)) and not np.allclose(symlet(6), daubechies(6)[::-1])
