"""Host-side pin of the separable fine path's atoms (no GPU): pcwd_plan_atom's W_{s,e}, placed at position l on the
periodic line, must equal the oracle's analysis functional of that coefficient — the row of Ψ* that
oracle/basis.analysis_matrix builds by transforming unit impulses with its own (independently written) cascade.
For every level s ≤ 5 the oracle is run with J = s, so both the level-s wavelet rows (e = 1) and the coarse scaling
rows (e = 0, the intermediate W_{s,0} the recursion reuses) are checked.  Reading R-S1."""
import numpy as np
import pytest

from oracle import basis
from paper_2005_09870_b200 import pcwd as P
from synth import filters as F


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2005_09870_b200 import _build
    _build.build()


FILTERS = {"db2": lambda: F.daubechies(2), "db4": lambda: F.daubechies(4), "db6": lambda: F.daubechies(6),
           "sym6": lambda: F.symlet(6)}


def _spec(h, n, J):
    u = np.zeros((1, n))
    u[0, 0] = 1.0
    return P.Spec(d=1, n=n, levels=J, h=h, u=u, v=np.ones((1, n)), retain="full")


@pytest.mark.parametrize("name", list(FILTERS))
def test_atoms_are_the_oracle_analysis_rows(name):
    h = FILTERS[name]()
    n = 256
    for s in range(1, 6):
        W = basis.analysis_matrix(1, n, s, h)
        lev, ec, _, l1 = basis.index_of(1, n, s)
        for e in (0, 1):
            taps, start = P.plan_atom(_spec(h, n, s), s, e)
            assert len(taps) == (2 ** s - 1) * (len(h) - 1) + 1
            rows = np.where((lev == s) & (ec == e))[0]
            for mu in rows[[0, 1, len(rows) // 2, len(rows) - 1]]:
                placed = np.zeros(n)
                np.add.at(placed, (2 ** s * l1[mu] + start + np.arange(len(taps))) % n, taps)
                assert np.max(np.abs(placed - W[mu])) <= 1e-13, (name, s, e, int(l1[mu]))


def test_atoms_orthonormal_translates():
    h = F.daubechies(4)
    for s in range(1, 6):
        for e in (0, 1):
            w, _ = P.plan_atom(_spec(h, 256, s), s, e)
            assert abs(np.dot(w, w) - 1.0) <= 1e-13
            st = 2 ** s   # shift by one position on the level-s grid: orthogonal translates
            assert abs(np.dot(w[st:], w[:-st])) <= 1e-13


def test_atom_argument_errors():
    h = F.daubechies(2)
    with pytest.raises(P.PcwdError):
        P.plan_atom(_spec(h, 64, 3), 0, 0)
    with pytest.raises(P.PcwdError):
        P.plan_atom(_spec(h, 64, 3), 2, 2)
