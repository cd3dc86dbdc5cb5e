"""d = 3 on the GPU (pcwd_rows3d: rows of Θ on the n³ torus) against
the pinned fp64 oracle (oracle/volume.py), element by element: every unit of small volumes (incl. a filter longer
than the grid and a support box covering whole axes), units of every sub-band at 16³ and 32³; bar 1e-12 relative
Frobenius per row (fp64 both sides, ≤ 3·J·taps + box·m rounded terms per entry); and the boundary's error codes."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import record_parity  # noqa: E402
from oracle import volume  # noqa: E402
from paper_2005_09870_b200 import PcwdError, pcwd  # noqa: E402
from synth.filters import daubechies, haar  # noqa: E402
from synth.volume import volume_problem  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_09870_b200 import _build
    _build.build()


def _compare(name, n, J, h, u, v, units):
    got = pcwd.rows3d(n, J, h, torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda(), units).cpu().numpy()
    num = den = 0.0
    for i, mu in enumerate(units):
        want = volume.theta_row3(n, J, h, u, v, int(mu))
        scale = max(np.linalg.norm(want), 1e-300)
        err = np.linalg.norm(got[i] - want) / scale
        assert err <= TOL, (name, int(mu), err)
        num += np.sum((got[i] - want) ** 2)
        den += np.sum(want ** 2)
    record_parity(name, "f64", float(np.sqrt(num / den)), len(units), n=n, J=J, taps=len(h))


ALL_UNIT_CASES = [("haar_n4_J2", 4, 2, 1, 2, 1, 11), ("db2_n8_J2", 8, 2, 2, 2, 1, 12), ("db2_n8_J3", 8, 3, 2, 3, 2, 13),
                  ("db4_n4_J2_folded", 4, 2, 4, 2, 1, 14), ("db3_n4_J1_wholebox", 4, 1, 3, 2, 2, 15)]


@pytest.mark.parametrize("case", ALL_UNIT_CASES, ids=[c[0] for c in ALL_UNIT_CASES])
def test_every_unit(case):
    name, n, J, M, m, R, seed = case
    h = haar() if M == 1 else daubechies(M)
    u, v = volume_problem(n, m, R, seed)
    _compare("vol3_" + name, n, J, h, u, v, np.arange(n ** 3))


SAMPLED = [("db3_n16_J3", 16, 3, 3, 3, 2, 21, 3), ("db4_n32_J2", 32, 2, 4, 2, 2, 22, 1), ("db2_n32_J5", 32, 5, 2, 3, 3, 23, 1),
           ("db2_n32_J1_finelaunchonly", 32, 1, 2, 2, 1, 24, 2)]   # no unit reaches the coarse launch


@pytest.mark.parametrize("case", SAMPLED, ids=[c[0] for c in SAMPLED])
def test_units_of_every_subband(case):
    """Per sub-band: its first and last position (the periodic seams) and seeded interior ones."""
    name, n, J, M, m, R, seed, per = case
    h = daubechies(M)
    u, v = volume_problem(n, m, R, seed)
    rng = np.random.default_rng(seed)
    units = []
    for (lev, e, off, nl) in volume.subbands3(n, J):
        cnt = nl ** 3
        units += [off, off + cnt - 1] + [off + int(x) for x in rng.integers(0, cnt, per)]
    _compare("vol3_" + name, n, J, h, u, v, np.unique(np.array(units)))


def test_units_order_and_repeats():
    """Rows come back in the caller's order; a repeated unit gives the same row twice."""
    n, J = 8, 2
    h = daubechies(2)
    u, v = volume_problem(n, 2, 1, 31)
    ud, vd = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
    units = np.array([300, 5, 300, 0, 511])
    got = pcwd.rows3d(n, J, h, ud, vd, units).cpu().numpy()
    ref = pcwd.rows3d(n, J, h, ud, vd, np.arange(n ** 3)).cpu().numpy()
    assert np.array_equal(got, ref[units])
    assert pcwd.rows3d(n, J, h, ud, vd, np.zeros(0, dtype=np.int64)).shape == (0, n ** 3)


def test_more_units_than_ctas():
    """4,096 units over at most 592 CTAs (grid-stride over the scratch slices): Θ Θᵀ-free check — the rows of the
    unitary-equivalent identity operator are the unit vectors."""
    n, J = 16, 2
    h = daubechies(2)
    N = n ** 3
    u = np.zeros((1, N))
    u[0, 0] = 1.0
    v = np.ones((1, N))
    got = pcwd.rows3d(n, J, h, torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda(), np.arange(N))
    assert torch.allclose(got, torch.eye(N, dtype=torch.float64, device="cuda"), atol=1e-12)


def test_errors():
    n, J = 8, 2
    h = daubechies(2)
    u, v = volume_problem(n, 1, 1, 41)
    ud, vd = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
    for kwargs, code in ((dict(n=6), 1), (dict(levels=4), 2), (dict(h=h * 1.01), 2), (dict(units=np.array([n ** 3])), 3)):   # E_SHAPE / E_CONFIG / E_PARAM
        a = dict(n=n, levels=J, h=h, units=np.array([0]))
        a.update(kwargs)
        with pytest.raises(PcwdError) as ei:
            out = torch.empty((1, a["n"] ** 3), dtype=torch.float64, device="cuda")
            hh = np.ascontiguousarray(a["h"], dtype=np.float64)
            uu = np.ascontiguousarray(a["units"], dtype=np.int64)
            pcwd._check(pcwd.lib().pcwd_rows3d(a["n"], a["levels"], ctypes.c_void_p(hh.ctypes.data), len(hh), 1,
                                                ctypes.c_void_p(ud.data_ptr()), ctypes.c_void_p(vd.data_ptr()),
                                                ctypes.c_void_p(uu.ctypes.data), 1, ctypes.c_void_p(out.data_ptr()),
                                                ctypes.c_void_p(0)), "pcwd_rows3d")
        assert ei.value.code == code, (kwargs, str(ei.value))
