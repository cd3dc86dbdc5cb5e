"""PATTERN retention (include/pcwd.h PCWD_RETAIN_PATTERN): the caller supplies the retained set as a CSR over
units — the A_L pattern of Theorem 2's Remark or any Θ_L of Eq. (7).
Parity against the dense oracle on every unit, bit-identity of the retained pattern, agreement with the BAND
rule when the pattern is the band pattern, shard invariance and argument checking."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import operator as op, retention as ret, rows as R  # noqa: E402
from paper_2005_09870_b200 import Decomposition, PcwdError, Spec  # noqa: E402
from paper_2005_09870_b200 import pcwd as PW  # noqa: E402
from synth import configs as C  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = {"f32": 1e-5, "f64": 1e-12}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_09870_b200 import _build
    _build.build()


def _run(p, dtype, rp, col, world=1, rank=0, device_pattern=False):
    if device_pattern:
        rp, col = torch.from_numpy(rp).cuda(), torch.from_numpy(col).cuda()
    dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(),
                             dtype=dtype, retain="pattern", pat_rowptr=rp, pat_col=col, rank=rank, world=world))
    dec.decompose()
    g = [t.numpy() for t in dec.csr(device="cpu")]
    info = dec.info()
    dec.close()
    return g, info


CASES = [  # n, d, M, J, m, R, seed, max partners per row
    (16, 2, 4, 3, 3, 2, 101, 40),     # DB4 with folded coarse lines
    (32, 2, 1, 5, 2, 2, 102, 64),     # Haar, full depth
    (64, 1, 4, 6, 2, 5, 103, 30),     # 1-D
    (16, 2, 2, 2, 2, -1, 104, 256),   # dense u (windows cover the torus), rows up to all of Λ
]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}d{c[1]}M{c[2]}J{c[3]}" for c in CASES])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_random_pattern_parity(case, dtype):
    n, d, M, J, m, Rr, seed, kmax = case
    p = C.micro(n, d, M, J, m, Rr, seed)
    rp, col = C.random_pattern(p.N, kmax, seed)
    p.retain, p.pat_rowptr, p.pat_col = "pattern", rp, col
    T = op.theta_dense(p)
    (grp, gcol, gval), info = _run(p, dtype, rp, col, device_pattern=(seed % 2 == 0))
    assert info.nnz == len(col)
    assert np.array_equal(grp, rp) and np.array_equal(gcol, col)       # the pattern is the caller's, bit for bit
    num = den = 0.0
    for mu in range(p.N):
        c, ref = ret.retained_row(p, mu, T[mu])
        v = gval[rp[mu]:rp[mu + 1]].astype(np.float64)
        num += float(np.sum((v - ref) ** 2))
        den += float(np.sum(ref ** 2))
    assert (num / den) ** 0.5 <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_band_pattern_equals_band_rule(dtype):
    """The oracle's band pattern given as PATTERN reproduces the BAND rule's CSR: the same columns, and values
    that agree to the rounding of two kernels (fp64: 1e-14 relative; fp32: the fp32 bar)."""
    p = C.micro(32, 2, 4, 4, 3, 3, 105, retain="band", band_L=64)
    pat = ret.band_pattern_dense(p, 64)
    rp = np.arange(p.N + 1, dtype=np.int64) * 64
    col = np.concatenate([pat[mu] for mu in range(p.N)]).astype(np.int32)
    (grp, gcol, gval), _ = _run(p, dtype, rp, col)
    dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(),
                             dtype=dtype, retain="band", band_L=64))
    dec.decompose()
    brp, bcol, bval = (t.numpy() for t in dec.csr(device="cpu"))
    dec.close()
    assert np.array_equal(gcol, bcol) and np.array_equal(grp, brp)
    rel = np.linalg.norm(gval.astype(np.float64) - bval) / np.linalg.norm(bval.astype(np.float64))
    assert rel <= (1e-14 if dtype == "f64" else TOL["f32"]), rel


def test_pattern_shards_concatenate():
    p = C.micro(32, 2, 4, 4, 3, 3, 106)
    rp, col = C.random_pattern(p.N, 50, 106)
    (frp, fcol, fval), _ = _run(p, "f32", rp, col)
    cols, vals, nxt = [], [], 0
    for r in range(3):
        (grp, gcol, gval), info = _run(p, "f32", rp, col, world=3, rank=r)
        assert info.row0 == nxt
        assert np.array_equal(grp, rp[info.row0:info.row1 + 1] - rp[info.row0])
        nxt = info.row1
        cols.append(gcol)
        vals.append(gval)
    assert nxt == p.N
    assert np.array_equal(np.concatenate(cols), fcol) and np.array_equal(np.concatenate(vals), fval)


def test_pattern_c3_sampled():
    """A random pattern on the c3 operator (256², DB4, J = 6, m = 8): sampled units against the oracle rows."""
    p = C.get("c3")
    rp, col = C.random_pattern(p.N, 96, 107, empty_every=0)
    q = C.Problem("c3pat", p.d, p.n, p.J, p.h, p.u, p.v, "pattern", pat_rowptr=rp, pat_col=col)
    (grp, gcol, gval), _ = _run(q, "f32", rp, col)
    units = sorted(set([0, 15, 16, 300, 1000, 4095, 4096, 20000, 40000, 65535]))
    rows = R.rows(q, units)
    num = den = 0.0
    for mu, row in zip(units, rows):
        c, ref = ret.retained_row(q, mu, row)
        num += float(np.sum((gval[rp[mu]:rp[mu + 1]] - ref) ** 2))
        den += float(np.sum(ref ** 2))
    assert (num / den) ** 0.5 <= TOL["f32"]


@pytest.mark.parametrize("bad", ["unsorted", "range", "rowptr"])
def test_invalid_pattern_rejected(bad):
    p = C.micro(16, 2, 2, 3, 1, 1, 108)
    rp, col = C.random_pattern(p.N, 8, 108)
    col = col.copy()
    rp = rp.copy()
    if bad == "unsorted":
        r = next(i for i in range(p.N) if rp[i + 1] - rp[i] >= 2)
        col[rp[r]], col[rp[r] + 1] = col[rp[r] + 1], col[rp[r]]
    elif bad == "range":
        col[-1] = p.N
    else:
        rp[5] = rp[6] + 1
    with pytest.raises(PcwdError) as e:
        _run(p, "f32", rp, col)
    assert e.value.code == 3
