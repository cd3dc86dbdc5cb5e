"""GPU edge cases of the boundary (include/pcwd.h): shards with no units (world larger than the units a cost-balanced
split can hand out), a retained set with no entries (PATTERN rows all empty; THRESHOLD with τ_rel > 1 keeps nothing,
since |θ| ≤ M < τ), and the consumers on such an empty Θ (apply, apply ᵀ, FISTA).  Every decomposition that is
not empty is checked against the dense fp64 oracle on the same seeded inputs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import operator as op, retention as ret  # noqa: E402
from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from synth import configs as C  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_09870_b200 import _build
    _build.build()


def _spec(p, dtype, **kw):
    return Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(), dtype=dtype,
                retain=kw.pop("retain", p.retain), tau_rel=kw.pop("tau_rel", p.tau_rel),
                band_L=kw.pop("band_L", p.band_L), **kw)


@pytest.mark.parametrize("retain", ["full", "band", "threshold", "pattern"])
def test_more_ranks_than_shards_of_units(retain):
    """N = 32 units (1-D, n = 32) over 40 ranks: the cost-balanced split leaves at least 8 ranks with no unit.
    Every rank's create and decompose succeed on its (possibly empty) shard; the shards partition Λ and their CSR
    rows concatenate to the one-rank CSR bit for bit; the values match the oracle."""
    p = C.micro(32, 1, 4, 5, 2, 3, 301, retain="band" if retain == "pattern" else retain, tau_rel=1e-3,
                band_L=9)
    kw = {}
    if retain == "pattern":
        rp, col = C.random_pattern(p.N, 12, 302)
        kw = {"retain": "pattern", "pat_rowptr": rp, "pat_col": col}
    whole = Decomposition(_spec(p, "f64", **kw))
    if retain == "threshold":
        M = whole.local_max()
        whole.set_global_max(M)
    whole.decompose()
    ref = [t.numpy() for t in whole.csr(device="cpu")]
    world = 40
    rows, cols, vals, empty = [0], [], [], 0
    for r in range(world):
        d = Decomposition(_spec(p, "f64", rank=r, world=world, **kw))
        info = d.info()
        if retain == "threshold":
            d.set_global_max(M)       # the MAX all-reduce of the ranks' local maxima (C-a), here the known M
        d.decompose()
        rp_r, col_r, val_r = (t.numpy() for t in d.csr(device="cpu"))
        assert len(rp_r) == info.row1 - info.row0 + 1 and rp_r[0] == 0
        empty += info.row1 == info.row0
        rows.extend((rp_r[1:] + rows[-1]).tolist())
        cols.append(col_r)
        vals.append(val_r)
        d.close()
    assert empty >= world - p.N
    assert np.array_equal(np.array(rows), ref[0])
    assert np.array_equal(np.concatenate(cols), ref[1]) and np.array_equal(np.concatenate(vals), ref[2])
    T = op.theta_dense(p)
    rp, col, val = ref
    for mu in range(p.N):
        c = col[rp[mu]:rp[mu + 1]]
        assert np.max(np.abs(val[rp[mu]:rp[mu + 1]] - T[mu, c]), initial=0.0) <= 1e-12 * np.abs(T).max()
    whole.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_threshold_keeping_nothing(dtype):
    """τ_rel > 1: no entry satisfies |θ| ≥ τ_rel·M (M = max|θ|), so the CSR has no entries and every row is empty;
    apply and apply ᵀ of the empty Θ return zeros, and FISTA on it returns the prox of the zero gradient."""
    p = C.micro(16, 2, 4, 3, 2, 2, 303, retain="threshold", tau_rel=1.5)
    dec = Decomposition(_spec(p, dtype))
    dec.decompose()
    rp, col, val = (t.numpy() for t in dec.csr(device="cpu"))
    assert dec.info().nnz == 0 and len(col) == 0 and np.all(rp == 0) and len(rp) == p.N + 1
    tdt = torch.float64 if dtype == "f64" else torch.float32
    x = torch.ones(p.N, dtype=tdt, device="cuda")
    assert torch.count_nonzero(dec.apply(x)).item() == 0
    assert torch.count_nonzero(dec.apply(x, transpose=True)).item() == 0
    z, tau = dec.fista(x, torch.zeros_like(x), 5, tau=0.5)
    assert torch.count_nonzero(z).item() == 0      # y stays 0: the gradient Θᵀ(Θ·0 − z0) is 0 on an empty Θ
    dec.close()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_pattern_with_no_entries(dtype):
    """A PATTERN whose rows are all empty: a valid retained set with no entries."""
    p = C.micro(16, 2, 4, 3, 2, 2, 304, retain="band", band_L=4)
    rp = np.zeros(p.N + 1, dtype=np.int64)
    col = np.zeros(0, dtype=np.int32)
    dec = Decomposition(_spec(p, dtype, retain="pattern", pat_rowptr=rp, pat_col=col))
    dec.decompose()
    rp_g, col_g, val_g = (t.numpy() for t in dec.csr(device="cpu"))
    assert dec.info().nnz == 0 and len(col_g) == 0 and np.all(rp_g == 0)
    dec.close()


def test_band_single_unit_grid():
    """The smallest torus the ABI accepts in 1-D (n = 2, J = 1, Haar): two units, band L = N = 2 equals the full
    rule, both against the oracle."""
    p = C.micro(2, 1, 1, 1, 1, 0, 305, retain="full")
    T = op.theta_dense(p)
    for retain, L in (("full", 0), ("band", 2)):
        dec = Decomposition(_spec(p, "f64", retain=retain, band_L=L))
        dec.decompose()
        rp, col, val = (t.numpy() for t in dec.csr(device="cpu"))
        assert np.array_equal(rp, [0, 2, 4]) and np.array_equal(col, [0, 1, 0, 1])
        assert np.max(np.abs(val - T.ravel())) <= 1e-14 * max(np.abs(T).max(), 1e-300)
        if retain == "band":
            assert all(np.array_equal(ret.band_partners(p, mu, 2), [0, 1]) for mu in range(2))
        dec.close()
