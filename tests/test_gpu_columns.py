"""Algorithm 2's column orientation on the GPU (pcwd_columns: Θ[·][λ] = Ψ*(H ψ_λ); the fixed-λ
kernel of SURVEY §8(f) NEXT 4 / ledger C1): whole columns against the dense oracle on micro cases, and at c3 size the
entries (μ, λ) of the oracle's cached rows (the same number reached from the other orientation) plus per-column
Parseval Σ_μ Θ[μ][λ]² = ‖H ψ_λ‖² with H ψ_λ through the oracle's FFTs."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import basis, operator as op  # noqa: E402
from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from synth import configs as C  # noqa: E402

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_09870_b200 import _build
    _build.build()


def _handle(p, dtype="f64"):
    return Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(),
                              dtype=dtype, retain="band", band_L=min(16, p.N)))


CASES = [(16, 2, 4, 3, 3, 2, 81), (16, 2, 2, 4, 2, -1, 82), (64, 1, 4, 5, 3, 4, 83), (32, 2, 1, 5, 2, 3, 84)]


@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}d{c[1]}M{c[2]}J{c[3]}R{c[5]}" for c in CASES])
def test_all_columns_match_dense(case):
    n, d, M, J, m, R, seed = case
    p = C.micro(n, d, M, J, m, R, seed)
    T = op.theta_dense(p)
    dec = _handle(p)
    cols = dec.columns(np.arange(p.N)).cpu().numpy()            # row i = column i of Θ
    assert np.linalg.norm(cols.T - T) <= 1e-12 * np.linalg.norm(T)
    dec.close()


def test_c3_columns_against_cached_rows():
    path = os.path.join(HERE, "golden", "cache", "c3_band_rows.npz")
    if not os.path.exists(path):
        pytest.skip("c3 oracle cache missing")
    z = np.load(path)
    p = C.get("c3")
    assert p.fingerprint_matches(list(z["inputs_fingerprint"]))
    units, rp, col, val = z["units"], z["row_ptr"], z["col"], z["val"]
    rng = np.random.default_rng(0)
    picks = [(int(units[i]), int(col[rp[i] + j]), float(val[rp[i] + j]))
             for i in rng.choice(len(units), 24, replace=False) for j in rng.choice(rp[i + 1] - rp[i], 2, replace=False)]
    lam = sorted({lm for (_, lm, _) in picks})
    dec = _handle(p)
    cols = dec.columns(lam).cpu().numpy()
    dec.close()
    where = {lm: i for i, lm in enumerate(lam)}
    got = np.array([cols[where[lm], mu] for (mu, lm, _) in picks])
    ref = np.array([v for (_, _, v) in picks])
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    for lm in lam[:6]:                                           # Parseval per column against H ψ_λ by FFT
        e = np.zeros(p.N)
        e[lm] = 1.0
        hpsi = op.apply_fft(p, basis.inverse(e, p.d, p.n, p.J, p.h))
        assert abs(np.sum(cols[where[lm]] ** 2) - np.sum(hpsi ** 2)) <= 1e-12 * np.sum(hpsi ** 2)
