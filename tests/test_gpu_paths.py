"""GPU: the alternative kernel paths (environment switches read once per process, so each runs in a
subprocess) give the same CSR as the default path on c3 and a 128² fp64 case: pattern bit-exact, values within
the fp32 / fp64 rounding of a different summation order.  The default path is the one the oracle parity tests
check; these keep the fallbacks (non-TMA k-sum, cp.async approximation steps, no tail, serial coarse levels,
no fine kernel, no direct partners, generic kernels) correct."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2005_09870_b200 import Decomposition, Spec
from synth import configs as C
name, dtype, out = sys.argv[1], sys.argv[2], sys.argv[3]
p = C.get(name) if name.startswith("c") else C.micro(128, 2, 4, 5, 3, 4, 45, retain="band", band_L=64)
dec = Decomposition(Spec(p.d, p.n, p.J, p.h, p.u, p.v, dtype=dtype, retain=p.retain, tau_rel=p.tau_rel,
                         band_L=p.band_L))
dec.decompose()
rp, col, val = (t.numpy() for t in dec.csr(device="cpu"))
np.savez(out, rp=rp, col=col, val=val.astype(np.float64))
"""

SWITCHES = [
    {"PCWD_NO_TMA_KSUM": "1"},
    {"PCWD_NO_TMA_APPROX": "1"},
    {"PCWD_NO_TAIL": "1"},
    {"PCWD_COARSE_SERIAL": "1"},
    {"PCWD_COARSE_OVERLAP": "0"},
    {"PCWD_OVERLAP_ALL": "0"},
    {"PCWD_GENERIC_SMEM_KB": "200"},
    {"PCWD_NO_FINE": "1"},
    {"PCWD_NO_DIRECT": "1"},
    {"PCWD_FINE_DIRECT": "1,1,1"},
    {"PCWD_NO_FINE": "1", "PCWD_NO_TILE": "1", "PCWD_NO_BATCHED": "1"},
    {"PCWD_SEP": "7"},
    {"PCWD_TAIL_NT": "128"},
    {"PCWD_TAIL_NT": "64"},
]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_09870_b200 import _build
    _build.build()


def _run(tmp_path, name, dtype, env):
    out = str(tmp_path / f"{name}_{dtype}_{abs(hash(tuple(sorted(env.items()))))}.npz")
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), name, dtype, out], env=e, check=True,
                   timeout=600)
    return np.load(out)


def test_threshold_recompute_matches_store_then_filter(tmp_path):
    """Threshold rule: the count / write passes recomputing the cascade (PCWD_NO_CAND) give the CSR the
    store-then-filter path gives (the same fp64 values, bit for bit)."""
    for name, dtype in (("c2", "f32"), ("c2", "f64")):
        ref = _run(tmp_path, name, dtype, {})
        got = _run(tmp_path, name, dtype, {"PCWD_NO_CAND": "1"})
        for k in ("rp", "col", "val"):
            assert np.array_equal(got[k], ref[k])


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_threshold_generic_smem_cap(tmp_path, dtype):
    """The threshold rule runs the generic unit kernel on every level: a 200 KB shared-memory cap moves the
    coarser levels of c2 from the global (L2) scratch into shared memory — the same fp64 arithmetic, so the
    same CSR bit for bit."""
    ref = _run(tmp_path, "c2", dtype, {})
    got = _run(tmp_path, "c2", dtype, {"PCWD_GENERIC_SMEM_KB": "200"})
    for k in ("rp", "col", "val"):
        assert np.array_equal(got[k], ref[k])


@pytest.mark.parametrize("case", [("c3", "f32"), ("micro128", "f64")], ids=["c3-f32", "128-f64"])
@pytest.mark.parametrize("env", SWITCHES, ids=["+".join(f"{k}={v}" for k, v in s.items()) for s in SWITCHES])
def test_switch_matches_default_path(tmp_path, case, env):
    name, dtype = case
    ref = _run(tmp_path, name, dtype, {})
    got = _run(tmp_path, name, dtype, env)
    assert np.array_equal(got["rp"], ref["rp"]) and np.array_equal(got["col"], ref["col"])
    err = np.linalg.norm(got["val"] - ref["val"]) / np.linalg.norm(ref["val"])
    assert err <= (2e-6 if dtype == "f32" else 1e-13), err


@pytest.mark.parametrize("env", [{"PCWD_NO_COMPACT": "1"}, {"PCWD_HYBRID_KB": "0"}, {"PCWD_HYBRID_KB": "200"}],
                         ids=["no-compact", "no-hybrid", "hybrid-200KB"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_threshold_filter_and_scratch_switches(tmp_path, env, dtype):
    """Threshold rule: the two-read filter (count pass + write pass, PCWD_NO_COMPACT) instead of the one-read
    in-place compaction + copy (fp32 values), and the generic kernel's step ≥ 2 buffers in global instead of shared
    memory (PCWD_HYBRID_KB=0) or a larger shared part: the same fp64 arithmetic and decisions, so the same CSR bit
    for bit."""
    ref = _run(tmp_path, "c2", dtype, {})
    got = _run(tmp_path, "c2", dtype, env)
    for k in ("rp", "col", "val"):
        assert np.array_equal(got[k], ref[k])
