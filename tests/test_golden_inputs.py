"""The stored oracle results are tied to the inputs they were computed from: every golden JSON / cache must match
the fingerprint of the seeded inputs synth/ builds today (a changed recipe would
otherwise silently compare the GPU against stale expected values)."""
import glob
import json
import os

import pytest

from synth import configs as C

HERE = os.path.dirname(os.path.abspath(__file__))
FILES = sorted(glob.glob(os.path.join(HERE, "golden", "*.json")))


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f) for f in FILES])
def test_golden_inputs_sha256(path):
    g = json.load(open(path))
    if "inputs_fingerprint" not in g:
        pytest.skip("no inputs fingerprint")
    # sha256 of the fp64 inputs is machine-dependent (LAPACK/BLAS/FFT last bits); the fingerprint is not
    assert C.get(g["config"]).fingerprint_matches(g["inputs_fingerprint"])


@pytest.mark.parametrize("cfg", ["c3", "c5"])
def test_cache_inputs_fingerprint(cfg):
    import numpy as np
    z = np.load(os.path.join(HERE, "golden", "cache", f"{cfg}_band_rows.npz"))
    assert C.get(cfg).fingerprint_matches(list(z["inputs_fingerprint"]))
