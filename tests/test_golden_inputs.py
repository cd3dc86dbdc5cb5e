"""The stored oracle results are tied to the inputs they were computed from: every golden JSON that names
an `inputs_sha256` must match the sha256 of the seeded inputs synth/ builds today (a changed recipe would
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
    if "inputs_sha256" not in g:
        pytest.skip("no inputs hash")
    assert C.get(g["config"]).sha256() == g["inputs_sha256"]
