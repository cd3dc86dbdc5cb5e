import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def root():
    return ROOT


def record_parity(name: str, dtype: str, err: float, units: int, **extra):
    """Append a measured parity error (relative Frobenius over the retained entries of the compared units) to
    gpurun_out/parity_errors.jsonl, so the achieved errors of every GPU run are kept next to the pass/fail bar
    (copied to profiles/ per round)."""
    import json
    import time
    d = os.path.join(ROOT, "gpurun_out")
    os.makedirs(d, exist_ok=True)
    rec = {"test": name, "dtype": dtype, "rel_frobenius": float(err), "units": int(units), "time": time.time()}
    rec.update(extra)
    with open(os.path.join(d, "parity_errors.jsonl"), "a") as f:
        f.write(json.dumps(rec) + "\n")
