"""GPU: the separable direct form of the fine kernel's a3 + a4 (geom.h "sep", switched on by PCWD_SEP, a bit
mask over fine levels 1..3) against the fp64 oracle.  The switch is read once per process, so the oracle parity
tests of test_gpu_parity.py that exercise the fine kernel — every fine class and seam unit of c3 and c5 (f32 and
f64), all 16,384 units of a 128² L = 128 case, the micro cases, c3 / c5 band — run again in a subprocess with every
fine level on the separable path."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_sep_path_oracle_parity():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ)
    env["PCWD_SEP"] = "7"
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-m", "gpu",
                        "-x", "-q", "-p", "no:cacheprovider", "-k",
                        "micro or c3_band or c5_band_fp32 or fine_kernel or every_fine or all_units_128 or symlet"],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
