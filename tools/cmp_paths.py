"""Compare the CSR of the default path with a reference path selected by env (debug tool).
python tools/cmp_paths.py c5 PCWD_NO_FINE   -> runs twice (in subprocesses) and compares."""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run_one(name, dtype, out):
    import torch
    from paper_2005_09870_b200 import Decomposition, Spec
    from synth import configs as C
    p = C.get(name) if name.startswith("c") else C.micro(*eval(name))
    dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(),
                             dtype=dtype, retain=p.retain, tau_rel=p.tau_rel, band_L=p.band_L))
    dec.decompose()
    rp, col, val = (t.numpy() for t in dec.csr(device="cpu"))
    np.savez(out, rp=rp, col=col, val=val)


if __name__ == "__main__":
    if sys.argv[1] == "--one":
        run_one(sys.argv[2], sys.argv[3], sys.argv[4])
        sys.exit(0)
    name, envvar = sys.argv[1], sys.argv[2]
    dtype = sys.argv[3] if len(sys.argv) > 3 else "f32"
    a, b = "/tmp/cmp_a.npz", "/tmp/cmp_b.npz"
    subprocess.check_call([sys.executable, __file__, "--one", name, dtype, a])
    env = dict(os.environ)
    env[envvar] = "1"
    subprocess.check_call([sys.executable, __file__, "--one", name, dtype, b], env=env)
    A, B = np.load(a), np.load(b)
    print("rowptr equal", np.array_equal(A["rp"], B["rp"]), "col equal", np.array_equal(A["col"], B["col"]))
    d = np.abs(A["val"].astype(np.float64) - B["val"].astype(np.float64))
    print("max |diff|", d.max(), "max |val|", np.abs(B["val"]).max(), "rel fro",
          np.linalg.norm(d) / np.linalg.norm(B["val"].astype(np.float64)))
    bad = np.nonzero(d > 1e-4 * np.abs(B["val"]).max())[0]
    print("bad entries", len(bad), "first rows", np.unique(np.searchsorted(A["rp"], bad[:50], side="right") - 1)[:20])
    colbad = np.nonzero(A["col"] != B["col"])[0]
    print("col mismatches", len(colbad), "rows", np.unique(np.searchsorted(A["rp"], colbad[:50], side="right") - 1)[:20])
