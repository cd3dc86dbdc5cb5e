"""Compute the global max M = max_{μ,λ} |Θ[μ][λ]| of config c4 with the ORACLE only.

The threshold rule of c4 keeps |θ| ≥ 1e-5·M (R15); M needs every unit.  This
script calls only oracle/ (and synth/ for the inputs) and writes
tests/golden/c4_global_max.json = {M, argmax unit, inputs sha256}.  Units are visited in
Λ order (coarse first) in chunks; a unit whose ‖H*ψ_μ‖₂ is below the running max is
skipped by the Parseval bound (oracle/rows.c).  Progress is checkpointed in /tmp.

Usage: python tools/c4_global_max.py [--threads T] [--config c4]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import rows as R  # noqa: E402
from synth import configs as C  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--config", default="c4")
    ap.add_argument("--chunk", type=int, default=2048)
    a = ap.parse_args()
    p = C.get(a.config)
    sha = p.sha256()
    ck = f"/tmp/{a.config}_gmax_{sha[:16]}.json"
    state = {"next": 0, "M": 0.0, "arg": -1}
    if os.path.exists(ck):
        state = json.load(open(ck))
    t0 = time.time()
    while state["next"] < p.N:
        lo = state["next"]
        hi = min(p.N, lo + (64 if lo < 4096 else a.chunk))
        rm = R.rowmax(p, np.arange(lo, hi), nthreads=a.threads, bound=state["M"])
        i = int(np.argmax(rm))
        if rm[i] > state["M"]:
            state["M"] = float(rm[i])
            state["arg"] = lo + i
        state["next"] = hi
        json.dump(state, open(ck, "w"))
        print(f"{hi}/{p.N} M={state['M']:.17g} arg={state['arg']} t={time.time()-t0:.0f}s", flush=True)
    out = {"config": a.config, "M": state["M"], "argmax_unit": state["arg"], "inputs_sha256": sha,
           "inputs_fingerprint": p.fingerprint(),
           "how": "oracle/rows.c over all units, Parseval-pruned (tools/c4_global_max.py)"}
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    json.dump(out, open(os.path.join(here, "tests", "golden", f"{a.config}_global_max.json"), "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()
