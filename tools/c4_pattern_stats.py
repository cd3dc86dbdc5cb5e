"""All-unit retained-pattern statistics of a threshold config (c4) with the ORACLE only.

For every unit μ of the config: the number of retained entries |Θ[μ][λ]| ≥ τ = τ_rel·M, an FNV-1a
hash of the retained column list, Σθ², a ±1 sketch Σθ·s(λ) and max|Θ[μ][·]| (oracle/rows.c
oracle_row_stats).  M comes from tests/golden/<config>_global_max.json (itself oracle-only).  The
GPU test compares every GPU row against these (count and hash: bit-exact pattern; sketch: an
unbiased estimate of the Frobenius error over all units, since E[(Σ s_i e_i)²] = Σ e_i²).

This script calls only oracle/ (and synth/ for the inputs).  Progress is checkpointed in /tmp.
Output: tests/golden/<config>_pattern_stats.npz (+ a JSON summary beside it).

Usage: python tools/c4_pattern_stats.py [--threads T] [--config c4]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import rows as R  # noqa: E402
from synth import configs as C  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--config", default="c4")
    ap.add_argument("--chunk", type=int, default=4096)
    a = ap.parse_args()
    p = C.get(a.config)
    sha = p.sha256()
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"{a.config}_global_max.json")))
    assert gold["inputs_sha256"] == sha, "inputs changed since the global max was computed"
    M = gold["M"]
    tau = p.tau_rel * M
    ck = f"/tmp/{a.config}_stats_{sha[:16]}.npz"
    keys = ("cnt", "hash", "ssq", "sketch", "rmax", "near")
    if os.path.exists(ck):
        z = np.load(ck)
        st = {k: z[k] for k in keys}
        nxt = int(z["next"])
    else:
        st = dict(cnt=np.zeros(p.N, np.int64), hash=np.zeros(p.N, np.uint32), ssq=np.zeros(p.N),
                  sketch=np.zeros(p.N), rmax=np.zeros(p.N), near=np.zeros(p.N, np.int64))
        nxt = 0
    t0 = time.time()
    while nxt < p.N:
        hi = min(p.N, nxt + (64 if nxt < 4096 else a.chunk))
        s = R.row_stats(p, np.arange(nxt, hi), tau, nthreads=a.threads)
        for k in keys:
            st[k][nxt:hi] = s[k]
        nxt = hi
        np.savez(ck, next=nxt, **st)
        print(f"{nxt}/{p.N} nnz so far {int(st['cnt'][:nxt].sum())} t={time.time() - t0:.0f}s", flush=True)
    out = os.path.join(ROOT, "tests", "golden", f"{a.config}_pattern_stats.npz")
    np.savez_compressed(out, cnt=st["cnt"].astype(np.int32), hash=st["hash"], sketch=st["sketch"],
                        ssq=st["ssq"], rmax=st["rmax"].astype(np.float64))
    summ = {"config": a.config, "inputs_sha256": sha, "inputs_fingerprint": p.fingerprint(), "M": M, "tau": tau, "nnz": int(st["cnt"].sum()),
            "max_per_unit": int(st["cnt"].max()), "near_tau": int(st["near"].sum()),
            "max_rowmax": float(st["rmax"].max()), "argmax_unit": int(np.argmax(st["rmax"])),
            "how": "oracle/rows.c oracle_row_stats over all units (tools/c4_pattern_stats.py)"}
    json.dump(summ, open(out.replace(".npz", ".json"), "w"), indent=1)
    print(summ)


if __name__ == "__main__":
    main()
