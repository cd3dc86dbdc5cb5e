"""Cache of ORACLE retained rows for the large band configs, keyed by the inputs' sha256.

For c5 (and c3) the GPU parity test compares units that cover every code path of the fine and
batched kernels: per fine sub-band (levels 1-3) one unit of every position class (p0 mod 4, p1 mod 4)
in the interior, plus units on row 0, row n_ℓ−1, column 0 and the last 8-unit round of a row for every
class of the other axis; per coarse sub-band (levels ≥ 4 and the scaling block) the seam units (corners,
edge midpoints) and two interior units, or every unit when the sub-band has ≤ 16.  The rows come from
oracle/rows.c, the retained columns from oracle/retention.py; nothing here touches the CUDA path.

Output: tests/golden/cache/<config>_band_rows.npz with units, row_ptr, col (int32), val (fp64) and the
inputs sha256.  Usage: python tools/oracle_cache.py --config c5 [--threads T]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import basis, retention as ret, rows as R  # noqa: E402
from synth import configs as C  # noqa: E402


def class_units(p, classes: int = 4, round_w: int = 8, seed: int = 0):
    rng = np.random.default_rng(seed)
    units = set()
    for (lev, e, off, nl) in basis.subbands(p.d, p.n, p.J):
        idx = lambda r, c: off + (r % nl) * nl + (c % nl)  # noqa: E731
        if lev <= 3 and e != 0 and nl >= 4 * classes:
            for a in range(classes):
                for b in range(classes):
                    r = classes * int(rng.integers(2, nl // classes - 2)) + a
                    c = classes * int(rng.integers(2, nl // classes - 2)) + b
                    units.add(idx(r, c))
                # boundary rows / columns, every class of the other axis
                c = classes * int(rng.integers(1, nl // classes - 1)) + a
                units.add(idx(0, c))
                units.add(idx(nl - 1, c))
                r = classes * int(rng.integers(1, nl // classes - 1)) + a
                units.add(idx(r, 0))
                units.add(idx(r, nl - round_w + int(rng.integers(round_w))))
                units.add(idx(r, nl - 1 - a))
        elif nl * nl <= 16:
            units.update(off + i for i in range(nl * nl))
        else:
            h = nl // 2
            for (r, c) in [(0, 0), (0, nl - 1), (nl - 1, 0), (nl - 1, nl - 1), (0, h), (h, 0), (nl - 1, h),
                           (h, nl - 1)]:
                units.add(idx(r, c))
            for _ in range(2):
                units.add(idx(int(rng.integers(nl)), int(rng.integers(nl))))
    return np.array(sorted(units), dtype=np.int64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--chunk", type=int, default=32)
    a = ap.parse_args()
    p = C.get(a.config)
    assert p.retain == "band"
    units = class_units(p)
    print(f"{a.config}: {len(units)} units", flush=True)
    cols, vals, rp = [], [], [0]
    t0 = time.time()
    # coarse units (front of Λ) are the expensive ones: small chunks keep memory at chunk × N doubles
    for i in range(0, len(units), a.chunk):
        us = units[i:i + a.chunk]
        rows = R.rows(p, us, nthreads=a.threads)
        for mu, row in zip(us, rows):
            c, v = ret.retained_row(p, int(mu), row)
            cols.append(c.astype(np.int32))
            vals.append(v)
            rp.append(rp[-1] + len(c))
        print(f"{i + len(us)}/{len(units)} t={time.time() - t0:.0f}s", flush=True)
    os.makedirs(os.path.join(ROOT, "tests", "golden", "cache"), exist_ok=True)
    out = os.path.join(ROOT, "tests", "golden", "cache", f"{a.config}_band_rows.npz")
    np.savez_compressed(out, units=units, row_ptr=np.array(rp, dtype=np.int64), col=np.concatenate(cols),
                        val=np.concatenate(vals), inputs_sha256=np.array(p.sha256()),
                        inputs_fingerprint=np.array(p.fingerprint()),
                        how=np.array("oracle/rows.c + oracle/retention.py (tools/oracle_cache.py)"))
    print("wrote", out)


if __name__ == "__main__":
    main()
