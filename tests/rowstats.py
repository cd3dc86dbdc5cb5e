"""Per-row statistics of a CSR in numpy, mirroring oracle/rows.c oracle_row_stats's bookkeeping (count, FNV-1a 32
hash of the column list as little-endian int32, ±1 sketch Σ θ·s(λ) with s from the top bit of splitmix64(λ)).
Test-side bookkeeping only: no arithmetic of the method."""
import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64_sign(col: np.ndarray) -> np.ndarray:
    x = col.astype(np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return np.where((x >> np.uint64(63)) != 0, -1.0, 1.0)


def row_stats(rp: np.ndarray, col: np.ndarray, val: np.ndarray):
    rows = len(rp) - 1
    cnt = np.diff(rp).astype(np.int64)
    h = np.full(rows, 2166136261, dtype=np.uint64)
    cu = col.astype(np.uint64)
    maxlen = int(cnt.max()) if rows else 0
    for j in range(maxlen):
        act = np.nonzero(cnt > j)[0]
        c = cu[rp[act] + j]
        hh = h[act]
        for b in range(4):
            hh = ((hh ^ ((c >> np.uint64(8 * b)) & np.uint64(0xFF))) * np.uint64(16777619)) & np.uint64(0xFFFFFFFF)
        h[act] = hh
    sk = np.zeros(rows)
    np.add.at(sk, np.repeat(np.arange(rows), cnt), val.astype(np.float64) * splitmix64_sign(col))
    return cnt, h.astype(np.uint32), sk
