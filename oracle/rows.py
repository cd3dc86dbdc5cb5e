"""ORACLE (test infrastructure) — ctypes wrapper around oracle/rows.c (plain fp64 C).

rows(p, units) returns the full fp64 rows Θ[μ][·] = Ψ*(H* ψ_μ) of the requested units;
rowmax(p, units) returns max_λ |Θ[μ][λ]| per unit (used for the global max M of the
threshold rule).  See rows.c's header for the passages followed.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rows.c")
_LIB = os.path.join(_HERE, "liboracle_rows.so")
_lib = None


class _Problem(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int), ("n", ctypes.c_int), ("J", ctypes.c_int), ("L", ctypes.c_int),
                ("h", ctypes.POINTER(ctypes.c_double)), ("m", ctypes.c_int),
                ("u", ctypes.POINTER(ctypes.c_double)), ("v", ctypes.POINTER(ctypes.c_double))]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_rows.restype = ctypes.c_int
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _run(p, units, want_rows: bool, nthreads: int | None, bound: float = 0.0):
    lib = _load()
    h = np.ascontiguousarray(p.h, dtype=np.float64)
    u = np.ascontiguousarray(p.u, dtype=np.float64)
    v = np.ascontiguousarray(p.v, dtype=np.float64)
    units = np.ascontiguousarray(np.asarray(units, dtype=np.int64))
    prob = _Problem(p.d, p.n, p.J, len(h), _ptr(h), p.m, _ptr(u), _ptr(v))
    cnt = len(units)
    rows = np.zeros((cnt, p.N)) if want_rows else None
    rmax = np.zeros(cnt)
    nt = nthreads or os.cpu_count() or 1
    rc = lib.oracle_rows(ctypes.byref(prob), units.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                         ctypes.c_int64(cnt), _ptr(rows) if want_rows else None, _ptr(rmax),
                         ctypes.c_int(nt), ctypes.c_double(bound))
    if rc != 0:
        raise MemoryError("oracle_rows failed")
    return rows, rmax


def rows(p, units, nthreads: int | None = None) -> np.ndarray:
    return _run(p, units, True, nthreads)[0]


def rowmax(p, units, nthreads: int | None = None, bound: float = 0.0) -> np.ndarray:
    """max_λ |Θ[μ][λ]| per unit; with bound > 0, units that provably hold no entry ≥ bound
    (Parseval) return -‖Θ[μ][·]‖₂ instead (see rows.c)."""
    return _run(p, units, False, nthreads, bound)[1]


def row_stats(p, units, tau: float, nthreads: int | None = None) -> dict:
    """Per-unit statistics of the row retained at the absolute threshold tau (|θ| ≥ tau, reading
    R15), from the oracle's own fp64 rows (rows.c oracle_row_stats): cnt, hash (FNV-1a 32 over the
    retained λ as int32 little-endian), ssq (Σ θ²), sketch (Σ θ·s(λ), s = ±1 from splitmix64),
    rmax (max|Θ[μ][·]|, or −‖H*ψ_μ‖₂ for units skipped by the Parseval bound), near (entries within
    1e-12·tau of tau)."""
    lib = _load()
    lib.oracle_row_stats.restype = ctypes.c_int
    h = np.ascontiguousarray(p.h, dtype=np.float64)
    u = np.ascontiguousarray(p.u, dtype=np.float64)
    v = np.ascontiguousarray(p.v, dtype=np.float64)
    units = np.ascontiguousarray(np.asarray(units, dtype=np.int64))
    prob = _Problem(p.d, p.n, p.J, len(h), _ptr(h), p.m, _ptr(u), _ptr(v))
    c = len(units)
    out = dict(cnt=np.zeros(c, np.int64), hash=np.zeros(c, np.uint32), ssq=np.zeros(c), sketch=np.zeros(c),
               rmax=np.zeros(c), near=np.zeros(c, np.int64))
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    rc = lib.oracle_row_stats(ctypes.byref(prob), P(units), ctypes.c_int64(c), ctypes.c_double(tau),
                              P(out["cnt"]), P(out["hash"]), P(out["ssq"]), P(out["sketch"]), P(out["rmax"]),
                              P(out["near"]), ctypes.c_int(nthreads or os.cpu_count() or 1))
    if rc != 0:
        raise MemoryError("oracle_row_stats failed")
    return out
