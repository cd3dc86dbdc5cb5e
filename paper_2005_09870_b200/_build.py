"""Build libpcwd.so in-tree with nvcc for sm_100a (called by __graft_entry__.build()).

Each translation unit is compiled to an object in parallel, then linked into the shared library."""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpcwd.so")
OBJ = os.path.join(CSRC, "obj")
SOURCES = ["api.cu", "kernels.cu", "band_tile.cu", "batched.cu", "fine.cu", "fista.cu", "approx.cu", "pca.cu", "sort.cu", "volume.cu", "plan.cpp"]
HEADERS = ["common.h", "kernels.cuh", "plan.h", "geom.h", "tma.h"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]


def _deps():
    deps = [os.path.join(CSRC, f) for f in HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "pcwd.h"))
    deps.append(os.path.abspath(__file__))
    return deps


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps() + [os.path.join(CSRC, f) for f in SOURCES])


def _obj_stale(src: str, obj: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in _deps() + [src])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    os.makedirs(OBJ, exist_ok=True)
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ, s + ".o")
        if force or _obj_stale(src, obj):
            jobs.append([nvcc, *NVCC_FLAGS, "-c", src, "-o", obj])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        list(ex.map(run, jobs))
    link = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
            *[os.path.join(OBJ, s + ".o") for s in SOURCES], "-o", LIB + ".tmp"]
    run(link)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
