"""Thin ctypes binding of libpcwd.so (include/pcwd.h) — argument marshalling only.

Every step of the decomposition runs in the library's CUDA kernels; this module only
passes pointers and sizes, allocates the torch tensors that receive copies of the CSR,
and (for multi-process runs) does the one MAX all-reduce of the threshold rule through
torch.distributed.  There is no CPU fallback: if the library is missing, loading fails.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpcwd.so")

PCWD_F32, PCWD_F64 = 0, 1
RETAIN = {"full": 0, "threshold": 1, "band": 2, "pattern": 3}
STATUS = {0: "OK", 1: "E_SHAPE", 2: "E_CONFIG", 3: "E_PARAM", 4: "E_CUDA", 5: "E_OOM", 6: "E_STATE",
          7: "E_UNSUPPORTED"}


class PcwdError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS.get(code, code)}: {msg}")
        self.code = code


class Desc(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("n", ctypes.c_int32), ("levels", ctypes.c_int32),
                ("filter_len", ctypes.c_int32), ("h", ctypes.c_void_p), ("m", ctypes.c_int32),
                ("u", ctypes.c_void_p), ("v", ctypes.c_void_p), ("dtype", ctypes.c_int32),
                ("retain", ctypes.c_int32), ("tau_rel", ctypes.c_double), ("band_L", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("pat_rowptr", ctypes.c_void_p), ("pat_col", ctypes.c_void_p)]


class Csr(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("row0", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col", ctypes.c_void_p), ("val", ctypes.c_void_p),
                ("dtype", ctypes.c_int32)]


class Info(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("row0", ctypes.c_int64), ("row1", ctypes.c_int64),
                ("nnz", ctypes.c_int64), ("global_max", ctypes.c_double),
                ("fma_algorithmic", ctypes.c_double), ("bytes_algorithmic", ctypes.c_double),
                ("kernel_launches", ctypes.c_int32), ("compute_dtype", ctypes.c_int32)]


class ApproxInfo(ctypes.Structure):
    _fields_ = [("eta", ctypes.c_double), ("m", ctypes.c_int32), ("S", ctypes.c_int32 * 64),
                ("eps", ctypes.c_double * 64), ("bound", ctypes.c_double * 64), ("nnz", ctypes.c_int64)]


EXPORTS = ["pcwd_create", "pcwd_decompose", "pcwd_local_max", "pcwd_set_global_max", "pcwd_get_csr",
           "pcwd_copy_csr", "pcwd_apply", "pcwd_info", "pcwd_destroy", "pcwd_error_string",
           "pcwd_last_error", "pcwd_validate", "pcwd_plan_shard", "pcwd_plan_stencil",
           "pcwd_plan_num_subbands", "pcwd_profile", "pcwd_phase_times", "pcwd_launch_profile",
           "pcwd_set_kernels", "pcwd_decompose_to_host", "pcwd_wavelet_transform", "pcwd_fista",
           "pcwd_fista_sharded", "pcwd_approx", "pcwd_operator_apply", "pcwd_pc_from_samples", "pcwd_pc_from_svir", "pcwd_columns",
           "pcwd_plan_atom", "pcwd_kernel_box", "pcwd_set_kernels_box", "pcwd_rows3d"]

REDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int, ctypes.c_void_p)   # pcwd_reduce_fn
_lib = None


def lib():
    """Load libpcwd.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64p, i32p = ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32)
        L.pcwd_create.argtypes = [ctypes.POINTER(Desc), ctypes.POINTER(vp)]
        L.pcwd_decompose.argtypes = [vp, vp]
        L.pcwd_local_max.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_double)]
        L.pcwd_set_global_max.argtypes = [vp, ctypes.c_double]
        L.pcwd_get_csr.argtypes = [vp, ctypes.POINTER(Csr)]
        L.pcwd_copy_csr.argtypes = [vp, vp, vp, vp, vp]
        L.pcwd_apply.argtypes = [vp, vp, vp, ctypes.c_int, vp]
        L.pcwd_info.argtypes = [vp, ctypes.POINTER(Info)]
        L.pcwd_destroy.argtypes = [vp]
        L.pcwd_error_string.restype = ctypes.c_char_p
        L.pcwd_error_string.argtypes = [ctypes.c_int]
        L.pcwd_last_error.restype = ctypes.c_char_p
        L.pcwd_validate.argtypes = [ctypes.POINTER(Desc)]
        L.pcwd_plan_shard.argtypes = [ctypes.POINTER(Desc), i64p, i64p]
        L.pcwd_plan_stencil.argtypes = [ctypes.POINTER(Desc), i32, i32p, i32p, i32p]
        L.pcwd_plan_num_subbands.argtypes = [ctypes.POINTER(Desc), i32p]
        L.pcwd_plan_atom.argtypes = [ctypes.POINTER(Desc), i32, i32, ctypes.POINTER(ctypes.c_double), i32, i32p, i32p]
        L.pcwd_profile.argtypes = [vp, ctypes.c_int]
        L.pcwd_phase_times.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        dp = ctypes.POINTER(ctypes.c_double)
        L.pcwd_launch_profile.argtypes = [vp, ctypes.c_int, i32p, dp, dp, i32p, i32p]
        L.pcwd_set_kernels.argtypes = [vp, vp, vp, vp]
        L.pcwd_set_kernels_box.argtypes = [vp, vp, vp, vp]
        L.pcwd_kernel_box.argtypes = [vp, i32p, i32p]
        L.pcwd_decompose_to_host.argtypes = [vp, vp, vp, vp, vp]
        L.pcwd_wavelet_transform.argtypes = [vp, vp, vp, ctypes.c_int, vp]
        L.pcwd_fista.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double), vp, vp]
        L.pcwd_fista_sharded.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double), vp,
                                         REDUCE_FN, vp, vp, vp, vp]
        L.pcwd_approx.argtypes = [vp, ctypes.c_double, ctypes.c_int, vp, ctypes.POINTER(ApproxInfo)]
        L.pcwd_operator_apply.argtypes = [vp, vp, vp, ctypes.c_int, vp]
        L.pcwd_pc_from_samples.argtypes = [i32, i32, i32, i32, i32, vp, vp, vp, vp, vp]
        L.pcwd_columns.argtypes = [vp, vp, ctypes.c_int64, vp, vp]
        L.pcwd_pc_from_svir.argtypes = [i32, i32, i32, i32, vp, i32, i32, ctypes.c_uint64, vp, vp, vp, vp]
        L.pcwd_rows3d.argtypes = [i32, i32, vp, i32, i32, vp, vp, vp, ctypes.c_int64, vp, vp]
        for f in EXPORTS:
            getattr(L, f)  # every declared symbol must exist
        _lib = L
    return _lib


def _check(rc: int, where: str):
    if rc != 0:
        raise PcwdError(rc, where, lib().pcwd_last_error().decode())


def _ptr(a) -> int:
    """Address of a contiguous numpy array or torch tensor."""
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    assert a.is_contiguous()
    return a.data_ptr()


@dataclass
class Spec:
    """The problem statement of the ABI (R2-R16)."""
    d: int
    n: int
    levels: int
    h: np.ndarray
    u: object            # (m, N) fp64 numpy array (host) or torch.float64 CUDA tensor
    v: object
    dtype: str = "f32"   # "f32" | "f64"
    retain: str = "band"
    tau_rel: float = 0.0
    band_L: int = 0
    rank: int = 0
    world: int = 1
    device: int = 0
    pat_rowptr: object = None   # PATTERN: int64 (N+1) and int32 (nnz) CSR over all units (numpy or CUDA tensor)
    pat_col: object = None


def make_desc(s: Spec, keep: list) -> Desc:
    h = np.ascontiguousarray(np.asarray(s.h, dtype=np.float64))
    keep.append(h)
    rp, pc = s.pat_rowptr, s.pat_col
    if isinstance(rp, np.ndarray):
        rp = np.ascontiguousarray(rp, dtype=np.int64)
    if isinstance(pc, np.ndarray):
        pc = np.ascontiguousarray(pc, dtype=np.int32)
    for a in (s.u, s.v, rp, pc):
        keep.append(a)
    m = int(s.u.shape[0])
    return Desc(s.d, s.n, s.levels, len(h), _ptr(h), m, _ptr(s.u), _ptr(s.v),
                PCWD_F64 if s.dtype == "f64" else PCWD_F32, RETAIN[s.retain], float(s.tau_rel),
                int(s.band_L), s.rank, s.world, s.device, _ptr(rp), _ptr(pc))


class Decomposition:
    """One handle: the shard of units (rank, world) of Θ = Ψ* H Ψ for the given operator."""

    def __init__(self, spec: Spec):
        self.spec = spec
        self._keep = []
        self._desc = make_desc(spec, self._keep)
        h = ctypes.c_void_p()
        _check(lib().pcwd_create(ctypes.byref(self._desc), ctypes.byref(h)), "pcwd_create")
        self._h = h

    # -- compute ------------------------------------------------------------------------
    def decompose(self, stream: int = 0):
        _check(lib().pcwd_decompose(self._h, ctypes.c_void_p(stream)), "pcwd_decompose")

    def set_kernels(self, u, v, stream: int = 0):
        """New operator kernels (u_k, v_k) on this handle's plan (pcwd_set_kernels): (m, N) fp64,
        host (pinned for overlap) or CUDA; supp u_k must stay inside the box the plan was built for."""
        self._keep = (u, v)
        _check(lib().pcwd_set_kernels(self._h, ctypes.c_void_p(_ptr(u)), ctypes.c_void_p(_ptr(v)),
                                      ctypes.c_void_p(stream)), "pcwd_set_kernels")

    def kernel_box(self):
        """(lo, w): the periodic bounding box of supp u_k the plan was built from (pcwd_kernel_box), per axis."""
        lo, w = (ctypes.c_int32 * 2)(), (ctypes.c_int32 * 2)()
        _check(lib().pcwd_kernel_box(self._h, lo, w), "pcwd_kernel_box")
        return (lo[0], lo[1]), (w[0], w[1])

    def set_kernels_box(self, u_box, v, stream: int = 0):
        """pcwd_set_kernels_box: u_k given on the plan's box only, (m, w0, w1) fp64 (see kernel_box()), v (m, N)."""
        self._keep = (u_box, v)
        _check(lib().pcwd_set_kernels_box(self._h, ctypes.c_void_p(_ptr(u_box)), ctypes.c_void_p(_ptr(v)),
                                          ctypes.c_void_p(stream)), "pcwd_set_kernels_box")

    def decompose_to_host(self, row_ptr, col, val, stream: int = 0):
        """Decompose with the CSR streamed into the given (pinned host) buffers as launches finish
        (pcwd_decompose_to_host); complete once `stream` is synchronised."""
        _check(lib().pcwd_decompose_to_host(self._h, ctypes.c_void_p(_ptr(row_ptr)), ctypes.c_void_p(_ptr(col)),
                                            ctypes.c_void_p(_ptr(val)), ctypes.c_void_p(stream)),
               "pcwd_decompose_to_host")

    def wavelet_transform(self, x, inverse: bool = False, stream: int = 0):
        """Ψ* x (or Ψ x) on this handle's grid: x a CUDA tensor of N values of the handle's dtype."""
        import torch
        out = torch.empty_like(x)
        _check(lib().pcwd_wavelet_transform(self._h, ctypes.c_void_p(_ptr(x)), ctypes.c_void_p(_ptr(out)),
                                            int(inverse), ctypes.c_void_p(stream)), "pcwd_wavelet_transform")
        return out

    def fista(self, z0, w, iters: int, precond: bool = False, tau: float = 0.0, stream: int = 0):
        """FISTA-W (precond=False) / FISTA-WP on the decomposed Θ_L (pcwd_fista); returns (z, τ)."""
        import torch
        z = torch.empty_like(z0)
        t = ctypes.c_double(tau)
        _check(lib().pcwd_fista(self._h, ctypes.c_void_p(_ptr(z0)), ctypes.c_void_p(_ptr(w)), int(iters), int(precond),
                                ctypes.byref(t), ctypes.c_void_p(_ptr(z)), ctypes.c_void_p(stream)), "pcwd_fista")
        return z, t.value

    def fista_sharded(self, z0, w, iters: int, reduce, precond: bool = False, tau: float = 0.0, stream: int = 0):
        """FISTA over this handle's rows of a row-sharded Θ_L (pcwd_fista_sharded); returns (z, τ).
        reduce(which, buf) must sum the CUDA tensor buf over the ranks in place, ordered on `stream` (which = 0:
        the gradient, N values of the handle's dtype; 1: the Jacobi column sums, N fp64)."""
        import torch
        z = torch.empty_like(z0)
        xg = torch.empty_like(z0)
        xd = torch.empty(z0.numel(), dtype=torch.float64, device=z0.device)
        err = []

        def cb(which, _ctx):
            try:
                reduce(int(which), xg if which == 0 else xd)
                return 0
            except Exception as e:   # reported through the library's return code
                err.append(e)
                return 1
        fn = REDUCE_FN(cb)
        t = ctypes.c_double(tau)
        rc = lib().pcwd_fista_sharded(self._h, ctypes.c_void_p(_ptr(z0)), ctypes.c_void_p(_ptr(w)), int(iters),
                                      int(precond), ctypes.byref(t), ctypes.c_void_p(_ptr(z)), fn, None,
                                      ctypes.c_void_p(_ptr(xg)), ctypes.c_void_p(_ptr(xd)), ctypes.c_void_p(stream))
        if err:
            raise err[0]
        _check(rc, "pcwd_fista_sharded")
        return z, t.value

    def approx(self, eta: float, rule: str = "index", stream: int = 0) -> dict:
        """Algorithm 1's η-approximation Θ̃ into this handle's CSR (pcwd_approx); rule "index" (the Remark's (i)/(ii))
        or "magnitude" (power-of-two thresholds); returns the per-k truncation."""
        inf = ApproxInfo()
        _check(lib().pcwd_approx(self._h, ctypes.c_double(eta), {"index": 0, "magnitude": 1}[rule],
                                 ctypes.c_void_p(stream), ctypes.byref(inf)), "pcwd_approx")
        m = inf.m
        return {"eta": inf.eta, "S": list(inf.S[:m]), "eps": list(inf.eps[:m]), "bound": list(inf.bound[:m]),
                "nnz": inf.nnz}

    def columns(self, lambdas, stream: int = 0):
        """Algorithm 2's columns Θ[·][λ] (pcwd_columns) for the given Λ indices: a (count, N) fp64 CUDA tensor."""
        import torch
        lam = np.ascontiguousarray(np.asarray(lambdas, dtype=np.int64))
        out = torch.empty((len(lam), int(self.info().N)), dtype=torch.float64,
                          device=torch.device("cuda", self.spec.device))
        _check(lib().pcwd_columns(self._h, ctypes.c_void_p(_ptr(lam)), ctypes.c_int64(len(lam)),
                                  ctypes.c_void_p(_ptr(out)), ctypes.c_void_p(stream)), "pcwd_columns")
        return out

    def operator_apply(self, x, adjoint: bool = False, stream: int = 0):
        """H x (or H* x) on the device (pcwd_operator_apply): x a CUDA tensor of N values of the handle's dtype."""
        import torch
        y = torch.empty_like(x)
        _check(lib().pcwd_operator_apply(self._h, ctypes.c_void_p(_ptr(x)), ctypes.c_void_p(_ptr(y)), int(adjoint),
                                         ctypes.c_void_p(stream)), "pcwd_operator_apply")
        return y

    def local_max(self, stream: int = 0) -> float:
        out = ctypes.c_double()
        _check(lib().pcwd_local_max(self._h, ctypes.c_void_p(stream), ctypes.byref(out)), "pcwd_local_max")
        return out.value

    def set_global_max(self, M: float):
        _check(lib().pcwd_set_global_max(self._h, ctypes.c_double(M)), "pcwd_set_global_max")

    def decompose_distributed(self, stream: int = 0):
        """Multi-process decompose: the threshold rule's one exchange is a MAX all-reduce of
        the per-rank maxima (torch.distributed, NCCL on GPUs); band/full need none."""
        if self.spec.retain == "threshold" and self.spec.world > 1:
            self.set_global_max(allreduce_max(self.local_max(stream), self.spec.device))
        self.decompose(stream)
        if self.spec.world > 1:   # C-b: where this shard's entries start in the global CSR
            self.row_offsets = global_row_offsets(self.info().nnz, self.spec.device)
        else:
            self.row_offsets = [0, self.info().nnz]
        return self.row_offsets

    # -- results ------------------------------------------------------------------------
    def info(self) -> Info:
        out = Info()
        _check(lib().pcwd_info(self._h, ctypes.byref(out)), "pcwd_info")
        return out

    def profile(self, enable: bool = True):
        _check(lib().pcwd_profile(self._h, int(enable)), "pcwd_profile")

    def phase_times(self):
        """(ms[3], fma[3]) of the last decompose: templates, unit kernels, rest."""
        ms = (ctypes.c_double * 3)()
        fm = (ctypes.c_double * 3)()
        _check(lib().pcwd_phase_times(self._h, ms, fm), "pcwd_phase_times")
        return list(ms), list(fm)

    def launch_profile(self):
        """[(ms, algorithmic_fma, kind, level)] per unit-kernel launch of the last decompose."""
        cnt = ctypes.c_int32()
        _check(lib().pcwd_launch_profile(self._h, 0, ctypes.byref(cnt), None, None, None, None), "pcwd_launch_profile")
        n = cnt.value
        ms = (ctypes.c_double * n)()
        fm = (ctypes.c_double * n)()
        kd = (ctypes.c_int32 * n)()
        lv = (ctypes.c_int32 * n)()
        _check(lib().pcwd_launch_profile(self._h, n, ctypes.byref(cnt), ms, fm, kd, lv), "pcwd_launch_profile")
        kinds = {0: "generic", 1: "tile", 2: "fine", 3: "batched"}
        return [(ms[i], fm[i], kinds[kd[i]], lv[i]) for i in range(n)]

    def csr_meta(self) -> Csr:
        out = Csr()
        _check(lib().pcwd_get_csr(self._h, ctypes.byref(out)), "pcwd_get_csr")
        return out

    def csr(self, device: str = "cuda", stream: int = 0, pin: bool = False):
        """Copies of (row_ptr int64, col int32, val) as torch tensors on `device`."""
        import torch
        meta = self.csr_meta()
        vdt = torch.float64 if self.spec.dtype == "f64" else torch.float32
        kw = {"pin_memory": True} if (pin and device == "cpu") else {}
        if device != "cpu":
            kw = {"device": torch.device("cuda", self.spec.device)}
        rp = torch.empty(meta.n_rows + 1, dtype=torch.int64, **kw)
        col = torch.empty(meta.nnz, dtype=torch.int32, **kw)
        val = torch.empty(meta.nnz, dtype=vdt, **kw)
        _check(lib().pcwd_copy_csr(self._h, _ptr(rp), _ptr(col) if meta.nnz else 0, _ptr(val) if meta.nnz else 0,
                                   ctypes.c_void_p(stream)), "pcwd_copy_csr")
        if device == "cpu" or stream == 0:
            torch.cuda.synchronize(self.spec.device)
        return rp, col, val

    def apply(self, x, transpose: bool = False, stream: int = 0):
        """y = Θ_ret x (or Θ_retᵀ x) on the device, x a CUDA tensor of the value dtype."""
        import torch
        meta = self.csr_meta()
        n_out = meta.n_rows if not transpose else int(self.info().N)
        y = torch.empty(n_out, dtype=x.dtype, device=x.device)
        _check(lib().pcwd_apply(self._h, _ptr(x), _ptr(y), int(transpose), ctypes.c_void_p(stream)), "pcwd_apply")
        return y

    def close(self):
        if getattr(self, "_h", None):
            lib().pcwd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- multi-process plumbing (torch.distributed; NCCL on GPUs, gloo in the CPU tests) ----------

def allreduce_max(x: float, device: int = 0) -> float:
    """MAX over ranks of one fp64 scalar — the threshold rule's only exchange."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", device) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x: float, device: int = 0) -> float:
    """SUM over ranks of one fp64 scalar (e.g. retained entries of all shards)."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", device) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def _pc_out(m: int, N: int, device: int):
    import torch
    dev = torch.device("cuda", device)
    return (torch.empty((m, N), dtype=torch.float64, device=dev), torch.empty((m, N), dtype=torch.float64, device=dev),
            np.zeros(m))


def pc_from_samples(d: int, n: int, R: int, g: int, m: int, irs, device: int = 0, stream: int = 0):
    """§3.3.2 on the GPU (pcwd_pc_from_samples): (u, v) as (m, N) fp64 CUDA tensors and the singular values."""
    irs = np.ascontiguousarray(irs, dtype=np.float64) if isinstance(irs, np.ndarray) else irs
    u, v, sig = _pc_out(m, n ** d, device)
    _check(lib().pcwd_pc_from_samples(d, n, R, g, m, ctypes.c_void_p(_ptr(irs)), ctypes.c_void_p(_ptr(u)),
                                      ctypes.c_void_p(_ptr(v)), sig.ctypes.data_as(ctypes.c_void_p),
                                      ctypes.c_void_p(stream)), "pcwd_pc_from_samples")
    return u, v, sig


def pc_from_svir(d: int, n: int, R: int, m: int, svir, oversample: int = 8, power_iters: int = 16, seed: int = 1,
                 device: int = 0, stream: int = 0):
    """§3.3.3 on the GPU (pcwd_pc_from_svir): randomized SVD of the SVIR given at every pixel (N × W)."""
    svir = np.ascontiguousarray(svir, dtype=np.float64) if isinstance(svir, np.ndarray) else svir
    u, v, sig = _pc_out(m, n ** d, device)
    _check(lib().pcwd_pc_from_svir(d, n, R, m, ctypes.c_void_p(_ptr(svir)), oversample, power_iters,
                                   ctypes.c_uint64(seed), ctypes.c_void_p(_ptr(u)), ctypes.c_void_p(_ptr(v)),
                                   sig.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(stream)), "pcwd_pc_from_svir")
    return u, v, sig


def _coll_device(device: int = 0):
    import torch
    import torch.distributed as dist
    return torch.device("cuda", device) if dist.get_backend() == "nccl" else torch.device("cpu")


def allreduce_max_vec(x, device: int = 0) -> np.ndarray:
    """Element-wise MAX over ranks of a small fp64 vector (per-step times: the slowest rank of every step)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(np.asarray(x, dtype=np.float64), device=_coll_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().numpy()


def global_row_offsets(nnz: int, device: int = 0) -> list:
    """C-b: all-gather of the per-rank nnz; returns the exclusive prefix [0, nnz_0, nnz_0+nnz_1, …,
    total] — rank r's entries start at offsets[r] of the global CSR (its rows at the handle's row0)."""
    import torch
    import torch.distributed as dist
    dev = _coll_device(device)
    w = dist.get_world_size()
    t = torch.tensor([int(nnz)], dtype=torch.int64, device=dev)
    out = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(w)]
    dist.all_gather(out, t)
    counts = [int(o.item()) for o in out]
    return [0] + list(np.cumsum(counts).tolist())


def gather_csr(row_ptr, col, val, row0: int, n_rows_all: int, dst: int = 0):
    """C-c: assemble the ranks' CSR shards (contiguous unit ranges, Λ order) into one CSR on rank
    `dst` — per-rank sizes by all-gather, then point-to-point transfers (NCCL over NVLink on GPUs, gloo on CPU).
    row_ptr (int64, shard-local, starting at 0), col (int32), val: this rank's shard as torch tensors on the
    collective's device.  Returns (row_ptr, col, val) of the whole Θ on `dst`, None elsewhere."""
    import torch
    import torch.distributed as dist
    r, w = dist.get_rank(), dist.get_world_size()
    dev = row_ptr.device
    meta = torch.tensor([int(row0), int(row_ptr.numel() - 1), int(col.numel())], dtype=torch.int64, device=dev)
    metas = [torch.zeros(3, dtype=torch.int64, device=dev) for _ in range(w)]
    dist.all_gather(metas, meta)
    metas = [[int(x) for x in m.tolist()] for m in metas]
    if r != dst:
        for t in (row_ptr, col, val):
            if t.numel():
                dist.send(t.contiguous(), dst)
        return None
    nnz_all = sum(m[2] for m in metas)
    rp_all = torch.zeros(n_rows_all + 1, dtype=torch.int64, device=dev)
    col_all = torch.empty(nnz_all, dtype=col.dtype, device=dev)
    val_all = torch.empty(nnz_all, dtype=val.dtype, device=dev)
    off = 0
    for q, (q_row0, q_rows, q_nnz) in enumerate(metas):
        if q == dst:
            parts = (row_ptr, col, val)
        else:
            parts = (torch.empty(q_rows + 1, dtype=torch.int64, device=dev), torch.empty(q_nnz, dtype=col.dtype, device=dev),
                     torch.empty(q_nnz, dtype=val.dtype, device=dev))
            for t in parts:
                if t.numel():
                    dist.recv(t, q)
        rp_all[q_row0 + 1:q_row0 + q_rows + 1] = parts[0][1:] + off
        col_all[off:off + q_nnz] = parts[1]
        val_all[off:off + q_nnz] = parts[2]
        off += q_nnz
    return rp_all, col_all, val_all


def apply_distributed(dec: "Decomposition", x, transpose: bool = False):
    """C-d: Θ_ret x over a sharded Θ.  transpose = 0: x is the full Λ-vector (replicated), each rank
    multiplies its rows (pcwd_apply) and the row blocks are all-gathered into the full y.  transpose = 1: x is the
    full vector too; each rank applies its rows' transpose to its slice x[row0:row1] (a full-length partial) and
    the partials are summed by an all-reduce — Θᵀx = Σ_r Θ_rᵀ x_r (the FISTA gradient Θ_L*(…))."""
    import torch
    import torch.distributed as dist
    info = dec.info()
    if not transpose:
        y_loc = dec.apply(x)
        sizes = [torch.zeros(1, dtype=torch.int64, device=x.device) for _ in range(dist.get_world_size())]
        dist.all_gather(sizes, torch.tensor([y_loc.numel()], dtype=torch.int64, device=x.device))
        mx = max(int(t.item()) for t in sizes)
        buf = torch.zeros(mx, dtype=x.dtype, device=x.device)
        buf[:y_loc.numel()] = y_loc
        outs = [torch.empty(mx, dtype=x.dtype, device=x.device) for _ in sizes]
        dist.all_gather(outs, buf)
        return torch.cat([o[:int(n.item())] for o, n in zip(outs, sizes)])
    y = dec.apply(x[info.row0:info.row1].contiguous(), transpose=True)
    dist.all_reduce(y, op=dist.ReduceOp.SUM)
    return y


def fista_distributed(dec: "Decomposition", z0, w, iters: int, precond: bool = False, tau: float = 0.0, group=None):
    """FISTA-W / WP over a Θ_L sharded by rows across the ranks of `group` (one handle per rank): the
    per-iteration exchange is one all-reduce of the N-vector gradient (NCCL on the current stream).  z0, w: the whole
    N-vectors on every rank; returns (z, τ), the same on every rank."""
    import torch
    import torch.distributed as dist
    stream = torch.cuda.current_stream(z0.device).cuda_stream if z0.is_cuda else 0

    def reduce(_which, buf):
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return dec.fista_sharded(z0, w, iters, reduce, precond=precond, tau=tau, stream=stream)


# ---- host-only plan queries (no GPU) ---------------------------------------------------------

def validate(spec: Spec) -> int:
    keep = []
    return lib().pcwd_validate(ctypes.byref(make_desc(spec, keep)))


def plan_shard(spec: Spec) -> tuple[int, int]:
    keep = []
    d = make_desc(spec, keep)
    r0, r1 = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().pcwd_plan_shard(ctypes.byref(d), ctypes.byref(r0), ctypes.byref(r1)), "pcwd_plan_shard")
    return r0.value, r1.value


def plan_stencil(spec: Spec, sb: int):
    keep = []
    d = make_desc(spec, keep)
    L = spec.band_L
    a = np.zeros(L, dtype=np.int32)
    b = np.zeros(L, dtype=np.int32)
    c = np.zeros(L, dtype=np.int32)
    p = lambda x: x.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))  # noqa: E731
    _check(lib().pcwd_plan_stencil(ctypes.byref(d), sb, p(a), p(b), p(c)), "pcwd_plan_stencil")
    return a, b, c


def plan_atom(spec: Spec, s: int, e: int):
    """The separable path's 1-D analysis atom W_{s,e} (host only): (taps, start) with W(start + i) = taps[i]."""
    keep = []
    d = make_desc(spec, keep)
    n, st = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().pcwd_plan_atom(ctypes.byref(d), s, e, None, 0, ctypes.byref(n), ctypes.byref(st)), "pcwd_plan_atom")
    out = np.zeros(n.value, dtype=np.float64)
    _check(lib().pcwd_plan_atom(ctypes.byref(d), s, e, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n.value,
                                ctypes.byref(n), ctypes.byref(st)), "pcwd_plan_atom")
    return out, st.value


def num_subbands(spec: Spec) -> int:
    keep = []
    d = make_desc(spec, keep)
    out = ctypes.c_int32()
    _check(lib().pcwd_plan_num_subbands(ctypes.byref(d), ctypes.byref(out)), "pcwd_plan_num_subbands")
    return out.value


def rows3d(n: int, levels: int, h, u, v, units, stream: int = 0):
    """d = 3 (pcwd_rows3d): rows `units` of Θ on the n³ torus.  u, v: (m, n³) torch.float64 CUDA tensors; returns a
    (len(units), n³) torch.float64 CUDA tensor."""
    import torch
    h = np.ascontiguousarray(h, dtype=np.float64)
    units = np.ascontiguousarray(units, dtype=np.int64)
    assert u.is_cuda and v.is_cuda and u.dtype == torch.float64 and v.dtype == torch.float64
    out = torch.empty((len(units), n ** 3), dtype=torch.float64, device=u.device)
    _check(lib().pcwd_rows3d(n, levels, ctypes.c_void_p(_ptr(h)), len(h), u.shape[0], ctypes.c_void_p(_ptr(u)),
                             ctypes.c_void_p(_ptr(v)), ctypes.c_void_p(_ptr(units)), len(units),
                             ctypes.c_void_p(_ptr(out)), ctypes.c_void_p(stream)), "pcwd_rows3d")
    return out
