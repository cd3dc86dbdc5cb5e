"""GPU tests of the plan-reuse and streamed-output entry points (include/pcwd.h):

* pcwd_decompose_to_host (CSR rows copied to the host per launch, overlapped with the computation)
  returns exactly what pcwd_decompose + pcwd_copy_csr return;
* pcwd_set_kernels (new u_k, v_k on an existing plan) returns exactly what a fresh handle built on
  those kernels returns, and refuses kernels whose support leaves the planned box.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2005_09870_b200 import Decomposition, PcwdError, Spec  # noqa: E402
from synth import configs as C  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_09870_b200 import _build
    _build.build()


def _spec(p, dtype, u=None, v=None):
    return Spec(p.d, p.n, p.J, p.h, p.u if u is None else u, p.v if v is None else v, dtype=dtype,
                retain=p.retain, tau_rel=p.tau_rel, band_L=p.band_L)


def _csr(dec):
    return tuple(t.numpy().copy() for t in dec.csr(device="cpu"))


def _to_host(dec, like):
    rp, col, val = (torch.empty(a.shape, dtype=torch.from_numpy(a).dtype).pin_memory() for a in like)
    s = torch.cuda.Stream()
    dec.decompose_to_host(rp, col, val, stream=s.cuda_stream)
    s.synchronize()
    return rp.numpy(), col.numpy(), val.numpy()


def _other_kernels(p, seed):
    """Kernels with the same support as p.u (values rescaled per k) and a fresh random v."""
    rng = np.random.default_rng(seed)
    u = np.ascontiguousarray(p.u * rng.uniform(0.5, 1.5, size=(p.u.shape[0], 1)))
    v = np.ascontiguousarray(rng.standard_normal(p.v.shape))
    return u, v


CASES = [("c5", "f32"), ("c3", "f32"), ("band-micro", "f64"), ("full-micro", "f32"), ("threshold-micro", "f64")]


def _problem(name):
    if name == "band-micro":
        return C.micro(128, 2, 4, 5, 3, 4, 45, retain="band", band_L=64)
    if name == "full-micro":
        return C.micro(32, 2, 4, 4, 3, 3, 8, retain="full")
    if name == "threshold-micro":
        return C.micro(32, 2, 4, 4, 3, 3, 12, retain="threshold", tau_rel=1e-3)
    return C.get(name)


@pytest.mark.parametrize("name,dtype", CASES, ids=[f"{a}-{b}" for a, b in CASES])
def test_decompose_to_host_equals_decompose_and_copy(name, dtype):
    p = _problem(name)
    dec = Decomposition(_spec(p, dtype))
    dec.decompose()
    ref = _csr(dec)
    for _ in range(2):     # twice: the copy stream and its events are reused
        got = _to_host(dec, ref)
        for a, b in zip(got, ref):
            assert np.array_equal(a, b)
    dec.close()


@pytest.mark.parametrize("name,dtype", CASES, ids=[f"{a}-{b}" for a, b in CASES])
def test_set_kernels_equals_fresh_handle(name, dtype):
    p = _problem(name)
    u2, v2 = _other_kernels(p, 7)
    fresh = Decomposition(_spec(p, dtype, u2, v2))
    fresh.decompose()
    ref = _csr(fresh)
    fresh.close()
    dec = Decomposition(_spec(p, dtype))
    dec.decompose()
    dec.set_kernels(torch.from_numpy(u2).pin_memory(), torch.from_numpy(v2).pin_memory())
    dec.decompose()
    got = _csr(dec)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)
    # device-resident kernels take the same path
    dec.set_kernels(torch.from_numpy(u2).cuda(), torch.from_numpy(v2).cuda())
    got = _to_host(dec, ref)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)
    dec.close()


def test_set_kernels_rejects_support_outside_the_plan():
    p = C.micro(32, 2, 4, 4, 3, 2, 9, retain="band", band_L=128)
    dec = Decomposition(_spec(p, "f32"))
    dec.decompose()
    before = _csr(dec)
    wide = C.micro(32, 2, 4, 4, 3, 3, 9, retain="band", band_L=128)   # support radius 3 > 2
    with pytest.raises(PcwdError):
        dec.set_kernels(wide.u, wide.v)
    dec.decompose()                        # the handle kept its kernels
    for a, b in zip(_csr(dec), before):
        assert np.array_equal(a, b)
    # a smaller support inside the box is accepted
    u = np.zeros_like(p.u)
    u[:, 0] = 1.0
    dec.set_kernels(u, p.v)
    dec.decompose()
    dec.close()


def _box_of(dec, p, u):
    """u restricted to the plan's periodic bounding box (pcwd_kernel_box), m × w0 × w1, computed on the host from
    the box the library reports; also checks that u vanishes outside that box."""
    (lo0, lo1), (w0, w1) = dec.kernel_box()
    m = u.shape[0]
    full = u.reshape(m, p.n, p.n) if p.d == 2 else u.reshape(m, 1, p.n)
    r = (lo0 + np.arange(w0)) % full.shape[1]
    c = (lo1 + np.arange(w1)) % p.n
    box = np.ascontiguousarray(full[:, r][:, :, c])
    rest = full.copy()
    rest[np.ix_(np.arange(m), r, c)] = 0.0
    assert not rest.any(), "u has nonzeros outside the reported box"
    return box


@pytest.mark.parametrize("name,dtype", CASES, ids=[f"{a}-{b}" for a, b in CASES])
def test_set_kernels_box_equals_set_kernels(name, dtype):
    """pcwd_set_kernels_box (u_k given on the plan's support box) = pcwd_set_kernels with the whole u."""
    p = _problem(name)
    u2, v2 = _other_kernels(p, 11)
    dec = Decomposition(_spec(p, dtype))
    dec.set_kernels(u2, v2)
    dec.decompose()
    ref = _csr(dec)
    box = _box_of(dec, p, u2)
    assert box.shape[0] == p.u.shape[0] and box.size < u2.size or p.n <= 32
    dec.set_kernels(p.u, p.v)              # something else in between
    dec.decompose()
    dec.set_kernels_box(torch.from_numpy(box).pin_memory(), torch.from_numpy(v2).pin_memory())
    dec.decompose()
    for a, b in zip(_csr(dec), ref):
        assert np.array_equal(a, b)
    dec.set_kernels_box(torch.from_numpy(box).cuda(), torch.from_numpy(v2).cuda())   # device-resident
    got = _to_host(dec, ref)
    for a, b in zip(got, ref):
        assert np.array_equal(a, b)
    dec.close()
