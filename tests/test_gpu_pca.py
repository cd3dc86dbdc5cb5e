"""GPU construction of the product-convolution expansion (pcwd_pc_from_samples / pcwd_pc_from_svir, §3.3)
against the oracle (oracle/pca.py): components (up to nothing: the sign rule is shared), singular values, coefficient
maps, the rank-m reconstruction, and the decomposition of the GPU-built operator fed straight into pcwd_set_kernels."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import pca as PC  # noqa: E402
from paper_2005_09870_b200 import Decomposition, Spec  # noqa: E402
from paper_2005_09870_b200 import pcwd as PW  # noqa: E402
from synth import configs as C  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2005_09870_b200 import _build
    _build.build()


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("device_input", [False, True])
def test_pc_from_samples_c2_recipe(device_input):
    """Config 2's PCA (8 × 8 sampled Gaussians, R = 9, m = 5; singular values 1 … 0.0027 relative)."""
    irs, n, R, g, m = C.c2_samples()
    src = torch.from_numpy(irs).cuda() if device_input else irs
    u, v, sig = PW.pc_from_samples(2, n, R, g, m, src)
    ur, vr, sr = PC.pc_from_samples(irs, 2, n, R, g, m)
    assert np.max(np.abs(sig - sr) / sr) < 1e-12
    u, v = u.cpu().numpy(), v.cpu().numpy()
    for k in range(m):
        assert _rel(u[k], ur[k]) < 1e-9, k
        assert _rel(v[k], vr[k]) < 1e-9, k
    # the expansion is the one synth/ built config 2 from (numpy on the host): the same operator
    p = C.get("c2")
    assert _rel(u, p.u) < 1e-9 and _rel(v, p.v) < 1e-9


def test_gpu_built_operator_feeds_set_kernels():
    """u, v produced on the device go straight into pcwd_set_kernels (no host round trip); the decomposition equals
    the one of the host-built operator to fp64 rounding of the construction."""
    irs, n, R, g, m = C.c2_samples()
    u, v, _ = PW.pc_from_samples(2, n, R, g, m, irs)
    p = C.get("c2")
    dec = Decomposition(Spec(p.d, p.n, p.J, p.h, torch.from_numpy(p.u).cuda(), torch.from_numpy(p.v).cuda(),
                             dtype="f64", retain="band", band_L=64))
    dec.decompose()
    ref = dec.csr(device="cpu")[2].numpy()
    dec.set_kernels(u, v)
    dec.decompose()
    got = dec.csr(device="cpu")[2].numpy()
    assert _rel(got, ref) < 1e-9
    dec.close()


def test_pc_from_svir_anisotropic_64():
    """Randomized SVD of config 3's SVIR recipe on a 64² torus (N = 4096 responses of 25² taps), m = 8: singular
    values and the rank-8 reconstruction Σ_k u_k v_kᵀ against the exact truncated SVD."""
    n, R, m = 64, 12, 8
    svir = C.svir_anisotropic(n, R)
    u, v, sig = PW.pc_from_svir(2, n, R, m, torch.from_numpy(svir).cuda(), oversample=12, power_iters=20, seed=3)
    ur, vr, sr = PC.pc_from_svir(svir, 2, n, R, m)
    assert np.max(np.abs(sig - sr) / sr) < 1e-8
    u, v = u.cpu().numpy(), v.cpu().numpy()
    # the rank-m operator Σ_k u_k ⊗ v_k (window part of u) against the oracle's
    recon = np.einsum("kw,ky->yw", u, v)
    recon_ref = np.einsum("kw,ky->yw", ur, vr)
    assert np.linalg.norm(recon - recon_ref) / np.linalg.norm(svir) < 1e-8
    for k in range(3):                                 # well-separated leading components individually
        assert _rel(u[k], ur[k]) < 1e-8 and _rel(v[k], vr[k]) < 1e-8


def test_identity_svir_rank_one_on_gpu():
    n, R = 32, 2
    W = (2 * R + 1) ** 2
    svir = np.zeros((n * n, W))
    svir[:, W // 2] = 1.0
    u, v, sig = PW.pc_from_svir(2, n, R, 1, svir)
    e = np.zeros(n * n)
    e[0] = 1.0
    assert np.max(np.abs(u.cpu().numpy()[0] - e)) < 1e-13 and np.max(np.abs(v.cpu().numpy()[0] - 1.0)) < 1e-12
    assert abs(sig[0] - n) < 1e-10
