"""The fused one-pass Wedin residual kernel (pod_wedin_residuals, replacing
quality.py:104-107) against numpy on ragged shapes: row counts off the
128-row slab and the 8/16-CTA cluster range, column counts off the 32-column
chunk, every k padding class (k = 1 ... 64), float32 storage, padded leading
dimensions; bitwise repeatability; the two-pass path beyond k = 64."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1905_05107_b200 as pod  # noqa: E402
from paper_1905_05107_b200 import quality  # noqa: E402
from paper_1905_05107_b200.device import ColMat, get_ctx, to_device_colmajor  # noqa: E402


def _np_residuals(a, u, s, v):
    r = a @ v - u * s
    q = a.T @ u - v * s
    return float(np.linalg.norm(r)), float(np.linalg.norm(q))


def _fused(a_dev, u, s, v):
    ctx = get_ctx()
    dev = ctx.device
    U = to_device_colmajor(np.asfortranarray(u), dev)
    V = to_device_colmajor(np.asfortranarray(v), dev)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    ctx.wedin(a_dev, U, V, torch.as_tensor(s, device=dev), u.shape[1], out)
    r2, s2 = out.cpu().numpy()
    return float(np.sqrt(r2)), float(np.sqrt(s2)), out


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (127, 31, 3), (128, 32, 8), (1000, 33, 9),
                                   (2049, 97, 20), (5000, 300, 33), (1025, 65, 50),
                                   (3000, 129, 64), (16411, 257, 24)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_fused_wedin_matches_numpy(m, n, k, dtype):
    rng = np.random.default_rng(m * 7 + n + k)
    a = rng.standard_normal((m, n)).astype(dtype)
    u = rng.standard_normal((m, k))
    v = rng.standard_normal((n, k))
    s = np.sort(rng.random(k))[::-1] * 10
    rr, ss = _np_residuals(a.astype(np.float64), u, s, v)
    r, q, _ = _fused(to_device_colmajor(np.asfortranarray(a), get_ctx().device), u, s, v)
    # random factors: R and S are O(sqrt(m n k)), no cancellation -> fp64 summation-order bound
    np.testing.assert_allclose(r, rr, rtol=1e-12)
    np.testing.assert_allclose(q, ss, rtol=1e-12)


def test_fused_wedin_padded_leading_dimension_and_repeatable():
    rng = np.random.default_rng(3)
    m, n, k, ld = 4099, 150, 17, 4103  # odd ld: the element-wise copy path
    buf = torch.zeros((n, ld), dtype=torch.float64, device=get_ctx().device)
    a = rng.standard_normal((m, n))
    buf[:, :m] = torch.as_tensor(a.T.copy(), device=buf.device)
    A = ColMat(buf, m)
    u, v = rng.standard_normal((m, k)), rng.standard_normal((n, k))
    s = np.linspace(3.0, 1.0, k)
    rr, ss = _np_residuals(a, u, s, v)
    r, q, o1 = _fused(A, u, s, v)
    np.testing.assert_allclose([r, q], [rr, ss], rtol=1e-12)
    _, _, o2 = _fused(A, u, s, v)
    assert torch.equal(o1, o2)  # fixed assignment and summation order


def test_fused_wedin_on_converged_factor_cancellation():
    """Exact singular triplets: R = A V - U S and S = A^T U - V S both
    vanish to rounding; they agree with numpy within ||A|| eps-scale."""
    rng = np.random.default_rng(11)
    m, n, k = 3000, 200, 12
    a = (rng.standard_normal((m, 40)) * np.exp(-np.arange(40) / 6.0)) @ rng.standard_normal((40, n))
    uu, ss_, vt = np.linalg.svd(a, full_matrices=False)
    f = pod.TruncatedFactor(uu[:, :k + 1], ss_[:k + 1], vt.T[:, :k + 1])
    rep = pod.wedin_measure(a, f, k)
    rr, sn = _np_residuals(a, uu[:, :k], ss_[:k], vt.T[:, :k])
    # exact SVD factors: both residuals are rounding noise (~1e-12 here)
    assert abs(rep.r_norm - rr) <= 1e-13 * np.linalg.norm(a)
    assert abs(rep.s_norm - sn) <= 1e-13 * np.linalg.norm(a)


def test_wedin_beyond_fused_k_uses_two_passes():
    rng = np.random.default_rng(5)
    m, n, k = 900, 120, quality.WEDIN_FUSED_MAX_K + 6
    a = rng.standard_normal((m, n))
    uu, ss_, vt = np.linalg.svd(a, full_matrices=False)
    f = pod.TruncatedFactor(uu[:, :k + 1], ss_[:k + 1], vt.T[:, :k + 1])
    rep = pod.wedin_measure(a, f, k)
    rr, sn = _np_residuals(a, uu[:, :k], ss_[:k], vt.T[:, :k])
    np.testing.assert_allclose(rep.r_norm, rr, rtol=1e-10)
    assert abs(rep.s_norm - sn) <= 1e-13 * np.linalg.norm(a)


def test_fused_wedin_config2_size_against_device_fp64():
    """Config-2 shape (m = 512^2 + 37 ragged rows, n = 2000, k = 20): against
    torch's fp64 GEMMs on the device (test-only reference)."""
    dev = get_ctx().device
    g = torch.Generator(device=dev).manual_seed(9)
    m, n, k = 262144 + 37, 2000, 20
    at = torch.randn((n, m), dtype=torch.float64, device=dev, generator=g)
    u = torch.randn((k, m), dtype=torch.float64, device=dev, generator=g)
    v = torch.randn((k, n), dtype=torch.float64, device=dev, generator=g)
    s = torch.linspace(5.0, 1.0, k, dtype=torch.float64, device=dev)
    rr = torch.linalg.norm(at.T @ v.T - u.T * s).item()
    ss = torch.linalg.norm(at @ u.T - v.T * s).item()
    ctx = get_ctx()
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    ctx.wedin(ColMat(at, m), ColMat(u, m), ColMat(v, n), s, k, out)
    r2, s2 = out.cpu().numpy()
    np.testing.assert_allclose([np.sqrt(r2), np.sqrt(s2)], [rr, ss], rtol=1e-12)
