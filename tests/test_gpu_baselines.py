"""Single-round baselines (ltsvd / ctsvd, baselines.py:35-142), the sampling
helpers they use (sampling.py:143-258) and the exact factorizations
(dense_svd / thin_qr / pod_via_gram / orthonormalize, matcore.py:178-254) on
the GPU, against the reference's golden outputs (tests/golden/baselines.npz)
and the CPU oracle."""

import warnings

import numpy as np
import pytest
from podtest_util import load_golden
from parity_util import ANGLE_TOL_RAD, SIGMA_RTOL, principal_angles_sin, sigma_relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1905_05107_b200 as pod  # noqa: E402
from oracle import isma_oracle as orc  # noqa: E402
from paper_1905_05107_b200 import workloads  # noqa: E402


@pytest.fixture(scope="module")
def golden():
    return load_golden("baselines")


@pytest.fixture(scope="module")
def a1():
    return workloads.config1(seed=0)


def _same_factor(u, s, u_ref, s_ref, angle_tol=ANGLE_TOL_RAD, srtol=SIGMA_RTOL):
    assert s.size == s_ref.size
    assert sigma_relerr(s, s_ref) <= srtol
    if s.size:
        assert principal_angles_sin(u, u_ref).max() <= angle_tol


# ------------------------------------------------------------ sampling ----

@pytest.mark.parametrize("dedup", [True, False])
def test_scale_sampled_columns_and_rows_match_reference_formulas(rng, dedup):
    a = rng.standard_normal((70, 40))
    dist = pod.column_norm_distribution(a)
    draw = pod.SampleDraw(np.array([2, 5, 17, 39]), np.array([1, 3, 2, 1]), 7)
    d = pod.scale_sampled_columns(a, draw, dist, 7, dedup=dedup)
    p = dist.weight_of(draw.unique_indices)
    if dedup:
        want = a[:, draw.unique_indices] * np.sqrt(draw.counts / (7 * p))
        assert np.array_equal(d, want)  # same factors, one multiply: bit-exact
        np.testing.assert_allclose(d @ d.T, pod.scale_sampled_columns(
            a, draw, dist, 7, dedup=False) @ pod.scale_sampled_columns(
            a, draw, dist, 7, dedup=False).T, rtol=1e-12, atol=1e-12)
    else:
        want = a[:, np.repeat(draw.unique_indices, draw.counts)] / np.sqrt(
            7 * np.repeat(p, draw.counts))
        np.testing.assert_allclose(d, want, rtol=1e-15, atol=0)
    assert d.flags.f_contiguous
    rd = pod.row_norm_distribution(d)
    np.testing.assert_allclose(rd.weights, orc.row_weights(d), rtol=1e-13)
    rdraw = pod.SampleDraw(np.array([0, 9, 33]), np.array([2, 1, 1]), 4)
    q = rd.weight_of(rdraw.unique_indices)
    y = pod.scale_sampled_rows(d, rdraw, rd, 4, dedup=dedup)
    want = orc.scaled_rows_any(d, rdraw.unique_indices, rdraw.counts, q, 4, dedup)
    if dedup:
        assert np.array_equal(y, want)
    else:
        np.testing.assert_allclose(y, want, rtol=1e-15, atol=0)


def test_leverage_and_residual_distributions_match_oracle(rng):
    a = rng.standard_normal((200, 60))
    u = np.linalg.qr(rng.standard_normal((200, 5)))[0]
    lev = pod.leverage_distribution(u)
    np.testing.assert_allclose(lev.weights, orc.leverage_weights(u), rtol=1e-13)
    cand = np.arange(3, 60, 2)
    res = pod.residual_distribution(a, u, cand)
    assert np.array_equal(res.indices, cand)
    np.testing.assert_allclose(res.weights, orc.residual_weights(a, u, cand), rtol=1e-11)
    # no basis columns -> column norms
    res0 = pod.residual_distribution(a, np.zeros((200, 0)), cand)
    np.testing.assert_allclose(res0.weights, pod.column_norm_distribution(a, cand).weights,
                               rtol=1e-14)
    # candidates inside span(u) -> degenerate
    b = u @ rng.standard_normal((5, 30))
    with pytest.raises(pod.DegenerateDistributionError):
        pod.residual_distribution(b, u)
    with pytest.raises(pod.ParameterError):
        pod.leverage_distribution(np.zeros((5, 0)))
    with pytest.raises(pod.ParameterError):
        pod.residual_distribution(a, u, np.zeros(0, dtype=np.int64))


# ----------------------------------------------------------- baselines ----

def test_gram_spectrum_and_lift_match_oracle(rng):
    d = rng.standard_normal((300, 24)) * np.logspace(0, -3, 24)
    s, v = pod.gram_spectrum(d)
    s2, v2 = orc.gram_eig(d)
    assert sigma_relerr(s, s2) <= SIGMA_RTOL
    assert v.shape == (24, 24) and v.flags.f_contiguous
    np.testing.assert_allclose(np.abs(v.T @ v2), np.eye(24), atol=1e-8)
    f = pod.lift_left_vectors(d, s, v, 10)
    u3, s3 = orc.lift(d, s2, v2, 10)
    np.testing.assert_allclose(f.sigma, s3, rtol=SIGMA_RTOL)
    np.testing.assert_allclose(f.u, u3, atol=1e-9)
    # exactly rank-deficient sample: dust zeroed, keep cut at the rank
    low = rng.standard_normal((50, 3)) @ rng.standard_normal((3, 12))
    s4, v4 = pod.gram_spectrum(low)
    assert np.count_nonzero(s4) == 3
    assert pod.lift_left_vectors(low, s4, v4, 8).nmodes == 3
    assert pod.lift_left_vectors(low, np.zeros(4), np.eye(4), 2).nmodes == 0


@pytest.mark.parametrize("dedup", [True, False])
def test_ltsvd_matches_reference_golden(golden, a1, dedup):
    dist = pod.column_norm_distribution(a1)
    f = pod.ltsvd(a1, dist, 10, 50, np.random.default_rng(3), dedup=dedup)
    key = f"lt{int(dedup)}"
    _same_factor(f.u, f.sigma, golden[f"{key}_u"], golden[f"{key}_s"])
    np.testing.assert_allclose(f.u, golden[f"{key}_u"], atol=1e-8)  # same signs
    f.validate(1e-10)


@pytest.mark.parametrize("dedup", [True, False])
@pytest.mark.parametrize("tag,eps", [("ct", 0.7), ("ctf", 30.0)])
def test_ctsvd_matches_reference_golden(golden, a1, dedup, tag, eps):
    dist = pod.column_norm_distribution(a1)
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        f = pod.ctsvd(a1, dist, 10, 60, 300, eps, np.random.default_rng(4), dedup=dedup)
    key = f"{tag}{int(dedup)}"
    _same_factor(f.u, f.sigma, golden[f"{key}_u"], golden[f"{key}_s"])
    assert (f.nmodes < 10) == any("energy filter" in str(w.message) for w in rec)


def test_baseline_warnings_and_errors(a1):
    dist = pod.column_norm_distribution(a1)
    with pytest.warns(UserWarning, match="rank shortfall"):
        f = pod.ltsvd(a1, dist, 10, 5, np.random.default_rng(0))
    assert f.nmodes <= 5
    for bad in (dict(k=0), dict(w=0), dict(epsilon=0.0)):
        kw = dict(k=3, c=10, w=20, epsilon=0.5) | bad
        with pytest.raises(pod.ParameterError):
            pod.ctsvd(a1, dist, kw["k"], kw["c"], kw["w"], kw["epsilon"],
                      np.random.default_rng(0))
    with pytest.raises(pod.ParameterError):
        pod.ltsvd(a1, dist, 0, 10, np.random.default_rng(0))


# ------------------------------------------------- exact factorizations ----

@pytest.mark.parametrize("name", ["tall", "wide", "skinny"])
def test_dense_svd_matches_reference_golden(golden, name):
    a = golden[f"svd_{name}_a"]
    f = pod.dense_svd(a)
    assert sigma_relerr(f.sigma, golden[f"svd_{name}_s"]) <= SIGMA_RTOL
    np.testing.assert_allclose(f.u, golden[f"svd_{name}_u"], atol=1e-8)
    np.testing.assert_allclose(f.v, golden[f"svd_{name}_v"], atol=1e-8)
    np.testing.assert_allclose((f.u * f.sigma) @ f.v.T, a, atol=1e-11 * np.abs(a).max())


def test_dense_svd_storage_variants(rng):
    a = rng.standard_normal((120, 30))
    ref = pod.dense_svd(a)
    f32 = pod.dense_svd(a.astype(np.float32))
    u, s, v = orc.dense_svd(a.astype(np.float32).astype(np.float64))
    assert sigma_relerr(f32.sigma, s) <= SIGMA_RTOL
    np.testing.assert_allclose(f32.u, u, atol=1e-9)
    dev = pod.dense_svd(torch.as_tensor(a, device="cuda"))
    np.testing.assert_allclose(dev.sigma, ref.sigma, rtol=1e-13)
    with pytest.raises(pod.ParameterError):
        pod.dense_svd(np.zeros((1100, 1100)))
    with pytest.raises(pod.ParameterError):
        pod.dense_svd(np.array([[1.0, np.nan]]))


def test_pod_via_gram_matches_reference_golden(golden, a1):
    f = pod.pod_via_gram(a1, 10)
    assert sigma_relerr(f.sigma, golden["gram_s"]) <= SIGMA_RTOL
    np.testing.assert_allclose(f.u, golden["gram_u"], atol=1e-8)
    np.testing.assert_allclose(f.v, golden["gram_v"], atol=1e-8)
    for k in (0, 501):
        with pytest.raises(pod.ParameterError):
            pod.pod_via_gram(a1, k)


def test_pod_via_gram_wide_gram_path(rng):
    """n > 512: the Gram's eigenproblem goes to the dense symmetric solver."""
    a = (np.linalg.qr(rng.standard_normal((900, 8)))[0] * np.arange(8, 0, -1.0)) @ \
        np.linalg.qr(rng.standard_normal((700, 8)))[0].T + 1e-4 * rng.standard_normal((900, 700))
    f = pod.pod_via_gram(a, 6)
    u, s, v = orc.pod_via_gram(a, 6)
    assert sigma_relerr(f.sigma, s) <= 1e-10
    np.testing.assert_allclose(f.u, u, atol=1e-7)
    np.testing.assert_allclose(f.v, v, atol=1e-7)
    z = np.zeros((40, 30))
    z[:, 0] = 1.0
    assert pod.pod_via_gram(z, 3).nmodes == 1  # exact zeros dropped


def test_thin_qr_and_orthonormalize_match_reference(golden):
    a = golden["svd_tall_a"]
    q, r = pod.thin_qr(a)
    np.testing.assert_allclose(q.T @ q, np.eye(40), atol=1e-13)
    np.testing.assert_allclose(q @ r, a, atol=1e-12)
    assert np.array_equal(r, np.triu(r)) and (np.diag(r) >= 0).all()
    np.testing.assert_allclose(np.abs(r), np.abs(golden["qr_r"]), atol=1e-11)
    with pytest.raises(pod.ParameterError):
        pod.thin_qr(a.T)
    q2, s2 = pod.orthonormalize(golden["orth_in"])
    np.testing.assert_allclose(s2, golden["orth_s"], rtol=1e-12)
    # singular values of R are 1 +- O(1e-7): its vectors carry a 1/gap
    # amplification of rounding, so columns match to ~1e-9, the span exactly
    np.testing.assert_allclose(q2, golden["orth_q"], atol=1e-6)
    assert principal_angles_sin(q2, golden["orth_q"]).max() <= ANGLE_TOL_RAD
