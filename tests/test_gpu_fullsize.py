"""Parity at BASELINE's full single-GPU size: config 2 (m = 262144, n = 2000,
fp64, k = 20, r = 60, c = 100, l2n, tau = 1 - 1e-8, seed 7) -- the bench
workload itself -- against the CPU oracle on the same matrix: identical
per-round remaining counts (the draws), sigma within 1e-10 relative, principal
angles below 1e-8 rad; plus size-independent properties of the factor."""

import numpy as np
import pytest
from parity_util import ANGLE_TOL_RAD, SIGMA_RTOL, principal_angles_sin, sigma_relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1905_05107_b200 as pod  # noqa: E402
from oracle import isma_oracle as orc  # noqa: E402
from paper_1905_05107_b200 import workloads  # noqa: E402
from paper_1905_05107_b200.device import ColMat  # noqa: E402


@pytest.mark.timeout(900)
def test_config2_full_size_matches_oracle():
    dev = torch.device("cuda", 0)
    side, n = 512, 2000
    at = workloads.config2_torch(0, side, n, device=dev)
    m = side * side
    cfg = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", criterion="modes",
                         seed=7)
    f, tr = pod.isma_run(ColMat(at, m), cfg)
    a_host = at.cpu().numpy().T  # F-ordered (m, n) view of the same matrix
    del at
    torch.cuda.empty_cache()
    o = orc.run(a_host, 20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", criterion="modes",
                seed=7)
    assert [t.remaining for t in tr] == [t["remaining"] for t in o["trace"]]
    assert [t.columns_sampled for t in tr] == [t["unique"].size for t in o["trace"]]
    assert sigma_relerr(f.sigma, o["sigma"]) <= SIGMA_RTOL
    assert principal_angles_sin(f.u, o["u"]).max() <= ANGLE_TOL_RAD
    assert principal_angles_sin(f.v, o["v"]).max() <= ANGLE_TOL_RAD
    # size-independent properties: orthonormal bases, descending sigma, and
    # the finalize identity A^T U = V Sigma (isma.py:295-301)
    f.validate(1e-11)
    assert np.all(np.diff(f.sigma) <= 0)
    atu = a_host.T @ f.u
    assert np.abs(atu - f.v * f.sigma).max() <= 1e-10 * f.sigma[0]


@pytest.mark.timeout(900)
def test_config4_full_size_properties():
    """Config 4 at full size (1024^2 x 8192 stored fp32, 34 GB; k = 64,
    r = 192, c = 256): too large for the CPU oracle, so size-independent
    properties -- exhaustion after ceil(n / distinct draws) rounds, bitwise
    reproducible reruns, orthonormal factors, descending sigma and the
    finalize identity A^T U = V Sigma checked in fp64 column chunks."""
    torch.cuda.empty_cache()
    dev = torch.device("cuda", 0)
    side, n = 1024, 8192
    at = workloads.config4_torch(7, side, n, device=dev)
    m = side * side
    A = ColMat(at, m)
    cfg = pod.IsmaConfig(k=64, r=192, c=256, tau=1 - 1e-8, strategy="l2n", seed=7)
    f1, tr1 = pod.isma_run(A, cfg)
    f2, tr2 = pod.isma_run(A, cfg)
    assert np.array_equal(f1.u, f2.u) and np.array_equal(f1.sigma, f2.sigma)
    assert [t.remaining for t in tr1] == [t.remaining for t in tr2]
    assert tr1[-1].remaining == 0
    assert sum(t.columns_sampled for t in tr1) == n
    f1.validate(1e-10)
    assert np.all(np.diff(f1.sigma) <= 0)
    u = torch.as_tensor(f1.u, device=dev)
    worst = 0.0
    for j0 in range(0, n, 1024):
        blk = at[j0:j0 + 1024].to(torch.float64)  # (cols, m): exact upcast
        atu = (blk @ u).cpu().numpy()
        worst = max(worst, float(np.abs(atu - f1.v[j0:j0 + 1024] * f1.sigma).max()))
    assert worst <= 1e-9 * f1.sigma[0]
