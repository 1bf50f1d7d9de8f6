"""ICRS row sampling (rows=True, strategies unf / ort / ls) on the GPU:
reference tests/test_isma.py semantics (exhaustive rows == column-only
update, leverage-driven draws, exact rank-3 recovery, orthonormal bases) and
parity with the CPU oracle on the same generator stream."""

import numpy as np
import pytest
from podtest_util import make_low_rank, make_noisy_low_rank
from parity_util import ANGLE_TOL_RAD, SIGMA_RTOL, principal_angles_sin, sigma_relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1905_05107_b200 as pod  # noqa: E402
from oracle import isma_oracle as orc  # noqa: E402
from paper_1905_05107_b200 import workloads  # noqa: E402

ALL_MODES = [("l2n", False), ("unf", False), ("ort", False), ("unf", True), ("ort", True),
             ("ls", True)]


class Queued:
    """Generator stub handing out prepared uniform batches in order."""

    def __init__(self, batches):
        self.b = [np.asarray(x, dtype=np.float64) for x in batches]

    def random(self, n):
        x = self.b.pop(0)
        assert x.shape == (n,)
        return x


def _spread(m):
    # one variate in the middle of each of m equal CDF cells
    return (np.arange(m) + 0.5) / m


def test_exhaustive_rows_match_column_only_update(rng):
    m, n = 12, 10
    a = rng.choice([-1.0, 1.0], size=(m, n)) * np.linspace(1.0, 2.5, n)
    s = np.arange(n)
    dist = pod.column_norm_distribution(a, s)
    col_u = rng.random(25)
    fc, rc, gc, _ = pod.get_update(a, s, None, dist, 25, 0, False, Queued([col_u]), 6)
    fr, rr, gr, h = pod.get_update(a, s, None, dist, 25, m, True,
                                   Queued([col_u, _spread(m)]), 6)
    assert gc == gr and np.array_equal(rc, rr)
    assert h == m
    assert fr.nmodes == fc.nmodes
    np.testing.assert_allclose(fr.sigma, fc.sigma, rtol=1e-8)
    np.testing.assert_allclose(fr.u, fc.u, atol=1e-8)


def test_row_draws_follow_previous_basis_leverage(rng):
    a = rng.standard_normal((8, 5))
    s = np.arange(5)
    dist = pod.column_norm_distribution(a, s)
    e0 = np.zeros((8, 1))
    e0[0, 0] = 1.0
    f, _, _, h = pod.get_update(a, s, pod.TruncatedFactor(e0, np.array([1.0])), dist, 6, 10,
                                True, rng, 3)
    assert h == 1
    assert f.nmodes <= 1


def test_get_update_rows_matches_oracle(rng):
    a = make_noisy_low_rank(300, 80, 5, np.random.default_rng(2), noise=0.05)
    s = np.arange(80)
    dist = pod.column_norm_distribution(a, s)
    cu, wu = rng.random(30), rng.random(120)
    f, rem, g, h = pod.get_update(a, s, None, dist, 30, 120, True, Queued([cu, wu]), 15)
    idx, cnt = orc.cdf_draw(s, dist.weights, cu)
    d = np.asfortranarray(a[:, idx])
    q = orc.row_weights(d)
    ridx, rcnt = orc.cdf_draw(np.arange(300), q, wu)
    sig, v = orc.gram_eig(orc.scaled_rows(d, ridx, rcnt, q, 120))
    u2, s2 = orc.lift(d, sig, v, 15)
    assert g == idx.size and h == ridx.size
    assert f.nmodes == s2.size
    assert sigma_relerr(f.sigma, s2) <= SIGMA_RTOL
    assert principal_angles_sin(f.u, u2).max() <= ANGLE_TOL_RAD
    # leverage-driven draw from a previous basis
    up = np.linalg.qr(rng.standard_normal((300, 4)))[0]
    f2, _, _, h2 = pod.get_update(a, s, pod.TruncatedFactor(up, np.ones(4)), dist, 30, 120,
                                  True, Queued([cu, wu]), 15)
    q2 = orc.leverage_weights(up)
    ridx2, rcnt2 = orc.cdf_draw(np.arange(300), q2, wu)
    sig2, v2 = orc.gram_eig(orc.scaled_rows(d, ridx2, rcnt2, q2, 120))
    u3, s3 = orc.lift(d, sig2, v2, 15)
    assert h2 == ridx2.size
    assert sigma_relerr(f2.sigma, s3) <= SIGMA_RTOL
    assert principal_angles_sin(f2.u, u3).max() <= ANGLE_TOL_RAD


@pytest.mark.parametrize("strategy,rows", ALL_MODES)
def test_recovers_exact_rank_three(strategy, rows):
    a = make_low_rank(100, 60, 3, np.random.default_rng(7))
    u, s, _ = np.linalg.svd(a, full_matrices=False)
    cfg = pod.IsmaConfig(k=3, strategy=strategy, rows=rows, tau=0.99, seed=11)
    f, tr = pod.isma_run(a, cfg)
    f.validate(1e-8)
    assert f.v is not None
    cosang = np.clip(np.abs(np.einsum("ij,ij->j", f.u, u[:, :3])), 0.0, 1.0)
    assert np.degrees(np.arccos(cosang)).max() < 1e-4
    np.testing.assert_allclose(f.sigma, s[:3], rtol=1e-8)
    assert tr[0].cosines.size == 0
    rem = [t.remaining for t in tr]
    assert all(b < a_ for a_, b in zip(rem, rem[1:]))
    for i, t in enumerate(tr):
        assert t.iteration == i
        assert (t.rows_sampled > 0) == rows
        if i:
            assert t.cosines.size == 3


@pytest.mark.parametrize("strategy", ["unf", "ort", "ls"])
@pytest.mark.parametrize("finalize", [True, False])
def test_rows_basis_always_orthonormal(strategy, finalize):
    a = make_noisy_low_rank(60, 30, 3, np.random.default_rng(4), noise=0.2)
    cfg = pod.IsmaConfig(k=3, strategy=strategy, rows=True, finalize=finalize, tau=0.99,
                         seed=6)
    f, _ = pod.isma_run(a, cfg)
    f.validate(1e-8)


@pytest.mark.parametrize("strategy,criterion", [("ls", "modes"), ("unf", "subspace"),
                                                ("ort", "modes")])
def test_rows_run_matches_oracle_and_consumes_generator(strategy, criterion):
    a = make_noisy_low_rank(400, 150, 6, np.random.default_rng(9),
                            sigma=np.linspace(10, 5, 6), noise=0.05)
    cfg = pod.IsmaConfig(k=6, c=24, w=160, tau=0.999, strategy=strategy, rows=True,
                         criterion=criterion, seed=0)
    g1 = np.random.default_rng(31)
    f, tr = pod.isma_run(a, cfg, rng=g1)
    g2 = np.random.default_rng(31)
    o = orc.run(a, 6, c=24, tau=0.999, strategy=strategy, criterion=criterion, rng=g2,
                rows=True, w=160)
    assert [t.remaining for t in tr] == [t["remaining"] for t in o["trace"]]
    assert [t.rows_sampled for t in tr] == [t["rows"].size for t in o["trace"]]
    assert g1.random() == g2.random()
    assert sigma_relerr(f.sigma, o["sigma"]) <= 1e-8
    assert principal_angles_sin(f.u, o["u"]).max() <= 1e-6


def test_rows_graph_replay_matches_eager_bitwise():
    a = workloads.config1(seed=0)
    cfg = pod.IsmaConfig(k=10, r=30, c=50, w=400, tau=0.999, strategy="ls", rows=True, seed=5)
    f1, t1 = pod.isma_run(a, cfg, use_graphs=True)
    f2, t2 = pod.isma_run(a, cfg, use_graphs=False)
    assert np.array_equal(f1.u, f2.u) and np.array_equal(f1.sigma, f2.sigma)
    assert [t.rows_sampled for t in t1] == [t.rows_sampled for t in t2]


def test_rows_zero_block_raises_degenerate():
    """A uniform column draw of only zero columns leaves no row mass: the
    reference raises DegenerateDistributionError (sampling.py:62-64)."""
    a = np.zeros((40, 30))
    a[:, 0] = np.linspace(1.0, 2.0, 40)
    cfg = pod.IsmaConfig(k=1, c=1, w=10, tau=1.0, strategy="unf", rows=True, seed=0)
    with pytest.raises(pod.DegenerateDistributionError):
        pod.isma_run(a, cfg)
    with pytest.raises(orc.OracleDegenerate):
        orc.run(a, 1, c=1, tau=1.0, strategy="unf", seed=0, rows=True, w=10)


@pytest.mark.gpu
def test_rows_zero_block_leaves_generator_where_reference_does():
    """The reference consumes the column batch, then raises on the zero row
    distribution before drawing the row batch (isma.py:162-173): a caller-owned
    generator must end in the same state (rollback point)."""
    a = np.zeros((40, 30))
    a[:, 0] = np.linspace(1.0, 2.0, 40)
    cfg = pod.IsmaConfig(k=1, c=1, w=10, tau=1.0, strategy="unf", rows=True, seed=0)
    for seed in range(6):
        g_gpu, g_orc = np.random.default_rng(seed), np.random.default_rng(seed)
        raised = []
        try:
            pod.isma_run(a, cfg, rng=g_gpu)
        except pod.DegenerateDistributionError:
            raised.append("gpu")
        try:
            orc.run(a, 1, c=1, tau=1.0, strategy="unf", rng=g_orc, rows=True, w=10)
        except orc.OracleDegenerate:
            raised.append("orc")
        assert raised in ([], ["gpu", "orc"])
        assert g_gpu.bit_generator.state == g_orc.bit_generator.state
