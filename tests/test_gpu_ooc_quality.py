"""GPU parity of the one-pass incremental driver (ooc.py:105-148) and the
quality metrics (quality.py:38-118) against reference goldens and the oracle."""

import os

import numpy as np
import pytest
from podtest_util import load_golden, make_low_rank, make_noisy_low_rank
from parity_util import ANGLE_TOL_RAD, SIGMA_RTOL, principal_angles_sin, sigma_relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1905_05107_b200 as pod  # noqa: E402
from oracle import isma_oracle as orc  # noqa: E402
from paper_1905_05107_b200 import workloads  # noqa: E402


def _podm(tmp_path, a):
    p = str(tmp_path / "a.podm")
    pod.write_matrix(p, a)
    return p


def test_incremental_matches_reference_golden(tmp_path):
    g = load_golden("incremental_t3")
    a = workloads.config1(seed=int(g["seed"]), m=300, n=120)
    cfg = pod.IsmaConfig(k=4, c=20, tau=0.999, strategy="l2n", seed=9)
    with pod.BlockReader(_podm(tmp_path, a), 3) as rd:
        f, tr = pod.incremental_pod(rd, cfg)
        assert rd.blocks_read == 3
    np.testing.assert_array_equal([t.remaining for t in tr], g["remaining"])
    assert [t.iteration for t in tr] == list(range(len(tr)))
    assert sigma_relerr(f.sigma, g["sigma"]) <= SIGMA_RTOL
    assert principal_angles_sin(f.u, g["u"]).max() <= ANGLE_TOL_RAD


def test_single_block_matches_in_memory_run(tmp_path):
    # ooc.py:11-13: t = 1 is the in-memory run with finalize off
    a = make_noisy_low_rank(80, 50, 4, np.random.default_rng(3), noise=0.05)
    cfg = pod.IsmaConfig(k=4, c=15, tau=0.999, strategy="unf", seed=5)
    with pod.BlockReader(_podm(tmp_path, a), 1) as rd:
        f1, t1 = pod.incremental_pod(rd, cfg)
    f2, t2 = pod.isma_run(a, pod.IsmaConfig(k=4, c=15, tau=0.999, strategy="unf", seed=5,
                                            finalize=False))
    assert [t.remaining for t in t1] == [t.remaining for t in t2]
    np.testing.assert_array_equal(f1.sigma, f2.sigma)
    np.testing.assert_array_equal(f1.u, f2.u)


@pytest.mark.parametrize("strategy,rows", [("l2n", False), ("ls", True), ("ort", True)])
def test_exact_rank_four_over_four_blocks(tmp_path, strategy, rows):
    a = make_low_rank(60, 40, 4, np.random.default_rng(11))
    cfg = pod.IsmaConfig(k=4, c=30, tau=0.999, strategy=strategy, rows=rows, seed=1)
    with pod.BlockReader(_podm(tmp_path, a), 4) as rd:
        f, _ = pod.incremental_pod(rd, cfg)
    exact = np.linalg.svd(a, full_matrices=False)
    assert principal_angles_sin(f.u, exact[0][:, :4]).max() < 1e-8
    if not rows:
        np.testing.assert_allclose(f.sigma, exact[1][:4], rtol=1e-10)
    else:
        # row-sampled sigmas are estimates (the reference's too): match the oracle
        o = orc.incremental(orc.column_blocks(a, 4), 4, c=30, tau=0.999, strategy=strategy,
                            seed=1, rows=True, w=cfg.row_budget())
        assert sigma_relerr(f.sigma, o["sigma"]) <= 1e-8


def test_single_column_blocks_still_merge(tmp_path):
    a = make_low_rank(30, 6, 2, np.random.default_rng(2))
    cfg = pod.IsmaConfig(k=2, c=5, tau=0.99, strategy="l2n", seed=3)
    with pod.BlockReader(_podm(tmp_path, a), 6) as rd:
        f, tr = pod.incremental_pod(rd, cfg)
    o = orc.incremental(orc.column_blocks(a, 6), 2, c=5, tau=0.99, seed=3)
    assert sigma_relerr(f.sigma, o["sigma"]) <= 1e-10
    assert principal_angles_sin(f.u, o["u"]).max() <= ANGLE_TOL_RAD


def test_split_budget_and_exhausted_reader(tmp_path):
    a = make_noisy_low_rank(50, 40, 3, np.random.default_rng(4), noise=0.1)
    p = _podm(tmp_path, a)
    cfg = pod.IsmaConfig(k=3, c=16, tau=0.99, strategy="l2n", seed=2)
    with pod.BlockReader(p, 4) as rd:
        _, tr = pod.incremental_pod(rd, cfg, scale_count_by_blocks=True)
    assert max(t.columns_sampled for t in tr) <= 4
    with pod.BlockReader(p, 2) as rd:
        list(rd)
        with pytest.raises(pod.ParameterError, match="no blocks"):
            pod.incremental_pod(rd, cfg)


def test_wedin_matches_reference_golden():
    g = load_golden("wedin_cfg1")
    a = workloads.config1(seed=0)
    f = pod.TruncatedFactor(g["u"], g["sigma"], g["v"])
    rep = pod.wedin_measure(a, f, 10)
    np.testing.assert_allclose(rep.r_norm, float(g["r_norm"]), rtol=1e-9)
    # S = A^T U_k - V_k S_k vanishes for a finalized factor: both sides are
    # rounding noise (~1e-15), compared absolutely against ||A|| eps
    assert abs(rep.s_norm - float(g["s_norm"])) <= 1e-13 * float(np.linalg.norm(a))
    assert rep.omega_hat == float(g["omega_hat"])
    np.testing.assert_allclose(rep.measure, float(g["measure"]), rtol=1e-9)
    assert not rep.degenerate and rep.advisory is None


def test_wedin_degenerate_and_errors():
    a = make_low_rank(40, 30, 3, np.random.default_rng(0), sigma=[2.0, 1.0, 1.0])
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    f = pod.TruncatedFactor(u[:, :4], np.array([2.0, 1.0, 1.0, 0.0]), vt.T[:, :4])
    rep = pod.wedin_measure(a, f, 2)
    assert rep.degenerate and rep.measure == np.inf and rep.advisory
    with pytest.raises(pod.ParameterError):
        pod.wedin_measure(a, pod.TruncatedFactor(u[:, :2], s[:2]), 1)


def test_angles_match_oracle():
    rng = np.random.default_rng(5)
    e = np.linalg.qr(rng.standard_normal((300, 8)))[0]
    x = np.linalg.qr(e + 1e-3 * rng.standard_normal((300, 8)))[0]
    fe, fx = pod.TruncatedFactor(e, np.arange(8, 0, -1.0)), pod.TruncatedFactor(x, np.arange(8, 0, -1.0))
    pa = pod.principal_angles(fe, fx, 8)
    ref = np.degrees(np.arccos(np.clip(np.linalg.svd(x.T @ e, compute_uv=False), 0, 1)))
    np.testing.assert_allclose(pa, ref, atol=1e-9)
    ma = pod.mode_angles(fe, fx, 8)
    np.testing.assert_allclose(ma, np.degrees(np.arccos(np.clip(np.abs(np.sum(e * x, 0)), 0, 1))),
                               atol=1e-9)


def test_duck_typed_reader_streams_like_block_reader(tmp_path):
    """incremental_pod accepts any object with block_count / read_block
    (ooc.py:105-148 duck typing); the prefetching stream gives the same
    factor as the PODM BlockReader path."""
    a = make_noisy_low_rank(120, 45, 4, np.random.default_rng(6), noise=0.05)
    cfg = pod.IsmaConfig(k=4, c=12, tau=0.999, strategy="l2n", seed=2)

    class ListReader:
        def __init__(self, blocks):
            self.blocks = list(blocks)
            self.block_count = len(self.blocks)

        def read_block(self):
            return self.blocks.pop(0) if self.blocks else None

    with pod.BlockReader(_podm(tmp_path, a), 3) as rd:
        f1, t1 = pod.incremental_pod(rd, cfg)
    f2, t2 = pod.incremental_pod(ListReader(orc.column_blocks(a, 3)), cfg)
    assert [t.remaining for t in t1] == [t.remaining for t in t2]
    np.testing.assert_array_equal(f1.sigma, f2.sigma)
    np.testing.assert_array_equal(f1.u, f2.u)


def test_truncated_file_raises_at_its_block(tmp_path):
    """A PODM payload cut inside block 3 of 4: the read-ahead stream surfaces
    the reference's FormatError (byte offset in the message) when that block
    is requested, after blocks 1-2 were read."""
    a = make_noisy_low_rank(64, 40, 3, np.random.default_rng(12), noise=0.05)
    path = _podm(tmp_path, a)
    size = os.path.getsize(path)
    with open(path, "r+b") as fh:
        fh.truncate(size - 8 * 64 * 12)  # inside the third block (columns 20..29)
    cfg = pod.IsmaConfig(k=3, c=10, tau=0.99, strategy="l2n", seed=1)
    with pod.BlockReader(path, 4) as rd:
        with pytest.raises(pod.FormatError, match="byte offset"):
            pod.incremental_pod(rd, cfg)
        assert rd.blocks_read == 2
