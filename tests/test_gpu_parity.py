"""End-to-end parity of the GPU isma_run / block_merge against the reference
golden fixtures (tests/golden, produced by the reference itself) and the
CPU oracle on the same seeded inputs."""

import numpy as np
import pytest
from podtest_util import load_golden, make_low_rank, make_noisy_low_rank, random_orthonormal
from parity_util import ANGLE_TOL_RAD, SIGMA_RTOL, principal_angles_sin, sigma_relerr

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1905_05107_b200 as pod  # noqa: E402
from oracle import isma_oracle as orc  # noqa: E402
from paper_1905_05107_b200 import workloads  # noqa: E402


class Recorder:
    """Wraps a numpy Generator and records each uniform batch."""

    def __init__(self, seed):
        self.g = np.random.default_rng(seed)
        self.batches = []

    def random(self, n):
        b = self.g.random(n)
        self.batches.append(b)
        return b


def _matrix(name):
    if name == "rank3_ort_fallback":
        return make_low_rank(60, 30, 3, np.random.default_rng(10))
    if name.startswith("cfg1"):
        return workloads.config1(seed=0)
    if name.startswith("rank3"):
        return make_low_rank(100, 60, 3, np.random.default_rng(7))
    if name == "exhaustive_40x18":
        return np.random.default_rng(13).standard_normal((40, 18))
    if name == "cfg2proxy_l2n":
        return workloads.config2(seed=1, side=64, n=300)
    raise KeyError(name)


GOLDEN_CASES = ["cfg1_l2n_modes", "cfg1_unf_subspace", "cfg1_l2n_nofinal_keep11",
                "rank3_unf", "rank3_l2n", "exhaustive_40x18", "cfg2proxy_l2n", "cfg1_ort_modes",
                "rank3_ort_fallback", "rank3_unf_rows", "rank3_ort_rows", "rank3_ls_rows",
                "cfg1_ls_rows", "cfg1_unf_rows_subspace"]


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_isma_run_matches_reference_golden(name):
    g = load_golden(name)
    k, r, c, fin, keep, w = (int(x) for x in g["meta"])
    cfg = pod.IsmaConfig(k=k, r=r, c=c, tau=float(g["tau"]), strategy=str(g["strategy"]),
                         criterion=str(g["criterion"]), seed=int(g["seed"]),
                         finalize=bool(fin), rows=w > 0, w=w or None)
    a = _matrix(name)
    factor, traces = pod.isma_run(a, cfg, keep=None if keep < 0 else keep)
    # rounds, index-set bookkeeping: exact
    assert len(traces) == int(g["n_rounds"])
    np.testing.assert_array_equal([t.remaining for t in traces], g["remaining"])
    np.testing.assert_array_equal([t.columns_sampled for t in traces], g["columns_sampled"])
    np.testing.assert_array_equal([t.rows_sampled for t in traces], g["rows_sampled"])
    # singular values and modes within the fp64 tolerance
    assert factor.nmodes == g["sigma"].size
    assert sigma_relerr(factor.sigma, g["sigma"]) <= SIGMA_RTOL
    ang = principal_angles_sin(factor.u, g["u"])
    assert ang.max() <= ANGLE_TOL_RAD, ang.max()
    if fin:
        assert factor.v is not None
        assert principal_angles_sin(factor.v, g["v"]).max() <= ANGLE_TOL_RAD
    factor.validate(1e-10)


def test_isma_run_index_sets_bit_exact_cfg1():
    """Per-round unique index sets of the GPU draw == the reference's
    (recorded in the golden file) for the same generator stream."""
    g = load_golden("cfg1_l2n_modes")
    a = workloads.config1(seed=0)
    cfg = pod.IsmaConfig(k=10, r=30, c=50, tau=1 - 1e-8, strategy="l2n", seed=7)
    # drive the oracle with the same uniforms and compare per-round sets
    rec = Recorder(7)
    factor, traces = pod.isma_run(a, cfg, rng=rec)
    out = orc.run(a, 10, r=30, c=50, tau=1 - 1e-8, strategy="l2n",
                  rng=np.random.default_rng(7), monitor=True)
    off = g["draw_off"]
    for i, t in enumerate(out["trace"]):
        np.testing.assert_array_equal(t["unique"], g["draw_idx"][off[i]:off[i + 1]])
    assert len(rec.batches) == len(out["trace"])
    assert min(t["margin"] for t in out["trace"]) > 1e-12


@pytest.mark.parametrize("strategy,criterion,tau", [("l2n", "modes", 0.99),
                                                     ("unf", "modes", 0.999),
                                                     ("unf", "subspace", 0.99)])
def test_isma_run_matches_oracle_noisy(strategy, criterion, tau):
    a = make_noisy_low_rank(300, 120, 6, np.random.default_rng(3),
                            sigma=np.linspace(10, 5, 6), noise=0.05)
    cfg = pod.IsmaConfig(k=6, c=24, tau=tau, strategy=strategy, criterion=criterion, seed=4)
    f, tr = pod.isma_run(a, cfg)
    o = orc.run(a, 6, c=24, tau=tau, strategy=strategy, criterion=criterion, seed=4)
    assert [t.remaining for t in tr] == [t["remaining"] for t in o["trace"]]
    assert sigma_relerr(f.sigma, o["sigma"]) <= SIGMA_RTOL
    assert principal_angles_sin(f.u, o["u"]).max() <= ANGLE_TOL_RAD


def test_block_merge_fixtures():
    g = load_golden("merges")
    for i in range(4):
        f1 = pod.TruncatedFactor(g[f"m{i}_u1"], g[f"m{i}_s1"])
        f2 = pod.TruncatedFactor(g[f"m{i}_u2"], g[f"m{i}_s2"])
        mg = pod.block_merge(f1, f2, int(g[f"m{i}_r"]))
        assert mg.nmodes == g[f"m{i}_s"].size
        assert sigma_relerr(mg.sigma, g[f"m{i}_s"]) <= 1e-12
        assert principal_angles_sin(mg.u, g[f"m{i}_u"]).max() <= 1e-10
        # same canonical signs column by column
        dots = np.einsum("ij,ij->j", mg.u, g[f"m{i}_u"])
        assert np.all(dots > 0.5)


# ---- reference tests/test_merge.py:25-93 semantics on the GPU -------------
def _exact(a):
    u, s, _ = np.linalg.svd(a, full_matrices=False)
    return pod.TruncatedFactor(u, s)


def test_merge_duplicate_rank_one_scales_by_sqrt2(rng):
    x = rng.standard_normal(9)
    u = (x / np.linalg.norm(x)).reshape(-1, 1)
    f = pod.TruncatedFactor(u, np.array([2.5]))
    mg = pod.block_merge(f, f, 4)
    assert mg.nmodes == 1
    np.testing.assert_allclose(mg.sigma[0], 2.5 * np.sqrt(2.0), rtol=1e-12)
    assert abs(abs(mg.u[:, 0] @ u[:, 0]) - 1.0) <= 1e-12


def test_merge_exactly_duplicate_factor_safe(rng):
    f = _exact(rng.standard_normal((20, 6)))
    mg = pod.block_merge(f, f, 12)
    assert np.abs(mg.u.T @ mg.u - np.eye(mg.nmodes)).max() <= 1e-10
    np.testing.assert_allclose(mg.sigma, np.sqrt(2.0) * f.sigma, rtol=1e-10)


def test_merge_nearly_parallel_stay_orthonormal(rng):
    u1 = random_orthonormal(50, 5, rng)
    u2 = np.linalg.qr(u1 + 1e-9 * rng.standard_normal((50, 5)))[0]
    s = np.linspace(5.0, 1.0, 5)
    mg = pod.block_merge(pod.TruncatedFactor(u1, s), pod.TruncatedFactor(u2, s), 10)
    assert np.abs(mg.u.T @ mg.u - np.eye(mg.nmodes)).max() <= 1e-10


def test_merge_row_mismatch_rejected(rng):
    f1 = _exact(rng.standard_normal((8, 3)))
    f2 = _exact(rng.standard_normal((9, 3)))
    with pytest.raises(pod.ParameterError, match="row spaces"):
        pod.block_merge(f1, f2, 3)


def test_merge_random_orthonormal_monotone(rng):
    for _ in range(20):
        m = int(rng.integers(10, 60))
        f1 = _exact(rng.standard_normal((m, int(rng.integers(2, 8)))))
        f2 = _exact(rng.standard_normal((m, int(rng.integers(2, 8)))))
        r = int(rng.integers(2, 10))
        mg = pod.block_merge(f1, f2, r)
        o_u, o_s = orc.merge(f1.u, f1.sigma, f2.u, f2.sigma, r)
        assert np.abs(mg.u.T @ mg.u - np.eye(mg.nmodes)).max() <= 1e-10
        assert sigma_relerr(mg.sigma, o_s) <= 1e-12


# ---- reference tests/test_isma.py behaviour on the GPU --------------------
def test_tau_zero_runs_one_update_round():
    a = make_noisy_low_rank(80, 40, 4, np.random.default_rng(0), noise=0.05)
    for criterion in ("modes", "subspace"):
        cfg = pod.IsmaConfig(k=4, tau=0.0, c=10, strategy="unf", criterion=criterion, seed=3)
        f, tr = pod.isma_run(a, cfg)
        assert len(tr) == 2 and tr[-1].remaining > 0 and f.nmodes == 4


def test_rank_shortfall_returns_fewer_modes(rng):
    x = rng.standard_normal(100)
    a = np.outer(x, rng.standard_normal(8) + 2.0)
    f, tr = pod.isma_run(a, pod.IsmaConfig(k=3, seed=1))
    assert f.nmodes == 1 and tr[-1].remaining == 0
    assert abs(f.u[:, 0] @ (x / np.linalg.norm(x))) >= 1 - 1e-8


def test_l2n_stops_when_only_zero_columns_remain(rng):
    a = np.zeros((50, 10))
    live = rng.standard_normal((50, 6))
    a[:, :6] = live / np.linalg.norm(live, axis=0)
    f, tr = pod.isma_run(a, pod.IsmaConfig(k=2, strategy="l2n", tau=1.0, c=200, seed=0))
    assert tr[-1].remaining == 4
    o = orc.run(a, 2, c=200, tau=1.0, strategy="l2n", seed=0)
    assert sigma_relerr(f.sigma, o["sigma"]) <= SIGMA_RTOL


def test_errors_match_reference():
    with pytest.raises(pod.ParameterError):
        pod.isma_run(np.ones((20, 8)), pod.IsmaConfig(k=9))
    with pytest.raises(pod.ParameterError):
        pod.isma_run(np.ones((20, 8)), pod.IsmaConfig(k=2), keep=7)
    bad = np.ones((30, 5))
    bad[3, 2] = np.inf
    with pytest.raises(pod.ParameterError, match="non-finite"):
        pod.isma_run(bad, pod.IsmaConfig(k=2))
    with pytest.raises(pod.DegenerateDistributionError):
        pod.isma_run(np.zeros((30, 5)), pod.IsmaConfig(k=2))


def test_same_seed_reproduces_bitwise():
    a = make_noisy_low_rank(70, 50, 5, np.random.default_rng(1), noise=0.1)
    cfg = pod.IsmaConfig(k=5, r=15, strategy="unf", tau=0.999, c=20, seed=42)
    f1, t1 = pod.isma_run(a, cfg)
    f2, t2 = pod.isma_run(a, cfg)
    assert np.array_equal(f1.u, f2.u) and np.array_equal(f1.sigma, f2.sigma)


def test_sample_with_replacement_known_answer():
    class Q:
        def __init__(self, b):
            self.b = [np.asarray(x, dtype=np.float64) for x in b]

        def random(self, n):
            x = self.b.pop(0)
            assert x.shape == (n,)
            return x

    d = pod.Distribution(np.array([3, 7, 9]), np.array([0.2, 0.3, 0.5]))
    dr = pod.sample_with_replacement(d, 5, Q([[0.05, 0.21, 0.45, 0.51, 0.99]]))
    np.testing.assert_array_equal(dr.unique_indices, [3, 7, 9])
    np.testing.assert_array_equal(dr.counts, [1, 2, 2])


def test_graph_replay_matches_eager_bitwise():
    """The CUDA-graph round and the eager launch sequence are the same
    kernels on the same data: identical results bit for bit."""
    a = workloads.config1(seed=0)
    cfg = pod.IsmaConfig(k=10, r=30, c=50, tau=1 - 1e-8, strategy="l2n", seed=7)
    f1, t1 = pod.isma_run(a, cfg, use_graphs=True)
    f2, t2 = pod.isma_run(a, cfg, use_graphs=False)
    assert np.array_equal(f1.u, f2.u) and np.array_equal(f1.sigma, f2.sigma)
    assert [t.remaining for t in t1] == [t.remaining for t in t2]
    for a1, a2 in zip(t1, t2):
        assert np.array_equal(a1.cosines, a2.cosines)


def test_large_rank_capacity_paths():
    """r > 64 exercises the 128/192-column NN tiles and Jacobi on >128 columns
    (the 384-column E of r = 192 runs on a 16-CTA cluster)."""
    a = workloads.config1(seed=3, m=3000, n=400)
    for k, r in ((30, 90), (40, 160), (64, 192)):  # 2r = 384: 16-CTA block-Jacobi cluster
        cfg = pod.IsmaConfig(k=k, r=r, c=150, tau=0.999, strategy="l2n", seed=2)
        f, tr = pod.isma_run(a, cfg)
        o = orc.run(a, k, r=r, c=150, tau=0.999, strategy="l2n", seed=2)
        assert [t.remaining for t in tr] == [t["remaining"] for t in o["trace"]]
        assert sigma_relerr(f.sigma, o["sigma"]) <= SIGMA_RTOL
        assert principal_angles_sin(f.u, o["u"]).max() <= ANGLE_TOL_RAD


def test_pipelined_rounds_consume_generator_like_reference():
    """The cross-round pipeline stages uniforms one round ahead; after the run
    the caller's generator must be exactly where the reference leaves it."""
    a = make_noisy_low_rank(200, 90, 5, np.random.default_rng(8), noise=0.05)
    for strategy, tau in (("unf", 0.99), ("l2n", 0.999), ("l2n", 1.0)):
        cfg = pod.IsmaConfig(k=5, c=12, tau=tau, strategy=strategy, seed=0)
        g1 = np.random.default_rng(21)
        f, tr = pod.isma_run(a, cfg, rng=g1)
        g2 = np.random.default_rng(21)
        o = orc.run(a, 5, c=12, tau=tau, strategy=strategy, rng=g2)
        assert [t.remaining for t in tr] == [t["remaining"] for t in o["trace"]]
        assert g1.random() == g2.random()
        assert sigma_relerr(f.sigma, o["sigma"]) <= SIGMA_RTOL


def test_pipelined_equals_unpipelined_bitwise():
    """A generator without a rollback-able state runs the unpipelined round:
    both orders of work produce identical results bit for bit."""
    a = workloads.config1(seed=0)
    cfg = pod.IsmaConfig(k=10, r=30, c=50, tau=1 - 1e-8, strategy="l2n", seed=7)
    f1, t1 = pod.isma_run(a, cfg)  # numpy Generator -> pipelined
    f2, t2 = pod.isma_run(a, cfg, rng=Recorder(7))  # plain object -> not pipelined
    assert np.array_equal(f1.u, f2.u) and np.array_equal(f1.sigma, f2.sigma)


def test_config3_proxy_matches_oracle():
    """BASELINE config 3 generator (power-law rank 200 + noise) at proxy size
    with config 3's k = 50, r = 150, c = 200: the 300-column E-SVD and the
    200-column Gram eigensolve of the block-Jacobi solver, 192-column NN tiles,
    against the oracle on the same seeded matrix."""
    a = workloads.config3(seed=0, m=12000, n=1400)
    cfg = pod.IsmaConfig(k=50, r=150, c=200, tau=1 - 1e-8, strategy="l2n", seed=7)
    f, tr = pod.isma_run(a, cfg)
    o = orc.run(a, 50, r=150, c=200, tau=1 - 1e-8, strategy="l2n", seed=7)
    assert [t.remaining for t in tr] == [t["remaining"] for t in o["trace"]]
    assert sigma_relerr(f.sigma, o["sigma"]) <= SIGMA_RTOL
    assert principal_angles_sin(f.u, o["u"]).max() <= ANGLE_TOL_RAD
    assert principal_angles_sin(f.v, o["v"]).max() <= ANGLE_TOL_RAD
    f.validate(1e-10)


@pytest.mark.parametrize("strategy,rows", [("l2n", False), ("ort", False), ("ls", True)])
def test_float32_storage_matches_fp64_oracle_on_upcast(strategy, rows):
    """BASELINE config 4 semantics: A stored float32 on the device (half the
    HBM); every kernel upcasts exactly, so the run equals the reference's
    float64 run on the upcast matrix (as_dense, matcore.py:49) at the fp64
    tolerances -- index sets included."""
    a32 = workloads.config4(seed=3, side=64, n=300)
    assert a32.dtype == np.float32
    a64 = a32.astype(np.float64)
    kw = dict(k=12, r=36, c=40, tau=1 - 1e-8, strategy=strategy, seed=5)
    cfg = pod.IsmaConfig(rows=rows, w=300 if rows else None, **kw)
    f32, t32 = pod.isma_run(a32, cfg)
    f64, t64 = pod.isma_run(a64, cfg)
    o = orc.run(a64, 12, r=36, c=40, tau=1 - 1e-8, strategy=strategy, seed=5, rows=rows,
                w=300 if rows else None)
    assert [t.remaining for t in t32] == [t["remaining"] for t in o["trace"]]
    assert [t.remaining for t in t32] == [t.remaining for t in t64]
    # ICRS included: its row norms (np.einsum "ij,ij->i") and row draw are in
    # numpy's exact order too, so the row sets match and the fp64 tolerances hold
    assert sigma_relerr(f32.sigma, o["sigma"]) <= SIGMA_RTOL
    assert principal_angles_sin(f32.u, o["u"]).max() <= ANGLE_TOL_RAD
    assert sigma_relerr(f32.sigma, f64.sigma) <= 1e-12
    rep = pod.wedin_measure(a32, f32, 10)
    rep64 = pod.wedin_measure(a64, f64, 10)
    assert abs(rep.measure - rep64.measure) <= 1e-8 * max(1.0, abs(rep64.measure))


@pytest.mark.parametrize("strategy,rows,criterion", [("l2n", False, "modes"),
                                                     ("unf", False, "subspace"),
                                                     ("ort", False, "modes"),
                                                     ("ls", True, "modes")])
def test_host_resident_streamed_run_is_bit_identical(strategy, rows, criterion):
    """Multi-pass streamed ISMA: A stays in page-locked host
    memory, read over PCIe (norm pass by the kernel, ort's U^T A and
    finalize's A^T U on DMA-streamed column chunks) and each round copies its
    sampled columns into HBM.  Index sets identical to the device-resident
    run; the chunked products only change split-K summation order (float64
    and float32 storage)."""
    a = workloads.config1(seed=0)
    cfg = pod.IsmaConfig(k=10, r=30, c=50, tau=0.999, strategy=strategy, rows=rows,
                         w=400 if rows else None, criterion=criterion, seed=7)
    for mat in (a, a.astype(np.float32)):
        fd, td = pod.isma_run(mat, cfg, residency="device")
        fh, th = pod.isma_run(mat, cfg, residency="host")
        assert [t.remaining for t in th] == [t.remaining for t in td]
        assert sigma_relerr(fh.sigma, fd.sigma) <= SIGMA_RTOL
        assert principal_angles_sin(fh.u, fd.u).max() <= ANGLE_TOL_RAD
        assert principal_angles_sin(fh.v, fd.v).max() <= ANGLE_TOL_RAD


@pytest.mark.parametrize("strategy", ["l2n", "unf"])
def test_config5_proxy_host_resident_matches_oracle(strategy):
    """BASELINE config 5's generator (rank 100, sigma_i = exp(-i/20),
    N(0, 1e-5), float32 in page-locked host memory, built block by block) at
    a CPU-checkable size, run out of core (residency="host": norm pass over
    PCIe, per-round sampled columns copied to HBM, finalize streamed) against
    the CPU oracle on the exact float64 upcast: every round's index set and
    counts identical, sigma within 1e-10, angles below 1e-8 rad."""
    from paper_1905_05107_b200 import engine, isma

    host = workloads.config5_host(seed=3, m=120_000, n=1500, device="cuda")
    a64 = host.numpy().T.astype(np.float64)
    cfg = pod.IsmaConfig(k=32, r=96, c=128, tau=1 - 1e-8, strategy=strategy, seed=5)
    engine.RECORD_DRAWS = True
    try:
        f, tr = pod.isma_run(host.T, cfg, residency="host")
        draws = isma.LAST_DRAWS
    finally:
        engine.RECORD_DRAWS = False
    o = orc.run(a64, 32, r=96, c=128, tau=1 - 1e-8, strategy=strategy, seed=5)
    assert len(draws) == len(o["trace"]) == len(tr)
    for (gi, gc), t in zip(draws, o["trace"]):
        assert np.array_equal(gi, t["unique"]) and np.array_equal(gc, t["counts"])
    assert sigma_relerr(f.sigma, o["sigma"]) <= SIGMA_RTOL
    assert principal_angles_sin(f.u, o["u"]).max() <= ANGLE_TOL_RAD
    assert principal_angles_sin(f.v, o["v"]).max() <= ANGLE_TOL_RAD
