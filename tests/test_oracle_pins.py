"""Pin the CPU oracle (oracle/isma_oracle.py) to the reference's own outputs
(tests/golden/*.npz, written by tests/golden/make_golden.py which runs the
reference package) and to the reference test suite's known-answer vectors."""

import numpy as np
import pytest
from podtest_util import load_golden

from oracle import isma_oracle as orc
from paper_1905_05107_b200 import workloads


def _case_matrix(name):
    if name.startswith("cfg1"):
        return workloads.config1(seed=0)
    if name == "rank3_ort_fallback":
        from conftest import make_low_rank
        return make_low_rank(60, 30, 3, np.random.default_rng(10))
    if name.startswith("rank3"):
        from conftest import make_low_rank
        return make_low_rank(100, 60, 3, np.random.default_rng(7))
    if name == "exhaustive_40x18":
        return np.random.default_rng(13).standard_normal((40, 18))
    if name == "cfg2proxy_l2n":
        return workloads.config2(seed=1, side=64, n=300)
    raise KeyError(name)


CASES = ["cfg1_l2n_modes", "cfg1_unf_subspace", "cfg1_l2n_nofinal_keep11",
         "rank3_unf", "rank3_l2n", "exhaustive_40x18", "cfg2proxy_l2n", "cfg1_ort_modes",
         "rank3_ort_fallback", "rank3_unf_rows", "rank3_ort_rows", "rank3_ls_rows",
         "cfg1_ls_rows", "cfg1_unf_rows_subspace"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_golden(name):
    g = load_golden(name)
    k, r, c, fin, keep, w = (int(x) for x in g["meta"])
    a = _case_matrix(name)
    out = orc.run(a, k, r=r, c=c, tau=float(g["tau"]), strategy=str(g["strategy"]),
                  criterion=str(g["criterion"]), seed=int(g["seed"]),
                  do_finalize=bool(fin), keep=None if keep < 0 else keep,
                  rows=w > 0, w=w or None)
    tr = out["trace"]
    assert len(tr) == int(g["n_rounds"])
    # per-round index sets and counts bit-exact (ICRS: column draw, row draw)
    off = g["draw_off"]
    per = 2 if w else 1
    for i, t in enumerate(tr):
        j = per * i
        np.testing.assert_array_equal(t["unique"], g["draw_idx"][off[j]:off[j + 1]])
        np.testing.assert_array_equal(t["counts"], g["draw_cnt"][off[j]:off[j + 1]])
        if w:
            np.testing.assert_array_equal(t["rows"], g["draw_idx"][off[j + 1]:off[j + 2]])
            np.testing.assert_array_equal(t["row_counts"], g["draw_cnt"][off[j + 1]:off[j + 2]])
            assert t["rows"].size == g["rows_sampled"][i]
        assert t["remaining"] == g["remaining"][i]
    # same arithmetic in the same order: bit-identical on this machine
    np.testing.assert_array_equal(out["sigma"], g["sigma"])
    np.testing.assert_array_equal(out["u"], g["u"])
    if fin:
        np.testing.assert_array_equal(out["v"], g["v"])


def test_merge_fixtures():
    g = load_golden("merges")
    for i in range(4):
        u, s = orc.merge(g[f"m{i}_u1"], g[f"m{i}_s1"], g[f"m{i}_u2"], g[f"m{i}_s2"],
                         int(g[f"m{i}_r"]))
        np.testing.assert_array_equal(s, g[f"m{i}_s"])
        np.testing.assert_array_equal(u, g[f"m{i}_u"])


def test_incremental_fixture():
    g = load_golden("incremental_t3")
    a = workloads.config1(seed=int(g["seed"]), m=300, n=120)
    out = orc.incremental(orc.column_blocks(a, 3), 4, c=20, tau=0.999, seed=9)
    np.testing.assert_array_equal(out["sigma"], g["sigma"])
    np.testing.assert_array_equal(out["u"], g["u"])
    np.testing.assert_array_equal([t["remaining"] for t in out["trace"]], g["remaining"])


def test_wedin_fixture():
    g = load_golden("wedin_cfg1")
    a = workloads.config1(seed=0)
    rep = orc.wedin(a, g["u"], g["sigma"], g["v"], 10)
    for key in ("r_norm", "s_norm", "omega_hat", "measure"):
        assert rep[key] == float(g[key])


def test_inverse_cdf_known_answer():
    # reference tests/test_sampling.py:197-203
    idx, cnt = orc.cdf_draw(np.array([3, 7, 9]), np.array([0.2, 0.3, 0.5]),
                            np.array([0.05, 0.21, 0.45, 0.51, 0.99]))
    np.testing.assert_array_equal(idx, [3, 7, 9])
    np.testing.assert_array_equal(cnt, [1, 2, 2])


def test_cdf_edge_trailing_zero_unreachable():
    # reference tests/test_sampling.py:236-242
    idx, _ = orc.cdf_draw(np.array([0, 1, 2]), np.array([0.5, 0.5, 0.0]),
                          np.array([1.0 - 1e-16, 0.999999999]))
    np.testing.assert_array_equal(idx, [1])


def test_norm_ratio_weights():
    # reference tests/test_sampling.py:75-78: column norms 1:2 -> weights 0.2, 0.8
    a = np.array([[1.0, 2.0], [0.0, 0.0]])
    w = orc.normalized_weights(orc.column_norms2(a))
    np.testing.assert_allclose(w, [0.2, 0.8], rtol=1e-15)


def test_budget_formula():
    # reference tests/test_sampling.py:363-373 (acceptance 8): k=1, eps=1, delta=0.5
    assert orc.ltsvd_count(10, 0.7, 0.6) == 746
    assert orc.ltsvd_count(20, 0.7, 0.6) == 1491


def _cfg1_weights():
    a1 = workloads.config1(seed=0)
    return a1, np.arange(a1.shape[1]), orc.normalized_weights(orc.column_norms2(a1))


@pytest.mark.parametrize("dedup", [True, False])
def test_single_round_baselines_match_reference(dedup):
    """oracle ltsvd / ctsvd (baselines.py:68-142) == the reference run in
    make_golden.py: identical draws, factors to rounding."""
    g = load_golden("baselines")
    a1, cand, wts = _cfg1_weights()
    key = f"lt{int(dedup)}"
    u, s, (idx, cnt) = orc.ltsvd(a1, cand, wts, 10, 50, np.random.default_rng(3), dedup)
    assert np.array_equal(idx, g[f"{key}_idx"]) and np.array_equal(cnt, g[f"{key}_cnt"])
    np.testing.assert_allclose(s, g[f"{key}_s"], rtol=1e-12)
    np.testing.assert_allclose(u, g[f"{key}_u"], atol=1e-10)
    for tag, eps in (("ct", 0.7), ("ctf", 30.0)):
        key = f"{tag}{int(dedup)}"
        u, s = orc.ctsvd(a1, cand, wts, 10, 60, 300, eps, np.random.default_rng(4), dedup)
        assert s.size == g[f"{key}_s"].size
        np.testing.assert_allclose(s, g[f"{key}_s"], rtol=1e-12)
        np.testing.assert_allclose(u, g[f"{key}_u"], atol=1e-9)
    assert g["ctf1_s"].size < 10  # the energy filter case really filters


def test_exact_factorizations_match_reference():
    g = load_golden("baselines")
    for name in ("tall", "wide", "skinny"):
        u, s, v = orc.dense_svd(g[f"svd_{name}_a"])
        np.testing.assert_allclose(s, g[f"svd_{name}_s"], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(u, g[f"svd_{name}_u"], atol=1e-9)
        np.testing.assert_allclose(v, g[f"svd_{name}_v"], atol=1e-9)
    u, s, v = orc.pod_via_gram(workloads.config1(seed=0), 10)
    np.testing.assert_allclose(s, g["gram_s"], rtol=1e-12)
    np.testing.assert_allclose(u, g["gram_u"], atol=1e-9)
    np.testing.assert_allclose(v, g["gram_v"], atol=1e-9)
