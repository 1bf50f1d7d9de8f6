"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference is only mounted here):

    python tests/golden/make_golden.py

It imports ``podsketch`` read-only from /root/reference/pkg/src, records every
``sample_with_replacement`` draw (the reference's traces do not keep index
sets) by wrapping the name ``podsketch.isma.sample_with_replacement``, and
writes small ``.npz`` files next to this script.  The fixtures pin
``oracle/isma_oracle.py`` (tests/test_oracle_pins.py) and are the golden
vectors the GPU parity tests compare against.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import podsketch  # noqa: E402  (the reference)
import podsketch.isma as ref_isma  # noqa: E402
from paper_1905_05107_b200 import workloads  # noqa: E402

DRAWS = []
_orig_sample = ref_isma.sample_with_replacement


def _recording_sample(dist, count, rng):
    draw = _orig_sample(dist, count, rng)
    DRAWS.append((draw.unique_indices.copy(), draw.counts.copy()))
    return draw


ref_isma.sample_with_replacement = _recording_sample


def run_case(a, cfg, keep=None, rng=None):
    DRAWS.clear()
    factor, traces = podsketch.isma_run(a, cfg, rng=rng, keep=keep)
    out = {
        "u": factor.u,
        "sigma": factor.sigma,
        "v": factor.v if factor.v is not None else np.zeros((0, 0)),
        "n_rounds": np.int64(len(traces)),
        "remaining": np.array([t.remaining for t in traces], dtype=np.int64),
        "columns_sampled": np.array([t.columns_sampled for t in traces], dtype=np.int64),
        "rows_sampled": np.array([t.rows_sampled for t in traces], dtype=np.int64),
        "cosines": np.array([np.pad(t.cosines, (0, cfg.k - t.cosines.size))
                             for t in traces]),
    }
    flat_idx = np.concatenate([d[0] for d in DRAWS])
    flat_cnt = np.concatenate([d[1] for d in DRAWS])
    offsets = np.cumsum([0] + [d[0].size for d in DRAWS]).astype(np.int64)
    out.update(draw_idx=flat_idx, draw_cnt=flat_cnt, draw_off=offsets)
    return out


def make_low_rank(m, n, k, rng, sigma=None):
    # same construction as the reference conftest (tests/conftest.py:10-22)
    if sigma is None:
        sigma = np.arange(k, 0, -1, dtype=np.float64)
    u = np.linalg.qr(rng.standard_normal((m, k)))[0]
    v = np.linalg.qr(rng.standard_normal((n, k)))[0]
    return (u * np.asarray(sigma, dtype=np.float64)) @ v.T


def main():
    cases = {}
    # BASELINE config 1 (data seed 0), tau = 1 - tol, seed 7
    a1 = workloads.config1(seed=0)
    cfg = podsketch.IsmaConfig(k=10, r=30, c=50, tau=1 - 1e-8, strategy="l2n",
                               criterion="modes", seed=7)
    cases["cfg1_l2n_modes"] = (a1, cfg, None)
    cases["cfg1_unf_subspace"] = (a1, podsketch.IsmaConfig(
        k=10, r=30, c=50, tau=0.99, strategy="unf", criterion="subspace", seed=3), None)
    cases["cfg1_l2n_nofinal_keep11"] = (a1, podsketch.IsmaConfig(
        k=10, r=30, c=50, tau=0.999, strategy="l2n", seed=5, finalize=False), 11)
    # reference-test-shaped small cases
    cases["rank3_unf"] = (make_low_rank(100, 60, 3, np.random.default_rng(7)),
                          podsketch.IsmaConfig(k=3, strategy="unf", tau=0.99, seed=11), None)
    cases["rank3_l2n"] = (make_low_rank(100, 60, 3, np.random.default_rng(7)),
                          podsketch.IsmaConfig(k=3, strategy="l2n", tau=0.99, seed=11), None)
    gen = np.random.default_rng(13)
    cases["exhaustive_40x18"] = (gen.standard_normal((40, 18)), podsketch.IsmaConfig(
        k=5, r=18, strategy="l2n", tau=1.0, c=60, seed=2), None)
    cases["cfg1_ort_modes"] = (a1, podsketch.IsmaConfig(
        k=10, r=30, c=50, tau=0.999, strategy="ort", seed=5), None)
    cases["rank3_ort_fallback"] = (make_low_rank(60, 30, 3, np.random.default_rng(10)),
                                   podsketch.IsmaConfig(k=3, strategy="ort", tau=0.99, c=100,
                                                        seed=5), None)
    # config-2 generator proxy (64 x 64 grid, n=300)
    a2 = workloads.config2(seed=1, side=64, n=300)
    cases["cfg2proxy_l2n"] = (a2, podsketch.IsmaConfig(
        k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7), None)

    # ICRS row sampling (rows=True): reference-test-shaped rank-3 cases for
    # every row strategy, and config-1 runs with explicit row budgets
    for strat in ("unf", "ort", "ls"):
        cases[f"rank3_{strat}_rows"] = (
            make_low_rank(100, 60, 3, np.random.default_rng(7)),
            podsketch.IsmaConfig(k=3, strategy=strat, rows=True, tau=0.99, seed=11), None)
    cases["cfg1_ls_rows"] = (a1, podsketch.IsmaConfig(
        k=10, r=30, c=50, w=400, tau=0.999, strategy="ls", rows=True, seed=5), None)
    cases["cfg1_unf_rows_subspace"] = (a1, podsketch.IsmaConfig(
        k=10, r=30, c=50, w=300, tau=0.99, strategy="unf", rows=True, criterion="subspace",
        seed=4), None)

    for name, (a, cfg, keep) in cases.items():
        out = run_case(a, cfg, keep=keep)
        meta = np.array([cfg.k, cfg.r, cfg.column_budget(), int(cfg.finalize),
                         -1 if keep is None else keep,
                         cfg.row_budget() if cfg.rows else 0], dtype=np.int64)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), meta=meta,
                            tau=np.float64(cfg.tau), strategy=cfg.strategy,
                            criterion=cfg.criterion, seed=np.int64(cfg.seed), **out)
        print(name, "rounds", len(out["remaining"]), "sigma0", out["sigma"][0])

    # merge fixtures (merge.py:37-91) on seeded random factors
    rng = np.random.default_rng(1234)
    mats = {}
    for i, (m, k1, k2, r) in enumerate([(40, 10, 10, 20), (50, 5, 5, 10), (30, 8, 8, 2),
                                          (200, 30, 30, 30)]):
        x = rng.standard_normal((m, k1))
        y = rng.standard_normal((m, k2))
        f1 = podsketch.dense_svd(x)
        f2 = podsketch.dense_svd(y)
        f1 = podsketch.TruncatedFactor(f1.u, f1.sigma)
        f2 = podsketch.TruncatedFactor(f2.u, f2.sigma)
        mg = podsketch.block_merge(f1, f2, r)
        mats[f"m{i}_u1"] = f1.u
        mats[f"m{i}_s1"] = f1.sigma
        mats[f"m{i}_u2"] = f2.u
        mats[f"m{i}_s2"] = f2.sigma
        mats[f"m{i}_r"] = np.int64(r)
        mats[f"m{i}_u"] = mg.u
        mats[f"m{i}_s"] = mg.sigma
    np.savez_compressed(os.path.join(HERE, "merges.npz"), **mats)

    # one-pass incremental (ooc.py:105-148) on a PODM file, t = 3
    import tempfile

    a3 = workloads.config1(seed=2, m=300, n=120)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "a.podm")
        podsketch.write_matrix(path, a3)
        cfg = podsketch.IsmaConfig(k=4, c=20, tau=0.999, strategy="l2n", seed=9)
        with podsketch.BlockReader(path, 3) as rd:
            f, tr = podsketch.incremental_pod(rd, cfg)
    np.savez_compressed(os.path.join(HERE, "incremental_t3.npz"), u=f.u, sigma=f.sigma,
                        remaining=np.array([t.remaining for t in tr], dtype=np.int64),
                        seed=np.int64(2))

    # single-round baselines (baselines.py:68-142) and exact factorizations
    # (matcore.py:187-254); draws recorded through the baselines module's name
    import podsketch.baselines as ref_base

    ref_base.sample_with_replacement = _recording_sample
    base = {}
    dist = podsketch.column_norm_distribution(a1)
    for tag, fn in (
            ("lt", lambda dd: podsketch.ltsvd(a1, dist, 10, 50, np.random.default_rng(3),
                                              dedup=dd)),
            ("ct", lambda dd: podsketch.ctsvd(a1, dist, 10, 60, 300, 0.7,
                                              np.random.default_rng(4), dedup=dd)),
            ("ctf", lambda dd: podsketch.ctsvd(a1, dist, 10, 60, 300, 30.0,
                                               np.random.default_rng(4), dedup=dd))):
        for dd in (True, False):
            DRAWS.clear()
            f = fn(dd)
            key = f"{tag}{int(dd)}"
            base[f"{key}_u"], base[f"{key}_s"] = f.u, f.sigma
            base[f"{key}_idx"] = DRAWS[0][0]
            base[f"{key}_cnt"] = DRAWS[0][1]
    gen = np.random.default_rng(21)
    mats = {"tall": gen.standard_normal((300, 40)), "wide": gen.standard_normal((40, 300)),
            "skinny": gen.standard_normal((5000, 30)) * np.logspace(0, -6, 30)}
    for name, x in mats.items():
        f = podsketch.dense_svd(x)
        base[f"svd_{name}_a"], base[f"svd_{name}_u"] = x, f.u
        base[f"svd_{name}_s"], base[f"svd_{name}_v"] = f.sigma, f.v
    f = podsketch.pod_via_gram(a1, 10)
    base["gram_u"], base["gram_s"], base["gram_v"] = f.u, f.sigma, f.v
    q, rr = podsketch.matcore.thin_qr(mats["tall"])
    base["qr_q"], base["qr_r"] = q, rr
    near = np.linalg.qr(gen.standard_normal((300, 20)))[0] + 1e-7 * gen.standard_normal((300, 20))
    q, sv = podsketch.matcore.orthonormalize(near)
    base["orth_in"], base["orth_q"], base["orth_s"] = near, q, sv
    np.savez_compressed(os.path.join(HERE, "baselines.npz"), **base)

    # Wedin report (quality.py:82-118) for the config-1 finalized factor, keep=k+1
    cfg = podsketch.IsmaConfig(k=10, r=30, c=50, tau=0.99, strategy="l2n", seed=7)
    f, _ = podsketch.isma_run(a1, cfg, keep=11)
    rep = podsketch.wedin_measure(a1, f, 10)
    np.savez_compressed(os.path.join(HERE, "wedin_cfg1.npz"), u=f.u, sigma=f.sigma, v=f.v,
                        r_norm=rep.r_norm, s_norm=rep.s_norm, omega_hat=rep.omega_hat,
                        measure=rep.measure)
    print("done")


if __name__ == "__main__":
    main()
