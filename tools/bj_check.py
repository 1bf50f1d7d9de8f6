"""Block-Jacobi smoke: block_merge / svd / isma_run vs the oracle, and timing
of merge_core against the row-distributed cluster solver (POD_JACOBI=cluster)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_05107_b200 as pod
from oracle import isma_oracle as orc
from paper_1905_05107_b200 import workloads
from paper_1905_05107_b200 import isma as isma_mod
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from parity_util import principal_angles_sin, sigma_relerr

rng = np.random.default_rng(0)
for (m, k1, k2, r) in [(400, 60, 60, 60), (300, 30, 30, 30), (1000, 150, 150, 150), (200, 12, 12, 12)]:
    f1 = pod.TruncatedFactor(*np.linalg.svd(rng.standard_normal((m, k1)), full_matrices=False)[:2])
    f2 = pod.TruncatedFactor(*np.linalg.svd(rng.standard_normal((m, k2)), full_matrices=False)[:2])
    mg = pod.block_merge(f1, f2, r)
    u, s = orc.merge(f1.u, f1.sigma, f2.u, f2.sigma, r)
    print("merge", m, k1, r, "sig", sigma_relerr(mg.sigma, s), "ang", principal_angles_sin(mg.u, u).max(), flush=True)
a = workloads.config1(seed=0)
for crit in ("modes", "subspace"):
    cfg = pod.IsmaConfig(k=10, r=30, c=50, tau=1 - 1e-8, strategy="l2n", criterion=crit, seed=7)
    f, tr = pod.isma_run(a, cfg)
    o = orc.run(a, 10, r=30, c=50, tau=1 - 1e-8, strategy="l2n", criterion=crit, seed=7)
    print("cfg1", crit, len(tr), len(o["trace"]), sigma_relerr(f.sigma, o["sigma"]), principal_angles_sin(f.u, o["u"]).max(), isma_mod.LAST_STATS.get("merge_sweeps")[:5], isma_mod.LAST_STATS.get("eigh_sweeps")[:5], flush=True)
print("ok")
