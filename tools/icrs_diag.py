import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import engine, isma, workloads
from oracle import isma_oracle as orc
from parity_util import principal_angles_sin, sigma_relerr
a32 = workloads.config4(seed=3, side=64, n=300); a64 = a32.astype(np.float64)
for strat in ("ls", "unf", "ort"):
    for mat in (a32, a64):
        cfg = pod.IsmaConfig(k=12, r=36, c=40, tau=1 - 1e-8, strategy=strat, seed=5, rows=True, w=300)
        engine.RECORD_DRAWS = True
        f, tr = pod.isma_run(mat, cfg)
        log = isma.LAST_DRAWS
        engine.RECORD_DRAWS = False
        o = orc.run(a64, 12, r=36, c=40, tau=1 - 1e-8, strategy=strat, seed=5, rows=True, w=300)
        same_cols = all(np.array_equal(l[0], t["unique"]) for l, t in zip(log, o["trace"]))
        same_rows = all(np.array_equal(l[2], t["rows"]) for l, t in zip(log, o["trace"]))
        print(strat, mat.dtype, "rounds", len(tr), len(o["trace"]), "cols", same_cols, "rows", same_rows,
              "sigma", sigma_relerr(f.sigma, o["sigma"]), "angle", principal_angles_sin(f.u, o["u"]).max())
