import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_1905_05107_b200 as pod
from conftest import make_low_rank
a = make_low_rank(100, 60, 3, np.random.default_rng(7))
for graphs in (False, True):
    for strat in ("l2n", "unf"):
        cfg = pod.IsmaConfig(k=3, strategy=strat, tau=0.99, seed=11)
        f, tr = pod.isma_run(a, cfg, use_graphs=graphs)
        import torch; torch.cuda.synchronize()
        print("graphs", graphs, strat, "ok", f.sigma, flush=True)
