import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads, isma as im
a = workloads.config1(seed=0)
for k in (10, 20):
    cfg = pod.IsmaConfig(k=k, seed=0)
    for i in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        f, tr = pod.isma_run(a, cfg)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    st = im.LAST_STATS
    print(f"k={k} c={cfg.column_budget()} rounds {len(tr)} {dt*1e3:.1f} ms; eigh sweeps {st.get('eigh_sweeps', [])[:5]} merge sweeps {st.get('merge_sweeps', [])[:5]}")
