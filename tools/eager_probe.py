import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads
from paper_1905_05107_b200.device import ColMat
dev = torch.device("cuda", 0)
at = workloads.config2_torch(7, 512, 2000, device=dev)
A = ColMat(at, 512 * 512)
cfg = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7)
class NoRB:
    def __init__(s, seed): s.g = np.random.default_rng(seed)
    def random(s, k): return s.g.random(k)
for graphs in (True, False):
    for rngk in ("gen", "norb"):
        ts = []
        for i in range(4):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            pod.isma_run(A, cfg, use_graphs=graphs, rng=None if rngk == "gen" else NoRB(7))
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        print(f"graphs={graphs} rng={rngk}: {min(ts[1:]):.4f} s")
