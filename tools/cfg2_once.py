"""One eager (unpipelined, no graphs) config-2 isma_run on the resident
device matrix -- a short ncu target with every hot kernel of a round."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads
from paper_1905_05107_b200.device import ColMat
dev = torch.device("cuda", 0)
at = workloads.config2_torch(7, 512, 2000, device=dev)
A = ColMat(at, 512 * 512)
cfg = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7)


class NoRollback:
    def __init__(self, seed):
        self.g = np.random.default_rng(seed)

    def random(self, k):
        return self.g.random(k)


f, tr = pod.isma_run(A, cfg, rng=NoRollback(7), use_graphs=False)
torch.cuda.synchronize()
print("ok", len(tr), f.sigma[:3])
