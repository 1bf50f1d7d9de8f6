"""Two block_merge calls at r = 60 (merge_core on a 120 x 120 E; ncu target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_05107_b200 as pod
r = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(0)
m = 4 * r
f1 = pod.TruncatedFactor(*np.linalg.svd(rng.standard_normal((m, r)) * np.exp(-np.arange(r) / 8.0), full_matrices=False)[:2])
f2 = pod.TruncatedFactor(*np.linalg.svd(rng.standard_normal((m, r)), full_matrices=False)[:2])
for _ in range(2):
    mg = pod.block_merge(f1, f2, r)
torch.cuda.synchronize()
print("ok", mg.nmodes)
