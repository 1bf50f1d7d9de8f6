"""One svd_small call on a 120 x 120 graded matrix (ncu target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200.device import get_ctx, dptr
ctx = get_ctx(); dev = ctx.device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 120
E = torch.as_tensor((np.random.default_rng(0).standard_normal((n, n)) * np.exp(-np.arange(n) / 8.0)).reshape(-1), device=dev)
s = torch.empty(n, dtype=torch.float64, device=dev)
for _ in range(2):
    ctx.svd_small(dptr(E), n, n, n, None, 1, s, None, 1)
torch.cuda.synchronize()
print("ok", ctx.read_info(1))
