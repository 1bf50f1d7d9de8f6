import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200.device import ColMat, dptr, get_ctx
ctx = get_ctx(); dev = ctx.device
K, n, r = 1 << 20, 8192, 192
a = torch.randn((n, K), dtype=torch.float32, device=dev)
A = ColMat(a, K, n)
hi = torch.randn((r, K), dtype=torch.float32, device=dev); lo = hi * 1e-4
C = torch.empty(n * r, dtype=torch.float64, device=dev)
for _ in range(2):
    ctx.tn_tf32x3(n, r, 1.0, A, ColMat(hi, K, r), dptr(C), n, Ylo=lo.reshape(-1))
torch.cuda.synchronize(); print("ok")
