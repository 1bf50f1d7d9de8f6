"""Launch each cfg-3-shaped FP64 GEMM twice (ncu target; no timing)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200.device import get_ctx, dptr, ColMat
ctx = get_ctx(); dev = ctx.device
m, r = 1_000_000, 150
U1 = ColMat(torch.randn((2 * r, m), dtype=torch.float64, device=dev), m)
U2 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
W = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
C = torch.empty(4 * r * r, dtype=torch.float64, device=dev)
T = torch.randn(4 * r * r, dtype=torch.float64, device=dev)
for _ in range(2):
    ctx.tn(r, r, 1.0, U1.cols(0, r), U2, dptr(C), r)
for _ in range(2):
    ctx.nn(r, r, -1.0, U1.cols(0, r), dptr(T), r, W, beta=1.0, Z=U2)
torch.cuda.synchronize()
print("ok")
