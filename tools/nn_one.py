"""Config-2 NN shapes once each after a warm-up (ncu target):
argv: resid | inplace | rotate | lift"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200.device import ColMat, dptr, get_ctx
ctx = get_ctx(); dev = ctx.device
m, n, r, g = 262144, 2000, 60, 100
S = ColMat(torch.randn((2 * r, m), dtype=torch.float64, device=dev), m)
U2 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
W = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
A = ColMat(torch.randn((n, m), dtype=torch.float64, device=dev), m)
idx = torch.as_tensor(np.sort(np.random.default_rng(0).choice(n, g, replace=False)).astype(np.int32), device=dev)
T = torch.randn(4 * r * r, dtype=torch.float64, device=dev)
Tg = torch.randn(g * r, dtype=torch.float64, device=dev)
op = sys.argv[1]
for _ in range(2):
    if op == "resid":
        ctx.nn(r, r, -1.0, S.cols(0, r), dptr(T), r, W, beta=1.0, Z=U2)
    elif op == "inplace":
        ctx.nn(r, r, 1.0, W, dptr(T), r, W)
    elif op == "rotate":
        ctx.nn(2 * r, r, 1.0, S, dptr(T), 2 * r, W)
    else:
        ctx.nn(g, r, 1.0, A, dptr(Tg), g, W, xcols=idx)
torch.cuda.synchronize()
print("ok")
