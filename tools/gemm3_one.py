"""Config-3 GEMM shapes (m = 1M, r = 150, g = 200), each op once after one
warm-up call -- the `ncu --set full` target for the config-3 GEMM kernels.
argv: comma list of resid | apply | rotate | lift | gram | tnproj"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200.device import ColMat, dptr, get_ctx
ctx = get_ctx(); dev = ctx.device
m, n, r, g = 1_000_000, 2000, 150, 200
S = ColMat(torch.randn((2 * r, m), dtype=torch.float64, device=dev), m)
U2 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
W = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
W2 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
A = ColMat(torch.randn((n, m), dtype=torch.float64, device=dev), m)
idx = torch.as_tensor(np.sort(np.random.default_rng(0).choice(n, g, replace=False)).astype(np.int32), device=dev)
T = torch.randn(4 * r * r, dtype=torch.float64, device=dev)
Tg = torch.randn(g * r, dtype=torch.float64, device=dev)
C = torch.empty(4 * n * r, dtype=torch.float64, device=dev)
ops = {"resid": lambda: ctx.nn(r, r, -1.0, S.cols(0, r), dptr(T), r, W, beta=1.0, Z=U2),
       "apply": lambda: ctx.nn(r, r, 1.0, W2, dptr(T), r, W),
       "rotate": lambda: ctx.nn(2 * r, r, 1.0, S, dptr(T), 2 * r, W),
       "lift": lambda: ctx.nn(g, r, 1.0, A, dptr(Tg), g, W, xcols=idx),
       "gram": lambda: ctx.tn(r, r, 1.0, W2, W2, dptr(C), r),
       "tnproj": lambda: ctx.tn(r, r, 1.0, W2, U2, dptr(C), r)}
for name in sys.argv[1].split(","):
    ops[name]()
    torch.cuda.synchronize()
    ops[name]()
    torch.cuda.synchronize()
print("ok")
