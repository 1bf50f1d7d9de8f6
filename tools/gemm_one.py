"""Launch cfg-3-shaped FP64 GEMMs (ncu target; no timing):
resid (beta), rotate 2r->r, lift gather g->r, in-place r->r, each twice."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200.device import get_ctx, dptr, ColMat
ctx = get_ctx(); dev = ctx.device
m, r, g, n = 1_000_000, 150, 200, 2000
U1 = ColMat(torch.randn((2 * r, m), dtype=torch.float64, device=dev), m)
U2 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
W = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
A = ColMat(torch.randn((n, m), dtype=torch.float64, device=dev), m)
idx = torch.as_tensor(np.sort(np.random.default_rng(0).choice(n, g, replace=False)).astype(np.int32), device=dev)
C = torch.empty(4 * r * r, dtype=torch.float64, device=dev)
T = torch.randn(4 * r * r, dtype=torch.float64, device=dev)
Tg = torch.randn(g * r, dtype=torch.float64, device=dev)
which = sys.argv[1:] or ["resid", "rotate", "lift", "inplace", "tn"]
for _ in range(2):
    if "tn" in which:
        ctx.tn(r, r, 1.0, U1.cols(0, r), U2, dptr(C), r)
    if "resid" in which:
        ctx.nn(r, r, -1.0, U1.cols(0, r), dptr(T), r, W, beta=1.0, Z=U2)
    if "rotate" in which:
        ctx.nn(2 * r, r, 1.0, U1, dptr(T), 2 * r, W)
    if "lift" in which:
        ctx.nn(g, r, 1.0, A, dptr(Tg), g, W, xcols=idx)
    if "inplace" in which:
        ctx.nn(r, r, 1.0, W, dptr(T), r, W)
torch.cuda.synchronize()
print("ok")
