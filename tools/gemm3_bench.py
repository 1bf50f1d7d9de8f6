"""Config-3 GEMM shapes (m = 1M, r = 150, g = 200, n = 20000 for finalize),
CUDA-event timed: NN (resid, apply, rotate, lift) and TN (gram, proj, gathered
gram, leak-shaped) -- A/B of kernel variants via POD_* switches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200.device import ColMat, dptr, get_ctx
ctx = get_ctx(); dev = ctx.device
m, n, r, g = (262144, 2000, 60, 100) if os.environ.get("CFG") == "2" else (1_000_000, 2000, 150, 200)
S = ColMat(torch.randn((2 * r, m), dtype=torch.float64, device=dev), m)
U2 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
W = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
W2 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
A = ColMat(torch.randn((n, m), dtype=torch.float64, device=dev), m)
idx = torch.as_tensor(np.sort(np.random.default_rng(0).choice(n, g, replace=False)).astype(np.int32), device=dev)
T = torch.randn(4 * r * r, dtype=torch.float64, device=dev)
Tg = torch.randn(g * r, dtype=torch.float64, device=dev)
C = torch.empty(4 * n * r, dtype=torch.float64, device=dev)
ops = {"resid": (lambda: ctx.nn(r, r, -1.0, S.cols(0, r), dptr(T), r, W, beta=1.0, Z=U2), 2 * m * r * r),
       "apply": (lambda: ctx.nn(r, r, 1.0, W2, dptr(T), r, W), 2 * m * r * r),
       "inplace": (lambda: ctx.nn(r, r, 1.0, W2, dptr(T), r, W2), 2 * m * r * r),
       "rotate": (lambda: ctx.nn(2 * r, r, 1.0, S, dptr(T), 2 * r, W), 4 * m * r * r),
       "lift": (lambda: ctx.nn(g, r, 1.0, A, dptr(Tg), g, W, xcols=idx), 2 * m * g * r),
       "tgram": (lambda: ctx.tn(r, r, 1.0, W2, W2, dptr(C), r), m * r * (r + 1)),
       "tproj": (lambda: ctx.tn(r, r, 1.0, S.cols(0, r), U2, dptr(C), r), 2 * m * r * r),
       "tgath": (lambda: ctx.tn(g, g, 1.0, A, A, dptr(C), g, xcols=idx, ycols=idx), m * g * (g + 1))}
sel = sys.argv[1].split(",") if len(sys.argv) > 1 else list(ops)
for name in sel:
    fn, fl = ops[name]
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name}: {ms:.3f} ms, {fl / ms / 1e9:.1f} TF/s")
