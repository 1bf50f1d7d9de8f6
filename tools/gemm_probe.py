"""Time the FP64 DMMA GEMMs on the shapes of a config-2 (default) or
config-3 (argv[1] == "3") round."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200.device import get_ctx, dptr, ColMat
ctx = get_ctx(); dev = ctx.device
m, n, r, g = (1_000_000, 2000, 150, 200) if sys.argv[1:] == ["3"] else (262144, 2000, 60, 100)
A = ColMat(torch.randn((n, m), dtype=torch.float64, device=dev), m)
U1 = ColMat(torch.randn((2 * r, m), dtype=torch.float64, device=dev), m)
U2 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
W = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
idx = torch.as_tensor(np.sort(np.random.default_rng(0).choice(n, g, replace=False)).astype(np.int32), device=dev)
C = torch.empty(4 * n * r, dtype=torch.float64, device=dev)
T = torch.randn(4 * r * r, dtype=torch.float64, device=dev)
Tg = torch.randn(g * r, dtype=torch.float64, device=dev)
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
cases = [
 ("tn U1^T U2 rxr", lambda: ctx.tn(r, r, 1.0, U1.cols(0, r), U2, dptr(C), r), 2.0*m*r*r, 8.0*m*2*r),
 ("tn W^T W rxr (sym)", lambda: ctx.tn(r, r, 1.0, W, W, dptr(C), r), 1.0*m*r*(r+1), 8.0*m*r),
 ("tn gram gather gxg (sym)", lambda: ctx.tn(g, g, 1.0, A, A, dptr(C), g, xcols=idx, ycols=idx), 1.0*m*g*(g+1), 8.0*m*g),
 ("tn A^T U nxr", lambda: ctx.tn(n, r, 1.0, A, U2, dptr(C), n), 2.0*m*n*r, 8.0*m*(n+r)),
 ("nn resid r->r (beta)", lambda: ctx.nn(r, r, -1.0, U1.cols(0, r), dptr(T), r, W, beta=1.0, Z=U2), 2.0*m*r*r, 8.0*m*3*r),
 ("nn lift gather g->r", lambda: ctx.nn(g, r, 1.0, A, dptr(Tg), g, W, xcols=idx), 2.0*m*g*r, 8.0*m*(g+r)),
 ("nn rotate 2r->r", lambda: ctx.nn(2 * r, r, 1.0, U1, dptr(T), 2 * r, W), 2.0*m*2*r*r, 8.0*m*3*r),
 ("nn inplace r->r", lambda: ctx.nn(r, r, 1.0, W, dptr(T), r, W), 2.0*m*r*r, 8.0*m*2*r),
]
for name, fn, fl, by in cases:
    us = t(fn)
    print(f"{name:28s} {us:8.1f} us  {fl/us/1e6:6.2f} TF/s  {by/us/1e3:7.1f} GB/s  (roof {max(fl/37.17e12, by/6.55e12)*1e6:6.1f} us)")
