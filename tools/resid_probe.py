"""Residual W = U2 - U1 M (beta = 1 epilogue) against the plain product of
the same shape, config-3/4 sizes: device time of the streamed NN kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1905_05107_b200.device import ColMat, dptr, get_ctx
ctx = get_ctx(); dev = ctx.device


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for m, r in ((1_000_000, 150), (1_048_576, 192)):
    U1 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
    U2 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
    W = ColMat.zeros(m, r, dev)
    T = torch.randn(r * r, dtype=torch.float64, device=dev)
    t_res = timeit(lambda: ctx.nn(r, r, -1.0, U1, dptr(T), r, W, beta=1.0, Z=U2))
    ref = (U2.t[:, :4096].T - U1.t[:, :4096].T @ T.reshape(r, r).T)
    err = (W.t[:, :4096].T - ref).abs().max().item()
    t_pl = timeit(lambda: ctx.nn(r, r, 1.0, U1, dptr(T), r, W))
    print(f"m={m} r={r}: residual {t_res:.3f} ms, plain {t_pl:.3f} ms, check {err:.1e}")
