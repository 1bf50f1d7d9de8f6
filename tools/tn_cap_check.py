"""TN X^T Y at the merge shapes under different grid caps (pod_set_grid_cap)
against torch's fp64 product: the capped plans must give the same C."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1905_05107_b200 import _lib
from paper_1905_05107_b200.device import ColMat, dptr, get_ctx
ctx = get_ctx()
dev = ctx.device
lib = _lib.load()
for m, p in ((262144, 60), (1_000_000, 150), (1 << 20, 192)):
    g = torch.Generator(device=dev); g.manual_seed(p)
    xt = torch.randn((p, m), dtype=torch.float64, device=dev, generator=g)
    yt = torch.randn((p, m), dtype=torch.float64, device=dev, generator=g)
    X, Y = ColMat(xt, m), ColMat(yt, m)
    ref = (xt @ yt.T).T.contiguous().reshape(-1)  # C col-major = (X^T Y) stored column by column
    for cap in (0, 8, 16, 32, 64, 100, 148):
        C = torch.zeros(p * p, dtype=torch.float64, device=dev)
        lib.pod_set_grid_cap(cap)
        ctx.tn(p, p, 1.0, X, Y, dptr(C), p)
        lib.pod_set_grid_cap(0)
        torch.cuda.synchronize()
        err = (C - ref).abs().max().item() / ref.abs().max().item()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        lib.pod_set_grid_cap(cap)
        e0.record()
        for _ in range(5):
            ctx.tn(p, p, 1.0, X, Y, dptr(C), p)
        e1.record()
        lib.pod_set_grid_cap(0)
        torch.cuda.synchronize()
        print(f"m={m} p={p} cap={cap:3d}: rel err {err:.2e}  {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
    del xt, yt
