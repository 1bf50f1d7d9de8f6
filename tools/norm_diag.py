"""Diagnose the einsum-order norm kernel: chain speed vs column count."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1905_05107_b200.device import ColMat, get_ctx
ctx = get_ctx(); dev = ctx.device
m = 262144
for n in (1, 50, 148, 296, 1000, 2000):
    t = torch.randn((n, m), dtype=torch.float64, device=dev)
    A = ColMat(t, m, n)
    nrm = torch.empty(n, dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    ctx.colnorms2(A, nrm, flag); ctx.colnorms2(A, nrm, flag)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ctx.colnorms2(A, nrm, flag)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"m={m} n={n}: {ms:.3f} ms, {ms*1e-3*1.965e9/(m/2):.1f} cycles per dependent add")
