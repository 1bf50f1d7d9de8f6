"""Kernel reads of page-locked host memory (zero-copy) vs DMA: norm pass and
sampled-column gather on the config-2 matrix."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200 import workloads
from paper_1905_05107_b200.device import ColMat, get_ctx
ctx = get_ctx(); dev = ctx.device
at = workloads.config2_torch(7, 512, 2000, device=dev)
n, m = at.shape
h = torch.empty((n, m), dtype=torch.float64, pin_memory=True); h.copy_(at)
A = ColMat(h, m)
norms = torch.empty(n, dtype=torch.float64, device=dev); flag = torch.zeros(1, dtype=torch.int32, device=dev)
def t(fn, reps=3):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
gb = n * m * 8 / 1e9
print(f"colnorms over host-mapped A: {gb / t(lambda: ctx.colnorms2(A, norms, flag)):.1f} GB/s")
d = torch.empty((n, m), dtype=torch.float64, device=dev)
print(f"DMA H2D copy: {gb / t(lambda: d.copy_(h, non_blocking=True)):.1f} GB/s")
idx = torch.as_tensor(np.sort(np.random.default_rng(0).choice(n, 100, replace=False)).astype(np.int32), device=dev)
D = ColMat.zeros(m, 100, dev)
print(f"gather 100 columns from host: {100 * m * 8 / 1e9 / t(lambda: ctx.gather_cols(A, idx, 100, D)):.1f} GB/s")
