"""gram_eigh on a sampled config-2-like Gram (ncu launch-time target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200.device import get_ctx, dptr
ctx = get_ctx(); dev = ctx.device
g = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(0)
D = rng.standard_normal((4000, g)) * np.exp(-np.arange(g) / 10.0)
G = torch.as_tensor(np.asfortranarray(D.T @ D).T.copy().reshape(-1), device=dev)
sig = torch.empty(g, dtype=torch.float64, device=dev)
T = torch.empty(g * g, dtype=torch.float64, device=dev)
for _ in range(3):
    ctx.gram_eigh(dptr(G), g, g, g // 2, sig, dptr(T), g)
torch.cuda.synchronize()
print("ok", ctx.read_info(3))
