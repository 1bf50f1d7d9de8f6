"""Probe the on-device small solvers: sweeps and time per call."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200.device import get_ctx, dptr

ctx = get_ctx()
dev = ctx.device
for g in (50, 100, 120, 200):
    rng = np.random.default_rng(g)
    d = rng.standard_normal((5 * g, g)) * np.exp(-np.arange(g) / 8.0)
    G = d.T @ d
    Gd = torch.as_tensor(np.asfortranarray(G).T.copy().reshape(-1), device=dev)
    sig = torch.empty(g, dtype=torch.float64, device=dev)
    T = torch.empty(g * g, dtype=torch.float64, device=dev)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ctx.gram_eigh(dptr(Gd), g, g, g, sig, dptr(T), g)
        info = ctx.read_info(3)
        t = time.perf_counter() - t0
    print(f"gram_eigh g={g}: {t*1e3:.3f} ms sweeps={info[2]} rank={info[0]}")
    E = rng.standard_normal((g, g)) * np.exp(-np.arange(g) / 8.0)
    Ed = torch.as_tensor(np.asfortranarray(E).T.copy().reshape(-1), device=dev)
    U = torch.empty(g * g, dtype=torch.float64, device=dev)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ctx.svd_small(dptr(Ed), g, g, g, None, 1, sig, None, 1)
        info = ctx.read_info(1)
        t = time.perf_counter() - t0
    print(f"svd_small(values) n={g}: {t*1e3:.3f} ms sweeps={info[0]}")
