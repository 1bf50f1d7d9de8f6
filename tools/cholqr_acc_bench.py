"""Device time of the l = 60 CholeskyQR factor: plain, with Racc
accumulation, and on Grams of growing condition number (shift retries)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_05107_b200.device import dptr, get_ctx  # noqa: E402

ctx = get_ctx()
dev = ctx.device
l = 60
for cond in (1e0, 1e4, 1e7, 1e9):
    rng = np.random.default_rng(1)
    q, _ = np.linalg.qr(rng.standard_normal((4 * l, l)))
    w = q * np.logspace(0, -np.log10(cond), l)
    G = torch.as_tensor((w.T @ w).T.copy().reshape(-1), device=dev)
    Rinv = torch.empty(l * l, dtype=torch.float64, device=dev)
    R = torch.empty(l * l, dtype=torch.float64, device=dev)
    Racc = torch.eye(l, dtype=torch.float64, device=dev).reshape(-1)
    for acc in (0, 1):
        def call():
            if acc:
                ctx.cholqr_factor_acc(dptr(G), l, l, 4 * l, dptr(Rinv), l, 0, l, dptr(Racc), l)
            else:
                ctx.cholqr_factor(dptr(G), l, l, 4 * l, dptr(Rinv), l, dptr(R), l)
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            call()
        e1.record()
        torch.cuda.synchronize()
        di = ctx.dinfo[:4].cpu().numpy()
        print(f"cond {cond:.0e} acc {acc}: {e0.elapsed_time(e1) / 50 * 1e3:7.1f} us/call, "
              f"defect {di[0]:.1e} attempts {int(di[1])} shift {di[3]:.1e}")
