"""Device time of the shared-memory (packed, in-place) CholeskyQR factor at
the config-3/4 merge ranks (l = 150, 192) and its edges."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_05107_b200.device import dptr, get_ctx  # noqa: E402

ctx = get_ctx()
dev = ctx.device
for l in (104, 150, 192, 230):
    rng = np.random.default_rng(1)
    q, _ = np.linalg.qr(rng.standard_normal((4 * l, l)))
    w = q * np.logspace(0, -3, l)
    G = torch.as_tensor((w.T @ w).T.copy().reshape(-1), device=dev)
    Rinv = torch.empty(l * l, dtype=torch.float64, device=dev)
    R = torch.empty(l * l, dtype=torch.float64, device=dev)

    def call():
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
    Rn = R.cpu().numpy().reshape(l, l).T
    err = np.abs(Rn.T @ Rn - w.T @ w).max() / np.abs(w.T @ w).max()
    print(f"l {l}: {e0.elapsed_time(e1) / 50 * 1e3:7.1f} us/call, |R^T R - G| rel {err:.1e}")
