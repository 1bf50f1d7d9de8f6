"""Device time of pod_cholqr_factor vs l (CUDA events over repeated calls)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_05107_b200.device import dptr, get_ctx  # noqa: E402

ctx = get_ctx()
dev = ctx.device
for l in (8, 16, 32, 48, 60, 64, 96, 150, 192):
    rng = np.random.default_rng(l)
    w = rng.standard_normal((4 * l, l))
    G = torch.as_tensor((w.T @ w).T.copy().reshape(-1), device=dev)
    Rinv = torch.empty(l * l, dtype=torch.float64, device=dev)
    R = torch.empty(l * l, dtype=torch.float64, device=dev)
    for _ in range(3):
        ctx.cholqr_factor(dptr(G), l, l, 4 * l, dptr(Rinv), l, dptr(R), l)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        ctx.cholqr_factor(dptr(G), l, l, 4 * l, dptr(Rinv), l, dptr(R), l)
    e1.record()
    torch.cuda.synchronize()
    Rh = R.view(l, l).cpu().numpy().T
    Ri = Rinv.view(l, l).cpu().numpy().T
    err = np.abs(Rh @ Ri - np.eye(l)).max()
    ref = np.linalg.cholesky(w.T @ w).T
    print(f"l={l:3d}: {e0.elapsed_time(e1) / 50 * 1e3:7.1f} us/call, |R Rinv - I| {err:.1e}, "
          f"|R - chol| {np.abs(Rh - ref).max() / np.abs(ref).max():.1e}")
