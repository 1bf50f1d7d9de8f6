import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200.device import get_ctx, dptr
rng = np.random.default_rng(0)
ctx = get_ctx()
for k in (1, 2, 3, 5, 8, 10):
    q = np.linalg.qr(rng.standard_normal((k, k)))[0]
    C = torch.as_tensor(np.asfortranarray(q).T.copy().reshape(-1), device=ctx.device)  # col-major
    C = torch.as_tensor(q.T.copy().reshape(-1), device=ctx.device)
    sv = torch.empty(k, dtype=torch.float64, device=ctx.device)
    ctx.svd_small(dptr(C), k, k, k, None, 1, sv, None, 1)
    s = sv.cpu().numpy()
    print(k, "1 - svd_small:", (1 - s).max(), "numpy:", (1 - np.linalg.svd(q, compute_uv=False)).max(),
          "colnorm:", (1 - np.linalg.norm(q, axis=0)).max())
    u = np.linalg.qr(rng.standard_normal((100, k)))[0]
    f = pod.TruncatedFactor(u, np.linspace(2, 1, k))
    print("   self angles (deg):", pod.principal_angles(f, f, k).max())
