"""Which small-solver sizes run: gram_eigh (g), svd_small (n x n with U, V),
and ISMA with the reference's default column budget on config 1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_05107_b200 as pod  # noqa: E402
from paper_1905_05107_b200 import workloads  # noqa: E402
from paper_1905_05107_b200.device import dptr, get_ctx  # noqa: E402

ctx = get_ctx()
dev = ctx.device
for g in (240, 300, 340, 384, 420, 460, 500, 512, 600, 800, 1024):
    a = torch.randn(g + 7, g, dtype=torch.float64, device=dev)
    G = (a.T @ a).contiguous().view(-1)
    sig = torch.empty(g, dtype=torch.float64, device=dev)
    T = torch.empty(g * g, dtype=torch.float64, device=dev)
    res = []
    try:
        ctx.gram_eigh(dptr(G), g, g, g, sig, dptr(T), g)
        torch.cuda.synchronize()
        ref = torch.linalg.eigvalsh(G.view(g, g)).flip(0).sqrt()
        res.append(f"gram_eigh ok err {float(((sig - ref).abs() / ref).max()):.1e}")
    except Exception as e:  # noqa: BLE001
        res.append(f"gram_eigh FAIL {str(e)[:60]}")
    U = torch.empty(g * g, dtype=torch.float64, device=dev)
    try:
        ctx.svd_small(dptr(G), g, g, g, dptr(U), g, sig, dptr(T), g)
        torch.cuda.synchronize()
        res.append("svd_small(U,V) ok")
    except Exception as e:  # noqa: BLE001
        res.append(f"svd_small FAIL {str(e)[:60]}")
    try:
        ctx.svd_small(dptr(G), g, g, g, None, 1, sig, dptr(T), g)
        torch.cuda.synchronize()
        res.append("svd_small(V) ok")
    except Exception as e:  # noqa: BLE001
        res.append(f"svd_small(V) FAIL {str(e)[:60]}")
    print(g, " | ".join(res), flush=True)

a1 = workloads.config1(seed=0)
try:
    f, tr = pod.isma_run(a1, pod.IsmaConfig(k=10, seed=0))
    print("cfg1 default c", pod.IsmaConfig(k=10).column_budget(), "rounds", len(tr),
          "g", [t.columns_sampled for t in tr][:4])
except Exception as e:  # noqa: BLE001
    print("cfg1 default c FAIL", e)
