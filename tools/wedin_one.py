"""One fused Wedin call at a given shape (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_05107_b200.device import ColMat, get_ctx  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
ctx = get_ctx()
dev = ctx.device
at = torch.randn((n, m), dtype=torch.float64, device=dev)
U = ColMat(torch.randn((k, m), dtype=torch.float64, device=dev), m)
V = ColMat(torch.randn((k, n), dtype=torch.float64, device=dev), n)
s = torch.linspace(5.0, 1.0, k, dtype=torch.float64, device=dev)
out = torch.zeros(2, dtype=torch.float64, device=dev)
for _ in range(2):
    ctx.wedin(ColMat(at, m), U, V, s, k, out)
torch.cuda.synchronize()
print(out.cpu().numpy())
