"""Each hot kernel of a config-2 round once, on config-2 sized operands
(after one warm-up call each) -- the `ncu --set full` target for profiles/."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200 import workloads
from paper_1905_05107_b200.device import ColMat, dptr, get_ctx
ctx = get_ctx(); dev = ctx.device
m, n, r, g = 262144, 2000, 60, 100
at = workloads.config2_torch(7, 512, 2000, device=dev)
A = ColMat(at, m)
rng = np.random.default_rng(0)
idx = torch.as_tensor(np.sort(rng.choice(n, g, replace=False)).astype(np.int32), device=dev)
S = ColMat(torch.linalg.qr(torch.randn((m, 2 * r), dtype=torch.float64, device=dev))[0].T.contiguous(), m)
U2 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
W = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
C = torch.empty(4 * n * r, dtype=torch.float64, device=dev)
T = torch.randn(4 * r * r, dtype=torch.float64, device=dev)
Tg = torch.randn(g * r, dtype=torch.float64, device=dev)
norms = torch.empty(n, dtype=torch.float64, device=dev)
flag = torch.zeros(1, dtype=torch.int32, device=dev)
D = torch.empty((g, m), dtype=torch.float64, device=dev)
D.copy_(at[idx.long()])
G = (D @ D.T).T.contiguous().reshape(-1)
sig = torch.empty(g, dtype=torch.float64, device=dev)
Tl = torch.empty(g * r, dtype=torch.float64, device=dev)
sig1 = torch.linspace(10, 1, r, dtype=torch.float64, device=dev)
M = torch.randn(r * r, dtype=torch.float64, device=dev) * 0.1
R = torch.triu(torch.randn((r, r), dtype=torch.float64, device=dev)).T.contiguous().reshape(-1)
Tm = torch.empty(2 * r * r, dtype=torch.float64, device=dev)
sn = torch.empty(r, dtype=torch.float64, device=dev)
Wt = W.t[:r, :m]
Gq = (Wt @ Wt.T).T.contiguous().reshape(-1)
Rinv = torch.empty(r * r, dtype=torch.float64, device=dev)
Rk = torch.empty(r * r, dtype=torch.float64, device=dev)
live = torch.ones(n, dtype=torch.uint8, device=dev)
Gq2 = torch.empty(r * r, dtype=torch.float64, device=dev)
Uw = ColMat(torch.randn((20, m), dtype=torch.float64, device=dev), m)
Vw = ColMat(torch.randn((20, n), dtype=torch.float64, device=dev), n)
sw = torch.linspace(5.0, 1.0, 20, dtype=torch.float64, device=dev)
w2 = torch.empty(2, dtype=torch.float64, device=dev)
uni = torch.rand(c := 100, dtype=torch.float64, device=dev)
didx = torch.empty(g, dtype=torch.int32, device=dev)
dcnt = torch.empty(g, dtype=torch.int64, device=dev)
ops = [
    ("colnorms2", lambda: ctx.colnorms2(A, norms, flag)),
    ("draw", lambda: (live.fill_(1), ctx.draw(0, norms, live, n, uni, c, didx, dcnt))),
    ("tn_gram_gather", lambda: ctx.tn(g, g, 1.0, A, A, dptr(C), g, xcols=idx, ycols=idx)),
    ("tn_merge_proj", lambda: ctx.tn(r, r, 1.0, S.cols(0, r), U2, dptr(C), r)),
    ("tn_cholqr_gram", lambda: ctx.tn(r, r, 1.0, W, W, dptr(C), r)),
    ("nn_lift_gather", lambda: ctx.nn(g, r, 1.0, A, dptr(Tg), g, W, xcols=idx)),
    ("nn_merge_resid", lambda: ctx.nn(r, r, -1.0, S.cols(0, r), dptr(T), r, W, beta=1.0, Z=U2)),
    ("nn_merge_rotate", lambda: ctx.nn(2 * r, r, 1.0, S, dptr(T), 2 * r, W)),
    ("gram_eigh", lambda: ctx.gram_eigh(dptr(G), g, g, r, sig, dptr(Tl), g)),
    ("merge_core", lambda: ctx.merge_core(dptr(sig1), r, dptr(M), r, dptr(R), r, dptr(sig1), r, r, r,
                                          dptr(Tm), 2 * r, r, dptr(sn))),
    ("cholqr_factor", lambda: ctx.cholqr_factor(dptr(Gq), r, r, m, dptr(Rinv), r, dptr(Rk), r)),
    ("nn_merge_resid+gram", lambda: ctx.nn_gram(r, r, -1.0, S.cols(0, r), dptr(T), r, W, dptr(Gq2), r,
                                                beta=1.0, Z=U2)),
    ("wedin_k20", lambda: ctx.wedin(A, Uw, Vw, sw, 20, w2)),
]
import sys as _s
only = _s.argv[1:]  # optional subset of op names
for name, fn in ops:
    if only and name not in only:
        continue
    fn(); fn()
torch.cuda.synchronize()
print("ok")
