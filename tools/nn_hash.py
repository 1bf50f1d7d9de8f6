"""Config-3 and config-2 NN shapes on seeded operands: prints a hash of each
output (compare two builds / switches for bitwise equality)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200.device import ColMat, dptr, get_ctx
ctx = get_ctx(); dev = ctx.device
torch.manual_seed(0)
for (m, r, g, n) in ((1_000_003, 150, 200, 2000), (262144, 60, 100, 2000), (77777, 20, 37, 300)):
    S = ColMat(torch.randn((2 * r, m), dtype=torch.float64, device=dev), m)
    U2 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
    W = ColMat(torch.zeros((r, m), dtype=torch.float64, device=dev), m)
    W2 = ColMat(torch.randn((r, m), dtype=torch.float64, device=dev), m)
    A = ColMat(torch.randn((n, m), dtype=torch.float64, device=dev), m)
    idx = torch.as_tensor(np.sort(np.random.default_rng(0).choice(n, g, replace=False)).astype(np.int32), device=dev)
    T = torch.randn(4 * r * r, dtype=torch.float64, device=dev)
    Tg = torch.randn(g * r, dtype=torch.float64, device=dev)
    C = torch.zeros(max(n * r, g * g), dtype=torch.float64, device=dev)
    ops = {"resid": lambda: ctx.nn(r, r, -1.0, S.cols(0, r), dptr(T), r, W, beta=1.0, Z=U2),
           "apply": lambda: ctx.nn(r, r, 1.0, W2, dptr(T), r, W),
           "inplace": lambda: ctx.nn(r, r, 1.0, W2, dptr(T), r, W2),
           "rotate": lambda: ctx.nn(2 * r, r, 1.0, S, dptr(T), 2 * r, W),
           "lift": lambda: ctx.nn(g, r, 1.0, A, dptr(Tg), g, W, xcols=idx),
           "tgram": lambda: ctx.tn(r, r, 1.0, W2, W2, dptr(C), r),
           "tproj": lambda: ctx.tn(r, r, 1.0, S.cols(0, r), U2, dptr(C), r),
           "tgath": lambda: ctx.tn(g, g, 1.0, A, A, dptr(C), g, xcols=idx, ycols=idx),
           "tfin": lambda: ctx.tn(n, r, 1.0, A, U2, dptr(C), n)}
    for name, fn in ops.items():
        fn(); torch.cuda.synchronize()
        out = W2.t if name == "inplace" else (C if name[0] == "t" else W.t)
        h = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12]
        print(m, r, name, h)
