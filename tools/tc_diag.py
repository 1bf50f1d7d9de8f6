import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1905_05107_b200.device import ColMat, dptr, get_ctx
ctx = get_ctx(); dev = ctx.device

def colmat(a):
    return ColMat(torch.as_tensor(np.ascontiguousarray(a.T), device=dev), a.shape[0], a.shape[1])

def tf32(a):
    return (a.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)

rng = np.random.default_rng(0)
for K in (32, 256, 1024, 8192, 32768, 262144):
    P, Q = 128, 64
    x = rng.standard_normal((K, P)).astype(np.float32)
    y = rng.standard_normal((K, Q)).astype(np.float32)
    xh, yh = tf32(x), tf32(y)
    xl, yl = tf32(x - xh), tf32(y - yh)
    ref_exact = x.astype(np.float64).T @ y.astype(np.float64)
    ref_3x = (xh.astype(np.float64).T @ yh.astype(np.float64) + xl.astype(np.float64).T @ yh.astype(np.float64)
              + xh.astype(np.float64).T @ yl.astype(np.float64))
    C = torch.zeros(P * Q, dtype=torch.float64, device=dev)
    ctx.tn_tf32x3(P, Q, 1.0, colmat(x), colmat(y), dptr(C), P)
    got = C.view(Q, P).cpu().numpy().T
    # hi-only variant: pass lo = zeros
    z = torch.zeros(K * P, dtype=torch.float32, device=dev); zq = torch.zeros(K * Q, dtype=torch.float32, device=dev)
    C2 = torch.zeros(P * Q, dtype=torch.float64, device=dev)
    ctx.tn_tf32x3(P, Q, 1.0, colmat(xh), colmat(yh), dptr(C2), P, Xlo=z, Ylo=zq)
    got2 = C2.view(Q, P).cpu().numpy().T
    ref_hh = xh.astype(np.float64).T @ yh.astype(np.float64)
    sc = np.abs(ref_exact).max()
    print(f"K={K}: 3x vs exact {np.abs(got-ref_exact).max()/sc:.2e}, 3x vs emulated-3x {np.abs(got-ref_3x).max()/sc:.2e}, "
          f"hi*hi vs exact-hh {np.abs(got2-ref_hh).max()/sc:.2e}, emulated-3x vs exact {np.abs(ref_3x-ref_exact).max()/sc:.2e}")

# timing at config-4 shapes: finalize A^T U (K = 1M, P = 8192, Q = 192) and
# the gathered Gram (P = Q = 256), vs the fp64 DMMA TN kernel
K, n, r, g = 1 << 20, 8192, 192, 256
a = torch.randn((n, K), dtype=torch.float32, device=dev)
A = ColMat(a, K, n)
u = torch.randn((r, K), dtype=torch.float64, device=dev)
U = ColMat(u, K, r)
hi = torch.empty(K * r, dtype=torch.float32, device=dev); lo = torch.empty_like(hi)
C = torch.empty(n * r, dtype=torch.float64, device=dev)
idx = torch.as_tensor(np.sort(rng.choice(n, g, replace=False)).astype(np.int32), device=dev)
G = torch.empty(g * g, dtype=torch.float64, device=dev)
def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
t_tc = timeit(lambda: (ctx.split_tf32(U, r, hi, lo), ctx.tn_tf32x3(n, r, 1.0, A, ColMat(hi.view(r, K), K, r), dptr(C), n, Ylo=lo)))
t_f64 = timeit(lambda: ctx.tn(n, r, 1.0, A, U, dptr(C), n))
tg_tc = timeit(lambda: ctx.tn_tf32x3(g, g, 1.0, A, A, dptr(G), g, xcols=idx, ycols=idx))
tg_f64 = timeit(lambda: ctx.tn(g, g, 1.0, A, A, dptr(G), g, xcols=idx, ycols=idx))
fl = 2.0 * K * n * r
print(f"finalize A^T U 1M x 8192 x 192: tcgen05 3xTF32 {t_tc:.2f} ms ({fl/t_tc/1e9:.1f} TF/s alg, "
      f"{K*n*4/t_tc/1e6:.0f} GB/s of A), fp64 DMMA {t_f64:.2f} ms; gathered Gram 256: tcgen05 "
      f"{tg_tc:.3f} ms, DMMA {tg_f64:.3f} ms")
