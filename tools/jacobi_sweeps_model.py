"""CPU model of the device's parallel round-robin one-sided Jacobi: count
sweeps on real merge matrices E and Gram matrices from a config-2-like run,
with and without QR-column-pivoting preconditioning (Jacobi on R^T)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.linalg as sla
from oracle import isma_oracle as orc
from paper_1905_05107_b200 import workloads

def rr_pairs(n):
    N = n + (n & 1); M1 = N - 1
    steps = []
    for st in range(M1):
        pr = [(0, 1 + st)]
        for p in range(1, N // 2):
            a = (st + p) % M1 + 1; b = (st - p + M1) % M1 + 1
            pr.append((min(a, b), max(a, b)))
        steps.append([(a, b) for a, b in pr if b < n])
    return steps

def jacobi_sweeps(W, tol=None, max_sweeps=60):
    W = W.copy(); n = W.shape[1]; tol = tol or 2.22e-16 * max(W.shape[0], 16)
    steps = rr_pairs(n)
    for sw in range(1, max_sweeps + 1):
        rot = False
        for pr in steps:
            a = np.array([p[0] for p in pr]); b = np.array([p[1] for p in pr])
            al = np.einsum('ij,ij->j', W[:, a], W[:, a]); be = np.einsum('ij,ij->j', W[:, b], W[:, b])
            ga = np.einsum('ij,ij->j', W[:, a], W[:, b])
            do = (ga * ga > tol * tol * al * be) & (al > 0) & (be > 0)
            if not do.any(): continue
            rot = True
            a, b, al, be, ga = a[do], b[do], al[do], be[do], ga[do]
            z = (be - al) / (2 * ga); t = np.sign(z) / (np.abs(z) + np.hypot(1, z)); t[z == 0] = 1.0
            c = 1 / np.sqrt(1 + t * t); s = c * t
            x, y = W[:, a].copy(), W[:, b].copy()
            W[:, a] = c * x - s * y; W[:, b] = s * x + c * y
        if not rot: return sw
    return max_sweeps

# capture E and D^T D matrices from an oracle run on a config-2 proxy
Es, Gs = [], []
orig_merge, orig_gram = orc.merge, orc.gram_eig
def rec_merge(u1, s1, u2, s2, r):
    l1, l2 = min(r, s1.size), min(r, s2.size)
    if l1 and l2:
        mm = u1[:, :l1].T @ u2[:, :l2]
        q, rr = np.linalg.qr(u2[:, :l2] - u1[:, :l1] @ mm)
        e = np.zeros((l1 + l2, l1 + l2)); e[:l1, :l1] = np.diag(s1[:l1]); e[:l1, l1:] = mm * s2[:l2]; e[l1:, l1:] = rr * s2[:l2]
        Es.append(e)
    return orig_merge(u1, s1, u2, s2, r)
def rec_gram(d):
    Gs.append(d.T @ d); return orig_gram(d)
orc.merge, orc.gram_eig = rec_merge, rec_gram
a = workloads.config2(seed=0, side=128, n=2000)
orc.run(a, 20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7, max_rounds=6)
for E in Es[:4]:
    s0 = jacobi_sweeps(E)
    q, r, p = sla.qr(E, pivoting=True)
    s1 = jacobi_sweeps(r.T)
    print(f"E {E.shape}: plain {s0} sweeps, QRCP R^T {s1} sweeps")
for G in Gs[1:4]:
    L = np.linalg.cholesky(G + 0 * np.eye(G.shape[0])) if np.all(np.linalg.eigvalsh(G) > 0) else None
    s0 = jacobi_sweeps(G)
    q, r, p = sla.qr(np.linalg.cholesky(G[np.ix_(np.arange(G.shape[0]), np.arange(G.shape[0]))]).T, pivoting=True) if L is not None else (None, None, None)
    rt = np.linalg.cholesky(G).T  # R with G = R^T R
    s1 = jacobi_sweeps(rt.T)
    q2, r2, p2 = sla.qr(rt, pivoting=True)
    s2 = jacobi_sweeps(r2.T)
    print(f"G {G.shape}: plain {s0}, chol R^T {s1}, chol+QRCP {s2}")

def jacobi_profile(W, tol, max_sweeps=60):
    W = W.copy(); n = W.shape[1]
    steps = rr_pairs(n); out = []
    for sw in range(1, max_sweeps + 1):
        nrot = 0; offmax = 0.0
        for pr in steps:
            a = np.array([p[0] for p in pr]); b = np.array([p[1] for p in pr])
            al = np.einsum('ij,ij->j', W[:, a], W[:, a]); be = np.einsum('ij,ij->j', W[:, b], W[:, b])
            ga = np.einsum('ij,ij->j', W[:, a], W[:, b])
            rel = np.abs(ga) / np.sqrt(np.maximum(al * be, 1e-300)); offmax = max(offmax, rel.max())
            do = (ga * ga > tol * tol * al * be) & (al > 0) & (be > 0)
            nrot += int(do.sum())
            if not do.any(): continue
            a, b, al, be, ga = a[do], b[do], al[do], be[do], ga[do]
            z = (be - al) / (2 * ga); t = np.sign(z) / (np.abs(z) + np.hypot(1, z)); t[z == 0] = 1.0
            c = 1 / np.sqrt(1 + t * t); s = c * t
            x, y = W[:, a].copy(), W[:, b].copy()
            W[:, a] = c * x - s * y; W[:, b] = s * x + c * y
        out.append((nrot, offmax))
        if nrot == 0: break
    return out, W

E = Es[2]
for tol in (2.7e-14, 1e-12, 1e-10):
    prof, W = jacobi_profile(E, tol)
    print(f"tol {tol}: sweeps {len(prof)}", [(a, f"{b:.1e}") for a, b in prof])
    s = np.sort(np.linalg.norm(W, axis=0))[::-1]
    print("   sigma err vs LAPACK:", np.max(np.abs(s[:60] - np.linalg.svd(E, compute_uv=False)[:60]) / np.linalg.svd(E, compute_uv=False)[:60]))
print("E sigma:", np.array2string(np.linalg.svd(E, compute_uv=False)[::10], precision=3))
