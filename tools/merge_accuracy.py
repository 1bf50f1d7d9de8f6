"""Acceptance criterion 2 (test_acceptance.py:95-124) decomposed: block_merge
vs LAPACK, dense_svd vs LAPACK, angle helpers vs numpy."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_1905_05107_b200 as pod
from podtest_util import make_low_rank


def ang_deg(u1, u2):
    q1 = np.linalg.qr(u1)[0]; q2 = np.linalg.qr(u2)[0]
    s = np.linalg.svd(q2 - q1 @ (q1.T @ q2), compute_uv=False)
    return np.degrees(np.arcsin(min(1.0, s.max())))


rng = np.random.default_rng(2718)
w = {"merge_vs_lapack": 0, "dense_vs_lapack": 0, "test_metric": 0, "merge_vs_dense": 0}
for trial in range(50):
    m = int(rng.integers(30, 121)); r1 = int(rng.integers(1, 6)); r2 = int(rng.integers(1, 6))
    n1 = r1 + int(rng.integers(0, 8)); n2 = r2 + int(rng.integers(0, 8))
    x = make_low_rank(m, n1, r1, rng); y = 1.7 * make_low_rank(m, n2, r2, rng)
    r = r1 + r2
    ex = lambda a, k: pod.dense_svd(a).truncate(k)
    merged = pod.block_merge(ex(x, r1), ex(y, r2), r)
    t = merged.nmodes
    U, S, _ = np.linalg.svd(np.hstack([x, y]), full_matrices=False)
    d = pod.dense_svd(np.hstack([x, y]))
    w["merge_vs_lapack"] = max(w["merge_vs_lapack"], ang_deg(U[:, :t], merged.u))
    w["dense_vs_lapack"] = max(w["dense_vs_lapack"], ang_deg(U[:, :t], d.u[:, :t]))
    w["merge_vs_dense"] = max(w["merge_vs_dense"], ang_deg(d.u[:, :t], merged.u))
    w["test_metric"] = max(w["test_metric"], float(np.max(pod.principal_angles(d.truncate(t), merged, t))))
print(w)
rng = np.random.default_rng(2718)
worst = {}
def orth(u):
    return np.abs(u.T @ u - np.eye(u.shape[1])).max()
for trial in range(50):
    m = int(rng.integers(30, 121)); r1 = int(rng.integers(1, 6)); r2 = int(rng.integers(1, 6))
    n1 = r1 + int(rng.integers(0, 8)); n2 = r2 + int(rng.integers(0, 8))
    x = make_low_rank(m, n1, r1, rng); y = 1.7 * make_low_rank(m, n2, r2, rng)
    r = r1 + r2
    fx, fy = pod.dense_svd(x).truncate(r1), pod.dense_svd(y).truncate(r2)
    merged = pod.block_merge(fx, fy, r)
    d = pod.dense_svd(np.hstack([x, y]))
    t = merged.nmodes
    for key, val in (("dense_x", orth(fx.u)), ("dense_hstack", orth(d.u[:, :t])), ("merged", orth(merged.u)),
                     ("lapack_hstack", orth(np.linalg.svd(np.hstack([x, y]), full_matrices=False)[0][:, :t]))):
        worst[key] = max(worst.get(key, 0), val)
print("orthogonality defects", worst)
