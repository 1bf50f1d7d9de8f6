"""Shared parity metrics (tolerances follow BASELINE.json north_star, fp64):
index sets bit-exact; sigma within 1e-10 relative; principal angles (sine
formula, tests/oracles.py:100-111 semantics) below 1e-8 rad."""

import numpy as np

SIGMA_RTOL = 1e-10
ANGLE_TOL_RAD = 1e-8


def principal_angles_sin(u1, u2):
    q1 = np.linalg.qr(np.asarray(u1, dtype=np.float64))[0]
    q2 = np.linalg.qr(np.asarray(u2, dtype=np.float64))[0]
    s = np.linalg.svd(q2 - q1 @ (q1.T @ q2), compute_uv=False)
    return np.arcsin(np.sort(np.clip(s, 0.0, 1.0)))


def sigma_relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if b.size else 0.0
