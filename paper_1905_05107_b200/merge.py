"""BLOCK MERGE on the GPU -- drop-in for ``podsketch.merge`` (merge.py:1-154).

``block_merge(f1, f2, r)`` keeps the reference's contract (merge.py:37-91):
both inputs truncated to r, empty factor = identity, ParameterError on a
row-space mismatch, result keeps min(r, #sigma_E > 1e-14 sigma_E0) modes,
no right vectors, canonical signs.  Numerics (projection, CholeskyQR with
the 1e-8 leak test and second projection, the small E-SVD, the rotation)
run in libpodsketch_b200.so through ``engine.MergeWorkspace``.
"""

from __future__ import annotations

import math
import warnings

from .errors import ParameterError
from .matcore import TruncatedFactor

SVD_FLOP_BETA = 6  # merge.py:29
_REORTH_TOL = 1e-8  # merge.py:34


def block_merge(f1, f2, r):
    from .device import get_ctx
    from .engine import MergeWorkspace

    if r < 1:
        raise ParameterError("merge rank r must be >= 1")
    f1 = f1.truncate(r)
    f2 = f2.truncate(r)
    if f1.is_empty:
        return f2
    if f2.is_empty:
        return f1
    m1, m2 = f1.u.shape[0], f2.u.shape[0]
    if m1 != m2:
        raise ParameterError(f"factors live in different row spaces ({m1} vs {m2})")
    ctx = get_ctx()
    ws = MergeWorkspace(ctx, m1, r)
    ws.load_factor(0, f1.u, f1.sigma)
    ws.load_factor("upd", f2.u, f2.sigma)
    nxt, keep = ws.merge_now(0)
    ws.cur, ws.l = nxt, keep
    if keep:
        ctx.fix_signs(ws.S[nxt].cols(0, keep), keep)
    u = ws.S[nxt].to_numpy(keep)
    s = ws.sig[nxt][:keep].cpu().numpy().copy()
    return TruncatedFactor(u, s)


def merge_chain(factors, r):
    """Left fold of block_merge (merge.py:94-102)."""
    factors = list(factors)
    if not factors:
        raise ParameterError("merge_chain needs at least one factor")
    acc = factors[0].truncate(r)
    for f in factors[1:]:
        acc = block_merge(acc, f, r)
    return acc


class MergeBoundInput:
    """Chain bound inputs (merge.py:105-117)."""

    def __init__(self, partitions, sigma_r_plus_1):
        if partitions < 1:
            raise ParameterError("partitions must be >= 1")
        if sigma_r_plus_1 < 0:
            raise ParameterError("sigma_{r+1} must be >= 0")
        self.partitions = partitions
        self.sigma_r_plus_1 = sigma_r_plus_1


def mat_error_bound(bound_input):
    """(2^(P+1) - 3) sigma_{r+1} (merge.py:120-141)."""
    p = bound_input.partitions
    coeff = (1 << (p + 1)) - 3
    if p > 60:
        warnings.warn(f"bound coefficient 2^{p + 1}-3 exceeds exact float range; "
                      "result is saturated", stacklevel=2)
    try:
        cf = float(coeff)
    except OverflowError:
        cf = math.inf
    return cf * bound_input.sigma_r_plus_1


def mat_flops_estimate(m, n, p, beta=SVD_FLOP_BETA):
    """14 m n^2 / P + 32 beta n^3 / P^2 (merge.py:144-154)."""
    if m < 1 or n < 1 or p < 1:
        raise ParameterError("m, n, p must all be >= 1")
    m, n, p = float(m), float(n), float(p)
    return 14.0 * m * n * n / p + 32.0 * beta * n ** 3 / (p * p)
