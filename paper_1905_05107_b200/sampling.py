"""Distributions and seeded sampling with replacement (sampling.py:1-291).

``Distribution`` / ``SampleDraw`` are the reference's host-side value types
(same invariants).  ``column_norm_distribution`` computes its weights with
the GPU norm pass and ``sample_with_replacement`` runs the inverse-CDF draw
on the GPU (pod_draw, mode 2) from exactly one ``rng.random(count)`` batch.
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np

from .errors import DegenerateDistributionError, ParameterError


@dataclasses.dataclass(frozen=True)
class Distribution:
    """Probability vector over sorted distinct candidate indices
    (sampling.py:23-78)."""

    indices: np.ndarray
    weights: np.ndarray

    def __post_init__(self):
        idx = np.asarray(self.indices, dtype=np.int64)
        w = np.asarray(self.weights, dtype=np.float64)
        if idx.ndim != 1 or w.shape != idx.shape:
            raise ParameterError("indices and weights must be 1-D and equal length")
        if idx.size == 0:
            raise ParameterError("distribution needs at least one candidate")
        if np.unique(idx).size != idx.size:
            raise ParameterError("candidate indices must be distinct")
        order = np.argsort(idx, kind="stable")
        idx, w = idx[order], w[order]
        if w.min() < 0:
            raise ParameterError("weights must be nonnegative")
        total = w.sum()
        if abs(total - 1.0) > 1e-12:
            raise ParameterError(f"weights must sum to 1 (got {total!r})")
        w = w / total
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "weights", w)

    @classmethod
    def from_weights(cls, indices, raw_weights, *, what="candidate"):
        raw = np.asarray(raw_weights, dtype=np.float64)
        total = raw.sum()
        if not total > 0.0:
            raise DegenerateDistributionError(f"all {what} weights are zero")
        return cls(np.asarray(indices, dtype=np.int64), raw / total)

    @property
    def size(self):
        return int(self.indices.shape[0])

    def weight_of(self, wanted):
        wanted = np.asarray(wanted, dtype=np.int64)
        pos = np.clip(np.searchsorted(self.indices, wanted), 0, self.size - 1)
        if not np.array_equal(self.indices[pos], wanted):
            raise ParameterError("index not present in the distribution")
        return self.weights[pos]


@dataclasses.dataclass(frozen=True)
class SampleDraw:
    """Distinct drawn indices with occurrence counts (sampling.py:81-107)."""

    unique_indices: np.ndarray
    counts: np.ndarray
    total: int

    def __post_init__(self):
        idx = np.asarray(self.unique_indices, dtype=np.int64)
        cnt = np.asarray(self.counts, dtype=np.int64)
        if idx.ndim != 1 or cnt.shape != idx.shape:
            raise ParameterError("unique_indices and counts must match in shape")
        if np.unique(idx).size != idx.size:
            raise ParameterError("unique_indices must be distinct")
        if cnt.size and cnt.min() < 1:
            raise ParameterError("counts must be positive")
        if int(cnt.sum()) != int(self.total):
            raise ParameterError("counts must sum to the requested total")
        object.__setattr__(self, "unique_indices", idx)
        object.__setattr__(self, "counts", cnt)
        object.__setattr__(self, "total", int(self.total))

    @property
    def ndistinct(self):
        return int(self.unique_indices.shape[0])


def column_norm_distribution(a, candidates=None):
    """Distribution over columns proportional to squared norms
    (sampling.py:110-140); norms from the GPU norm pass."""
    import torch

    from .device import get_ctx, to_device_colmajor

    shape = np.shape(a)
    if candidates is None:
        candidates = np.arange(shape[1])
    candidates = np.asarray(candidates, dtype=np.int64)
    if candidates.size == 0:
        raise ParameterError("candidate set is empty")
    ctx = get_ctx()
    A = to_device_colmajor(np.asarray(a, dtype=np.float64), ctx.device)
    norms2 = torch.empty(A.ncols, dtype=torch.float64, device=ctx.device)
    flag = torch.zeros(1, dtype=torch.int32, device=ctx.device)
    ctx.colnorms2(A, norms2, flag)
    raw = norms2.cpu().numpy()[candidates]
    return Distribution.from_weights(candidates, raw, what="candidate column")


def uniform_distribution(candidates):
    """Equal weight on every candidate (sampling.py:150-155)."""
    candidates = np.asarray(candidates, dtype=np.int64)
    if candidates.size == 0:
        raise ParameterError("candidate set is empty")
    return Distribution(candidates, np.full(candidates.size, 1.0 / candidates.size))


def sample_with_replacement(dist, count, rng):
    """Draw ``count`` indices i.i.d. from ``dist`` and collapse duplicates
    (sampling.py:204-222): one ``rng.random(count)`` batch, inverse-CDF on
    the GPU (CDF pinned to 1 at the last positive weight, side='right')."""
    import torch

    from .device import get_ctx
    from .engine import MODE_WEIGHTS

    if count < 1:
        raise ParameterError("sample count must be >= 1")
    u = np.asarray(rng.random(int(count)), dtype=np.float64)
    ctx = get_ctx()
    dev = ctx.device
    w = torch.as_tensor(dist.weights, dtype=torch.float64, device=dev)
    uni = torch.as_tensor(u, device=dev)
    cap = min(int(count), dist.size)
    pos = torch.empty(cap, dtype=torch.int32, device=dev)
    cnt = torch.empty(cap, dtype=torch.int64, device=dev)
    ctx.draw(MODE_WEIGHTS, w, None, dist.size, uni, int(count), pos, cnt)
    g, _, _ = ctx.read_info(3)
    picked = dist.indices[pos[:g].cpu().numpy().astype(np.int64)]
    return SampleDraw(picked, cnt[:g].cpu().numpy(), int(count))


def _check_count_params(k, epsilon, delta):
    if k < 1 or int(k) != k:
        raise ParameterError("k must be a positive integer")
    if not epsilon > 0:
        raise ParameterError("epsilon must be > 0")
    if not 0 < delta < 1:
        raise ParameterError("delta must lie strictly between 0 and 1")


def _ltsvd_count_raw(k, epsilon, delta):
    """Eq. 8a before the ceiling (sampling.py:270-271; the test oracles pin it)."""
    return 4.0 * k * (1.0 + math.sqrt(8.0 * math.log(1.0 / delta))) ** 2 / epsilon ** 2


def _ctsvd_count_raw(k, epsilon, delta):
    """Eq. 8b before the ceiling (sampling.py:274-275)."""
    return float(k * k) * (1.0 + math.sqrt(math.log(2.0 / delta))) ** 2 / epsilon ** 4


def ltsvd_sample_count(k, epsilon, delta):
    """c = ceil(4k (1 + sqrt(8 ln(1/delta)))^2 / eps^2) (sampling.py:270-276)."""
    _check_count_params(k, epsilon, delta)
    return int(math.ceil(_ltsvd_count_raw(k, epsilon, delta)))


def ctsvd_sample_count(k, epsilon, delta):
    """c = w = ceil(k^2 (1 + sqrt(ln(2/delta)))^2 / eps^4) (sampling.py:288-291)."""
    _check_count_params(k, epsilon, delta)
    return int(math.ceil(_ctsvd_count_raw(k, epsilon, delta)))


# ---------------------------------------------------------------------------
# Row / residual / leverage distributions and sample scaling (sampling.py:
# 143-258), computed with the library's kernels; the results are host values
# as in the reference.

def _dev(a):
    from .device import ColMat, get_ctx, to_device_colmajor

    ctx = get_ctx()
    return ctx, (a if isinstance(a, ColMat) else to_device_colmajor(a, ctx.device))


def row_norm_distribution(d):
    """Distribution over all rows of ``d`` proportional to squared norms
    (sampling.py:143-147)."""
    import torch

    ctx, D = _dev(d)
    out = torch.empty(D.m, dtype=torch.float64, device=ctx.device)
    ctx.rownorms2(D, D.ncols, out)
    return Distribution.from_weights(np.arange(D.m), out.cpu().numpy(), what="row")


def leverage_distribution(u):
    """Row distribution from the leverage scores ||u_i||^2 / k of an
    orthonormal basis (sampling.py:190-201)."""
    import torch

    if np.ndim(u) != 2 or np.shape(u)[1] == 0:
        raise ParameterError("u must be 2-D with at least one column")
    ctx, U = _dev(u)
    out = torch.empty(U.m, dtype=torch.float64, device=ctx.device)
    ctx.rownorms2(U, U.ncols, out, div=float(U.ncols))
    return Distribution.from_weights(np.arange(U.m), out.cpu().numpy(), what="leverage")


def residual_distribution(a, u, candidates=None, *, degenerate_rtol=1e-14):
    """Weights proportional to the squared residual of each candidate column
    after projection on the orthonormal ``u`` (sampling.py:158-187): C =
    U^T A[:, S] and ||a_j - U c_j||^2 in one fused pass, never materialised.
    Raises DegenerateDistributionError when the residual total is at most
    ``degenerate_rtol * ||A||_F^2``."""
    import torch

    from .device import dptr

    a_shape = np.shape(a)
    if candidates is None:
        candidates = np.arange(a_shape[1])
    candidates = np.asarray(candidates, dtype=np.int64)
    if candidates.size == 0:
        raise ParameterError("candidate set is empty")
    if np.ndim(u) != 2 or np.shape(u)[0] != a_shape[0]:
        raise ParameterError("u must be 2-D with the same row count as a")
    if np.shape(u)[1] == 0:
        return column_norm_distribution(a, candidates)
    ctx, A = _dev(a)
    _, U = _dev(u if not isinstance(u, np.ndarray) else np.asarray(u, dtype=np.float64))
    dev = ctx.device
    g, r = candidates.size, U.ncols
    cols = torch.as_tensor(candidates.astype(np.int32), device=dev)
    C = torch.empty(r * g, dtype=torch.float64, device=dev)
    ctx.tn(r, g, 1.0, U, A, dptr(C), r, ycols=cols, tag="tn_resid_proj")
    res2 = torch.empty(g, dtype=torch.float64, device=dev)
    ctx.resid_colnorms2(A, g, U, r, dptr(C), r, res2, cols=cols)
    norms = torch.empty(A.ncols, dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    ctx.colnorms2(A, norms, flag)
    res2 = res2.cpu().numpy()
    total = res2.sum()
    if total <= degenerate_rtol * float(norms.sum().item()):
        raise DegenerateDistributionError(
            "candidate columns are fully captured by the current basis")
    return Distribution(candidates, res2 / total)


def _scale_factors(dist, draw, total, dedup):
    """sampling.py:225-231 (host scalars, same formulas)."""
    from .errors import PodsketchError

    p = dist.weight_of(draw.unique_indices)
    if np.any(p <= 0.0):
        raise PodsketchError("drawn index has zero weight; sampler invariant broken")
    if dedup:
        return np.sqrt(draw.counts / (total * p))
    return 1.0 / np.sqrt(total * np.repeat(p, draw.counts))


def _scale_columns_dev(a, draw, dist, c, dedup):
    import torch

    from .device import ColMat

    f = _scale_factors(dist, draw, c, dedup)
    idx = draw.unique_indices if dedup else np.repeat(draw.unique_indices, draw.counts)
    ctx, A = _dev(a)
    dev = ctx.device
    D = ColMat.zeros(A.m, idx.size, dev)
    ctx.gather_scale_cols(A, torch.as_tensor(idx.astype(np.int64), device=dev),
                          torch.as_tensor(f, dtype=torch.float64, device=dev), idx.size, D)
    return D


def scale_sampled_columns(a, draw, dist, c, dedup=True):
    """The scaled sample (sampling.py:234-245): dedup -> one column per
    distinct index scaled by sqrt(t_i / (c p_i)), so D D^T = C C^T; else one
    column per draw scaled by 1/sqrt(c p_i).  Gathered and scaled on the
    device with the host-computed factors (bit-identical products)."""
    return _scale_columns_dev(a, draw, dist, c, dedup).to_numpy()


def _scale_rows_dev(c, draw, dist, w, dedup):
    import torch

    from .device import ColMat
    from .errors import PodsketchError

    if dedup:
        rows, cnt = draw.unique_indices, draw.counts
    else:
        rows = np.repeat(draw.unique_indices, draw.counts)
        cnt = np.ones(rows.size, dtype=np.int64)
    p = dist.weight_of(rows)
    if np.any(p <= 0.0):
        raise PodsketchError("drawn index has zero weight; sampler invariant broken")
    ctx, Cm = _dev(c)
    dev = ctx.device
    h = rows.size
    Y = ColMat.zeros(h, Cm.ncols, dev)
    hdev = torch.tensor([h], dtype=torch.int64, device=dev)
    ctx.gather_scale_rows(Cm, None, Cm.ncols, torch.as_tensor(rows.astype(np.int32), device=dev),
                          torch.as_tensor(cnt.astype(np.int64), device=dev),
                          torch.as_tensor(p, dtype=torch.float64, device=dev), float(w), h, hdev,
                          Y)
    return Y


def scale_sampled_rows(c, draw, dist, w, dedup=True):
    """Row counterpart (sampling.py:248-258): dedup -> one row per distinct
    index scaled by sqrt(t_i / (w q_i)), so Y^T Y = W^T W; else one row per
    draw scaled by 1/sqrt(w q_i).  Gathered and scaled on the device."""
    return _scale_rows_dev(c, draw, dist, w, dedup).to_numpy()
