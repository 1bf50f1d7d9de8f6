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


def ltsvd_sample_count(k, epsilon, delta):
    """c = ceil(4k (1 + sqrt(8 ln(1/delta)))^2 / eps^2) (sampling.py:270-276)."""
    _check_count_params(k, epsilon, delta)
    return int(math.ceil(4.0 * k * (1.0 + math.sqrt(8.0 * math.log(1.0 / delta))) ** 2
                         / epsilon ** 2))


def ctsvd_sample_count(k, epsilon, delta):
    """c = w = ceil(k^2 (1 + sqrt(ln(2/delta)))^2 / eps^4) (sampling.py:288-291)."""
    _check_count_params(k, epsilon, delta)
    return int(math.ceil(float(k * k) * (1.0 + math.sqrt(math.log(2.0 / delta))) ** 2
                         / epsilon ** 4))
