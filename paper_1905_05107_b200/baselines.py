"""Single-round sampled SVD baselines on the GPU -- drop-in for
``podsketch.baselines`` (baselines.py:1-142).

``gram_spectrum`` forms the sample's Gram matrix with the TN GEMM and
eigen-decomposes it with the block-Jacobi SVD (for the PSD Gram, singular
values are the eigenvalues and J the eigenvectors, a complete orthonormal
basis); ``lift_left_vectors`` is the NN GEMM plus the sign convention;
``ltsvd`` / ``ctsvd`` compose them with the device draw and sample scaling,
with the reference's warnings and energy filter.
"""

from __future__ import annotations

import warnings

import numpy as np

from . import _lib
from .errors import ParameterError
from .matcore import GRAM_EIG_RTOL, ZERO_SIGMA_RTOL, TruncatedFactor, _nn
from .sampling import (
    _scale_columns_dev,
    _scale_rows_dev,
    row_norm_distribution,
    sample_with_replacement,
)


def _gram_eigh_dev(D, r):
    """The update path's Gram-and-lift setup (a6): G = D^T D by the symmetric
    TN kernel, pod_gram_eigh -> all sigmas (dust-zeroed, descending, host)
    and T = V[:, :keep] / sigma[:keep] (g x r device, zero beyond keep)."""
    import torch

    from .device import dptr, get_ctx

    ctx = get_ctx()
    dev = ctx.device
    g = D.ncols
    G = torch.empty(g * g, dtype=torch.float64, device=dev)
    ctx.tn(g, g, 1.0, D, D, dptr(G), g, tag="tn_gram")
    sig = torch.empty(g, dtype=torch.float64, device=dev)
    T = torch.empty(g * r, dtype=torch.float64, device=dev)
    info = torch.zeros(4, dtype=torch.int64, device=dev)
    ctx.gram_eigh_any(G, g, r, sig, T, info)
    return sig.cpu().numpy(), T


def gram_spectrum(mat):
    """(sigma, V) of ``mat`` through its Gram matrix (baselines.py:35-48):
    G by the symmetric TN kernel, the full eigenvector basis by one-sided
    Jacobi on G (for a PSD matrix its singular pairs), descending, clipped
    at zero, eigenvalue dust <= 1e-12 lambda_1 zeroed, sigma = sqrt(lambda);
    V is g x g.  (ltsvd / ctsvd use the update path's pod_gram_eigh, which
    returns only the kept vectors, pre-divided by sigma.)"""
    from .sampling import _dev

    if np.ndim(mat) != 2:
        raise ParameterError("matrix must be 2-D")
    g = np.shape(mat)[1]
    if g == 0:
        return np.zeros(0), np.zeros((0, 0), order="F")
    import torch

    from .device import dptr, get_ctx

    ctx, D = _dev(mat)
    dev = ctx.device
    G = torch.empty(g * g, dtype=torch.float64, device=dev)
    ctx.tn(g, g, 1.0, D, D, dptr(G), g, tag="tn_gram")
    lam = torch.empty(g, dtype=torch.float64, device=dev)
    V = torch.empty(g * g, dtype=torch.float64, device=dev)
    ctx.svd_small(dptr(G), g, g, g, None, 1, lam, dptr(V), g)
    lam = np.clip(lam.cpu().numpy(), 0.0, None)
    lam[lam <= GRAM_EIG_RTOL * max(lam[0], np.finfo(float).tiny)] = 0.0
    return np.sqrt(lam), np.asfortranarray(V.view(g, g).cpu().numpy().T)


def _lift_T(S, sigma, T, keep):
    """U = S T[:, :keep] (T = V / sigma from _gram_eigh_dev) and the sign
    rule, on the device -- the update path's lift (a7)."""
    from .device import ColMat, get_ctx

    m = S.m
    if keep == 0:
        return TruncatedFactor.empty(m)
    ctx = get_ctx()
    U = ColMat.zeros(m, keep, ctx.device)
    _nn(ctx, S.ncols, keep, S, T, S.ncols, U, "nn_lift")
    ctx.fix_signs(U, keep)
    return TruncatedFactor(U.to_numpy(), sigma[:keep].copy())


def _rank(sigma):
    if sigma.size == 0 or not sigma[0] > 0.0:
        return 0
    return int(np.count_nonzero(sigma > ZERO_SIGMA_RTOL * sigma[0]))


def lift_left_vectors(source, sigma, v, keep):
    """U = source V[:, :keep] / sigma[:keep] with keep = min(keep, rank),
    rank = #sigma > 1e-14 sigma_1, then the sign convention
    (baselines.py:51-65); NN GEMM and signs on the device."""
    import torch

    from .device import get_ctx
    from .sampling import _dev

    sigma = np.asarray(sigma, dtype=np.float64)
    m = np.shape(source)[0]
    rank = _rank(sigma)
    if rank == 0:
        return TruncatedFactor.empty(m)
    keep = min(int(keep), rank)
    _, S = _dev(source)
    v = np.asarray(v, dtype=np.float64)
    T = np.asfortranarray(v[:, :keep] / sigma[:keep])
    Td = torch.as_tensor(T.T.reshape(-1), device=get_ctx().device)
    return _lift_T(S, sigma, Td, keep)


def ltsvd(a, dist, k, c, rng, dedup=True):
    """Sampled truncated SVD from c column draws (baselines.py:68-109); the
    sample stays on the device between the gather, Gram and lift."""
    if k < 1:
        raise ParameterError("k must be >= 1")
    if c < k:
        warnings.warn(f"sampling c={c} columns for k={k} modes; expect a rank shortfall",
                      stacklevel=2)
    draw = sample_with_replacement(dist, c, rng)
    D = _scale_columns_dev(a, draw, dist, c, dedup)
    sigma, T = _gram_eigh_dev(D, k)
    factor = _lift_T(D, sigma, T, min(k, _rank(sigma)))
    if factor.nmodes < k:
        warnings.warn(f"sample has rank {factor.nmodes} < k={k}; returning fewer modes",
                      stacklevel=2)
    return factor


def ctsvd(a, dist, k, c, w, epsilon, rng, dedup=True):
    """Sampled truncated SVD from c column draws then w row draws of the
    sampled block, with the energy filter gamma = epsilon / (100 k)
    (baselines.py:112-142); all blocks stay on the device."""
    if k < 1:
        raise ParameterError("k must be >= 1")
    if w < 1:
        raise ParameterError("w must be >= 1")
    if not epsilon > 0:
        raise ParameterError("epsilon must be > 0")
    draw = sample_with_replacement(dist, c, rng)
    Dc = _scale_columns_dev(a, draw, dist, c, dedup)
    row_dist = row_norm_distribution(Dc)
    row_draw = sample_with_replacement(row_dist, w, rng)
    Dw = _scale_rows_dev(Dc, row_draw, row_dist, w, dedup)
    sigma, T = _gram_eigh_dev(Dw, k)
    gamma = epsilon / (100.0 * k)
    frob2 = float(np.sum(sigma * sigma))
    passing = int(np.count_nonzero(sigma * sigma >= gamma * frob2))
    factor = _lift_T(Dc, sigma, T, min(k, passing, _rank(sigma)))
    if factor.nmodes < k:
        warnings.warn(f"energy filter kept {factor.nmodes} of k={k} modes", stacklevel=2)
    return factor
