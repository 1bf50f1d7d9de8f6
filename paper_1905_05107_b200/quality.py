"""Accuracy metrics on the GPU -- drop-in for ``podsketch.quality``
(quality.py:1-118).

``wedin_measure`` computes ||R||_F and ||S||_F of the residuals
R = A V_k - U_k S_k and S = A^T U_k - V_k S_k in ONE pass over A
(``pod_wedin_residuals``: every A tile feeds both FP64 DMMA products from
shared memory, R is reduced in the epilogue without being written, S across a
thread-block cluster); k > 64 falls back to two GPU passes (NN for A V_k,
split-K TN for A^T U_k).  ``principal_angles`` / ``mode_angles`` use the TN
GEMM + Jacobi singular values and the column dot kernel.
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np

from .errors import ParameterError
from .matcore import ZERO_SIGMA_RTOL

#: largest k of the fused single-pass residual kernel (pod_wedin_residuals)
WEDIN_FUSED_MAX_K = 64

#: quality.py:15-19
DEGENERATE_OMEGA_ADVICE = (
    "sigma_k and sigma_{k+1} are (numerically) equal, so the error measure "
    "is unbounded; increase k by one or two and rerun"
)


def _top_k_bases(exact, approx, k):
    """quality.py:22-35"""
    if k < 1:
        raise ParameterError("k must be >= 1")
    if exact.u.shape[0] != approx.u.shape[0]:
        raise ParameterError(
            f"factors have different row counts ({exact.u.shape[0]} vs {approx.u.shape[0]})")
    if exact.nmodes < k or approx.nmodes < k:
        raise ParameterError(
            f"both factors need at least k={k} modes (have {exact.nmodes} and {approx.nmodes})")
    return exact.u[:, :k], approx.u[:, :k]


def _upload(x):
    from .device import get_ctx, to_device_colmajor

    ctx = get_ctx()
    return ctx, to_device_colmajor(np.asfortranarray(np.asarray(x, dtype=np.float64)), ctx.device)


def mode_angles(exact, approx, k):
    """Per-mode angles in degrees, arccos |u_i . u~_i| (quality.py:38-46)."""
    import torch

    ue, ua = _top_k_bases(exact, approx, k)
    ctx, E = _upload(ue)
    _, Aa = _upload(ua)
    out = torch.zeros(k, dtype=torch.float64, device=ctx.device)
    ctx.coldots(E, Aa, k, k, True, out)
    cos = out.cpu().numpy()
    return np.degrees(np.arccos(np.clip(cos, 0.0, 1.0)))


def principal_angles(exact, approx, k):
    """Principal angles in degrees from the singular values of
    approx_k^T exact_k (quality.py:49-57)."""
    import torch

    from .device import dptr

    ue, ua = _top_k_bases(exact, approx, k)
    ctx, E = _upload(ue)
    _, Aa = _upload(ua)
    C = torch.empty(k * k, dtype=torch.float64, device=ctx.device)
    ctx.tn(k, k, 1.0, Aa, E, dptr(C), k, tag="tn_angles")
    sv = torch.empty(k, dtype=torch.float64, device=ctx.device)
    ctx.svd_small(dptr(C), k, k, k, None, 1, sv, None, 1)
    cos = sv.cpu().numpy()
    return np.degrees(np.arccos(np.clip(cos, 0.0, 1.0)))


@dataclasses.dataclass(frozen=True)
class WedinReport:
    """quality.py:60-79"""

    r_norm: float
    s_norm: float
    omega_hat: float
    measure: float
    ceiling: float
    degenerate: bool

    @property
    def advisory(self):
        return DEGENERATE_OMEGA_ADVICE if self.degenerate else None


def _frobenius(ctx, M):
    """||M||_F with the column-norm reduction (fixed order)."""
    import torch

    nrm = torch.empty(M.ncols, dtype=torch.float64, device=ctx.device)
    flag = torch.zeros(1, dtype=torch.int32, device=ctx.device)
    ctx.colnorms2(M, nrm, flag)
    return math.sqrt(float(np.sum(nrm.cpu().numpy())))


def wedin_measure(a, factor, k):
    """Wedin-style error measure (quality.py:82-118) on the GPU."""
    import torch

    from .device import ColMat, dptr, get_ctx, to_device_colmajor

    if k < 1:
        raise ParameterError("k must be >= 1")
    if factor.v is None:
        raise ParameterError("factor must carry right singular vectors")
    if factor.nmodes < k + 1:
        raise ParameterError(f"need k+1={k + 1} singular values, factor has {factor.nmodes}")
    shape = getattr(a, "shape", None) if not isinstance(a, ColMat) else (a.m, a.ncols)
    if shape is None:
        a = np.asarray(a)
        shape = a.shape
    m, n = shape
    if m != factor.u.shape[0] or n != factor.v.shape[0]:
        raise ParameterError("factor dimensions do not match the matrix")
    ctx = get_ctx()
    dev = ctx.device
    A = to_device_colmajor(a, dev)
    Uk = to_device_colmajor(np.asfortranarray(factor.u[:, :k]), dev)
    Vk = to_device_colmajor(np.asfortranarray(factor.v[:, :k]), dev)
    sk = np.asarray(factor.sigma[:k], dtype=np.float64)
    if k <= WEDIN_FUSED_MAX_K:
        # quality.py:104-107 fused: one pass over A, Frobenius sums in the epilogues
        sig_d = torch.as_tensor(sk, device=dev)
        out2 = torch.zeros(2, dtype=torch.float64, device=dev)
        ctx.wedin(A, Uk, Vk, sig_d, k, out2)
        r2, s2 = out2.cpu().numpy()
        r_norm, s_norm = math.sqrt(r2), math.sqrt(s2)
    else:
        r_norm, s_norm = _wedin_two_pass(ctx, A, Uk, Vk, sk, m, n, k)
    sig = factor.sigma
    omega_hat = float(min(abs(sig[k - 1] - sig[k]), sig[k - 1]))
    degenerate = bool(omega_hat <= ZERO_SIGMA_RTOL * max(sig[0], 1e-300))
    measure = math.inf if degenerate else math.hypot(r_norm, s_norm) / omega_hat
    return WedinReport(r_norm=r_norm, s_norm=s_norm, omega_hat=omega_hat, measure=measure,
                       ceiling=math.sqrt(2.0 * k), degenerate=degenerate)


def _wedin_two_pass(ctx, A, Uk, Vk, sk, m, n, k):
    """k > 64: R and S materialised by the NN / TN GEMMs (two passes over A)."""
    import torch

    from .device import ColMat, dptr

    dev = ctx.device
    D = torch.as_tensor(np.diag(sk).T.copy().reshape(-1), device=dev)  # k x k, column-major
    # R = A V_k - U_k S_k   (quality.py:104)
    Rm = ColMat.zeros(m, k, dev)
    ctx.nn(n, k, 1.0, A, Vk.ptr, Vk.ld, Rm, tag="nn_wedin_AV")
    ctx.small_gemm(m, k, k, -1.0, Uk.ptr, Uk.ld, 0, dptr(D), k, 1.0, Rm.ptr, Rm.ld)
    # S = A^T U_k - V_k S_k (quality.py:105)
    Sm = ColMat.zeros(n, k, dev)
    ctx.tn(n, k, 1.0, A, Uk, Sm.ptr, Sm.ld, tag="tn_wedin_AtU")
    ctx.small_gemm(n, k, k, -1.0, Vk.ptr, Vk.ld, 0, dptr(D), k, 1.0, Sm.ptr, Sm.ld)
    return _frobenius(ctx, Rm), _frobenius(ctx, Sm)
