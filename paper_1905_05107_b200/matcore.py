"""Core types with the reference's semantics (matcore.py:1-254).

``TruncatedFactor`` is the host-side result type (numpy arrays, frozen,
validated exactly as matcore.py:63-145).  ``fix_signs`` runs on the GPU
(pod_fix_signs).  ``as_dense`` is the reference's input normaliser; the
ISMA driver itself validates on the device (non-finite flag of the norm
pass) instead of calling it.
"""

from __future__ import annotations

import dataclasses

import numpy as np

from .errors import ParameterError

#: matcore.py:20 -- relative threshold below which a singular value is zero.
ZERO_SIGMA_RTOL = 1e-14
#: matcore.py:26 -- relative eigenvalue dust threshold on Gram paths.
GRAM_EIG_RTOL = 1e-12


def as_dense(a, *, copy=False):
    """Read-only column-major float64 view/copy; 2-D, non-empty, finite
    (matcore.py:29-60)."""
    arr = np.array(a, dtype=np.float64, order="F", copy=copy or None)
    if arr.ndim != 2:
        raise ParameterError(f"expected a 2-D matrix, got ndim={arr.ndim}")
    if arr.size == 0:
        raise ParameterError("matrix must have at least one row and column")
    if not np.isfinite(arr).all():
        raise ParameterError("matrix contains non-finite entries")
    if arr is a:
        arr = arr.view()
    arr.flags.writeable = False
    return arr


@dataclasses.dataclass(frozen=True)
class TruncatedFactor:
    """(U, sigma, optional V) with the invariants of matcore.py:63-145."""

    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray | None = None

    def __post_init__(self):
        u = np.asarray(self.u, dtype=np.float64)
        sigma = np.asarray(self.sigma, dtype=np.float64)
        if u.ndim != 2 or sigma.ndim != 1:
            raise ParameterError("u must be 2-D and sigma 1-D")
        if u.shape[1] != sigma.shape[0]:
            raise ParameterError(
                f"u has {u.shape[1]} columns but sigma has {sigma.shape[0]} entries")
        if u.shape[1] > u.shape[0]:
            raise ParameterError("factor cannot carry more modes than rows")
        if sigma.size:
            if sigma.min() < 0:
                raise ParameterError("sigma entries must be nonnegative")
            slack = ZERO_SIGMA_RTOL * max(sigma[0], 1.0)
            if np.any(np.diff(sigma) > slack):
                raise ParameterError("sigma must be nonincreasing")
        if self.v is not None:
            v = np.asarray(self.v, dtype=np.float64)
            if v.ndim != 2 or v.shape[1] != sigma.shape[0]:
                raise ParameterError("v must be 2-D with one column per sigma")
            if v.shape[1] > v.shape[0]:
                raise ParameterError("factor cannot carry more modes than v rows")
            object.__setattr__(self, "v", v)
        object.__setattr__(self, "u", u)
        object.__setattr__(self, "sigma", sigma)

    @property
    def nmodes(self):
        return int(self.sigma.shape[0])

    @property
    def is_empty(self):
        return self.nmodes == 0

    @classmethod
    def empty(cls, m, with_v=None):
        v = np.zeros((with_v, 0)) if with_v is not None else None
        return cls(np.zeros((m, 0)), np.zeros(0), v)

    def truncate(self, r):
        if r < 0:
            raise ParameterError("truncation rank must be nonnegative")
        if r >= self.nmodes:
            return self
        return TruncatedFactor(self.u[:, :r].copy(), self.sigma[:r].copy(),
                               None if self.v is None else self.v[:, :r].copy())

    def validate(self, tol=1e-8):
        for name, mat in (("u", self.u), ("v", self.v)):
            if mat is None or mat.shape[1] == 0:
                continue
            err = np.abs(mat.T @ mat - np.eye(mat.shape[1])).max()
            if err > tol:
                raise ParameterError(
                    f"{name} columns deviate from orthonormal by {err:.3e} (> {tol:.1e})")
        return self


def fix_signs(u, v=None):
    """Largest-|entry| of each u column made positive, v flipped alongside
    (matcore.py:148-165), computed by pod_fix_signs on the GPU."""
    from .device import get_ctx, to_device_colmajor

    u = np.asarray(u, dtype=np.float64)
    if u.ndim != 2:
        raise ParameterError("u must be 2-D")
    if u.shape[1] == 0 or u.shape[0] == 0:
        return np.array(u, order="F"), (None if v is None else np.array(v, order="F"))
    ctx = get_ctx()
    du = to_device_colmajor(np.array(u, order="F"), ctx.device)
    dv = None
    if v is not None:
        v = np.asarray(v, dtype=np.float64)
        dv = to_device_colmajor(np.array(v, order="F"), ctx.device)
    ctx.fix_signs(du, u.shape[1], dv, 0 if dv is None else dv.m)
    return du.to_numpy(), (None if dv is None else dv.to_numpy())
