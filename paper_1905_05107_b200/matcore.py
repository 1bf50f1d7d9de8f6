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


def mean_center_rows(a):
    """Subtract each row's mean (matcore.py:168-175); a host preprocessing
    step of the CLI's ``convert --center``, outside the GPU path."""
    a = as_dense(a)
    return as_dense(a - a.mean(axis=1, keepdims=True))


# ---------------------------------------------------------------------------
# Exact dense factorizations on the device (matcore.py:187-254).  The data
# matrix may be numpy or a torch tensor (host or CUDA, fp64 or fp32 storage);
# results are host numpy arrays as in the reference.

#: widest block the one-sided Jacobi solvers (pod_svd_small) take
SMALL_MAX_COLS = 1024
#: tallest block pod_svd_small takes directly; taller inputs are QR'd first
SMALL_MAX_ROWS = 4096


def _device_input(a):
    import torch

    from .device import get_ctx, to_device_colmajor

    ctx = get_ctx()
    if isinstance(a, torch.Tensor):
        if a.ndim != 2 or a.numel() == 0:
            raise ParameterError("matrix must be 2-D and non-empty")
        return ctx, to_device_colmajor(a, ctx.device)
    arr = np.asarray(a)
    if arr.dtype != np.float32:
        arr = as_dense(arr)
    elif arr.ndim != 2 or arr.size == 0 or not np.isfinite(arr).all():
        arr = as_dense(arr)  # raises the reference's error
    return ctx, to_device_colmajor(arr, ctx.device)


def _transpose(A):
    import torch

    from .device import ColMat

    t = A.t[A.col0:A.col0 + A.ncols, :A.m].to(torch.float64)
    return ColMat(t.T.contiguous(), A.ncols, A.m)


def _f64(A):
    import torch

    from .device import ColMat

    if A.code == 0 and A.col0 == 0:
        return A
    return ColMat(A.t[A.col0:A.col0 + A.ncols].to(torch.float64).contiguous(), A.m, A.ncols)


NN_MAX_Q = 192  # output columns per pod_gemm_nn launch


def _nn(ctx, p, q, X, T, ldt, Y, tag):
    """Y (m x q) = X (m x p) T (p x q, column-major torch, ld ldt), in
    launches of <= 192 output columns; Y must not alias X."""
    from .device import dptr

    for a in range(0, q, NN_MAX_Q):
        b = min(q, a + NN_MAX_Q)
        ctx.nn(p, b - a, 1.0, X, dptr(T, a * ldt), ldt, Y.cols(a, b), tag=tag)


def _qr_device(ctx, A, l):
    """A (m x l device) = Q R: CholeskyQR2, then up to two more passes while
    pod_cholqr_factor reports an orthogonality defect (the merge QR's pass
    rule), ping-ponging between two m x l blocks.  Returns Q (ColMat) and R
    (torch, l x l column-major).  Exactly-zero directions give zero Q
    columns."""
    import torch

    from .device import ColMat, dptr

    dev = ctx.device
    f = dict(dtype=torch.float64, device=dev)
    G, Rinv, Rk = (torch.empty(l * l, **f) for _ in range(3))
    R = torch.zeros(l * l, **f)
    Rtmp = torch.empty(l * l, **f)
    gates = torch.zeros(5, dtype=torch.int32, device=dev)
    bufs = (ColMat.zeros(A.m, l, dev), ColMat.zeros(A.m, l, dev))
    src = A
    for p in range(4):
        if p >= 2 and not int(gates[p].item()):
            break
        dst = bufs[p % 2]
        ctx.tn(l, l, 1.0, src, src, dptr(G), l, tag="tn_qr_gram")
        ctx.cholqr_factor(dptr(G), l, l, src.m, dptr(Rinv), l, dptr(Rk), l,
                          gate_out=gates[p + 1:p + 2], first_pass=1 if p == 0 else 0)
        _nn(ctx, l, l, src, Rinv, l, dst, "nn_qr_apply")
        if p == 0:
            ctx.small_copy(l, l, dptr(Rk), l, dptr(R), l)
        else:
            ctx.small_gemm(l, l, l, 1.0, dptr(Rk), l, 0, dptr(R), l, 0.0, dptr(Rtmp), l)
            ctx.small_copy(l, l, dptr(Rtmp), l, dptr(R), l)
        src = dst
    return src, R


def _svd_device(ctx, A):
    """Thin SVD of a tall device block (m >= n, n <= 1024): U (ColMat),
    sigma, V (torch n x n column-major), descending."""
    import torch

    from .device import ColMat, dptr

    dev = ctx.device
    m, n = A.m, A.ncols
    sig = torch.empty(n, dtype=torch.float64, device=dev)
    V = torch.empty(n * n, dtype=torch.float64, device=dev)
    if m <= SMALL_MAX_ROWS:
        A = _f64(A)
        U = ColMat.zeros(m, n, dev)
        ctx.svd_small(A.ptr, A.ld, m, n, U.ptr, U.ld, sig, dptr(V), n)
        return U, sig, V
    Q, R = _qr_device(ctx, A, n)
    UR = torch.empty(n * n, dtype=torch.float64, device=dev)
    ctx.svd_small(dptr(R), n, n, n, dptr(UR), n, sig, dptr(V), n)
    U = ColMat.zeros(m, n, dev)
    _nn(ctx, n, n, Q, UR, n, U, "nn_svd_lift")
    return U, sig, V


def _polish_orthonormal(ctx, U, l):
    """One-sided Jacobi's left vectors w_j / sigma_j are orthogonal to ~2e-14
    (measured on the reference's acceptance-2 inputs; LAPACK: 2e-15), which
    the arccos-based principal angles (quality.py:49-57) turn into 1e-5 deg.
    A CholeskyQR of the l nonzero columns (R = I + O(1e-14), positive
    diagonal) restores working-precision orthonormality and moves each column
    by O(1e-14)."""
    if l < 1:
        return
    Q, _ = _qr_device(ctx, U.cols(0, l), l)
    U.t[U.col0:U.col0 + l, :U.m].copy_(Q.t[Q.col0:Q.col0 + l, :Q.m])


def _square(t, n):
    from .device import ColMat

    return ColMat(t.view(n, n), n, n)


def dense_svd(a):
    """Full thin SVD as a TruncatedFactor with V (matcore.py:187-197), signs
    by the largest-entry-positive rule.  One-sided Jacobi on the device
    (pod_svd_small) directly for up to 4096 rows, after a CholeskyQR of the
    tall block otherwise; min(m, n) <= 1024.  Exactly rank-deficient inputs
    give zero left vectors for their zero singular values (the reference's
    LAPACK call completes them to an orthonormal set)."""
    ctx, A = _device_input(a)
    m, n = A.m, A.ncols
    if min(m, n) > SMALL_MAX_COLS:
        raise ParameterError(f"dense_svd on the B200 path supports min(m, n) <= "
                             f"{SMALL_MAX_COLS} (got {min(m, n)})")
    flip = m < n
    if flip:
        A = _transpose(A)
    U, sig, V = _svd_device(ctx, A)
    l = A.ncols
    _polish_orthonormal(ctx, U, int((sig > 0).sum().item()))
    Vm = _square(V, l)
    ctx.fix_signs(Vm if flip else U, l, U if flip else Vm, U.m if flip else l)
    u, v = U.to_numpy(), Vm.to_numpy()
    if flip:
        u, v = v, u
    return TruncatedFactor(u, sig.cpu().numpy(), v)


def thin_qr(a):
    """Economy QR ``a = q @ r`` with rows >= cols (matcore.py:200-210) by
    CholeskyQR passes on the device; ``r`` has a nonnegative diagonal (the
    reference's LAPACK R may differ by column signs of q / row signs of r)."""
    ctx, A = _device_input(a)
    if A.m < A.ncols:
        raise ParameterError("thin_qr requires rows >= cols")
    if A.ncols > SMALL_MAX_COLS:
        raise ParameterError(f"thin_qr on the B200 path supports <= {SMALL_MAX_COLS} columns")
    Q, R = _qr_device(ctx, A, A.ncols)
    return Q.to_numpy(), np.asfortranarray(R.view(A.ncols, A.ncols).T.cpu().numpy())


def pod_via_gram(a, k):
    """Top-k POD modes through the Gram matrix (matcore.py:213-241): G = A^T A
    by the symmetric TN kernel; for n up to pod_gram_eigh_max_g the update
    path's eigensolver (pivoted Cholesky + one-sided Jacobi, grid-wide beyond
    one cluster), beyond it cuSOLVER's symmetric solver through torch; dust
    <= 1e-12 lambda_1 dropped, u = A v / sigma by the NN kernel, signs fixed
    on the device."""
    import torch

    from . import _lib
    from .device import ColMat, dptr

    ctx, A = _device_input(a)
    m, n = A.m, A.ncols
    if not 1 <= k <= min(m, n):
        raise ParameterError(f"k={k} outside 1..min(m, n)={min(m, n)}")
    dev = ctx.device
    G = torch.empty(n * n, dtype=torch.float64, device=dev)
    ctx.tn(n, n, 1.0, A, A, dptr(G), n, tag="tn_gram")
    if n <= int(_lib.load().pod_gram_eigh_max_g()):
        sig = torch.empty(n, dtype=torch.float64, device=dev)
        T = torch.empty(n * k, dtype=torch.float64, device=dev)
        info = torch.zeros(4, dtype=torch.int64, device=dev)
        ctx.gram_eigh(dptr(G), n, n, k, sig, dptr(T), n, info=info)
        sig_h = sig[:k].cpu().numpy()
        keep = int(np.count_nonzero(sig_h > 0.0))  # dust already zeroed
        T = T.view(k, n)[:keep]
        V = T * sig[:keep, None]  # rows: eigenvectors
    else:
        w, vec = torch.linalg.eigh(G.view(n, n))  # symmetric: layout-agnostic
        lam = w.flip(0)[:k].clamp(min=0.0)
        lam_h = lam.cpu().numpy()
        keep = int(np.count_nonzero(lam_h > GRAM_EIG_RTOL * max(lam_h[0], np.finfo(float).tiny)))
        sig_h = np.sqrt(lam_h)
        V = vec.flip(1)[:, :keep].T.contiguous()  # (keep, n): row j = eigenvector j
        T = V / torch.as_tensor(sig_h[:keep], device=dev)[:, None]
        del w, vec
    if keep == 0:
        return TruncatedFactor(np.zeros((m, 0), order="F"), np.zeros(0),
                               np.zeros((n, 0), order="F"))
    Vk = ColMat(V.contiguous(), n, keep)
    U = ColMat.zeros(m, keep, dev)
    _nn(ctx, n, keep, A, T.contiguous().view(-1), n, U, "nn_gram_lift")
    ctx.fix_signs(U, keep, Vk, n)
    return TruncatedFactor(U.to_numpy(), sig_h[:keep].copy(), Vk.to_numpy())


def orthonormalize(u):
    """(q, s): q = Q U_R spans u with orthonormal columns, s the singular
    values of R (matcore.py:244-254); QR, SVD of R, lift and signs all on the
    device."""
    import torch

    from .device import ColMat, dptr

    ctx, U0 = _device_input(u)
    l = U0.ncols
    if U0.m < l:
        raise ParameterError("thin_qr requires rows >= cols")
    if l > SMALL_MAX_COLS:
        raise ParameterError(f"orthonormalize on the B200 path supports <= {SMALL_MAX_COLS} "
                             "columns")
    dev = ctx.device
    Q0, R = _qr_device(ctx, U0, l)
    UR = torch.empty(l * l, dtype=torch.float64, device=dev)
    s = torch.empty(l, dtype=torch.float64, device=dev)
    ctx.svd_small(dptr(R), l, l, l, dptr(UR), l, s, None, 1)
    Q = ColMat.zeros(U0.m, l, dev)
    _nn(ctx, l, l, Q0, UR, l, Q, "nn_orthonormalize")
    ctx.fix_signs(Q, l)
    return Q.to_numpy(), s.cpu().numpy()
