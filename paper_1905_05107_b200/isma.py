"""Iterative sampling and merging on the GPU -- drop-in for the reference's
``podsketch.isma`` (isma.py:1-303).

Same names, arguments, defaults, validation and error classes as the
reference: ``IsmaConfig`` (isma.py:59-119), ``IterationTrace``
(isma.py:122-141), ``isma_run`` (isma.py:225-303), ``get_update``
(isma.py:144-178) and ``convergence_cosines`` (isma.py:181-201).  All
numerics run in libpodsketch_b200.so (see engine.py); the caller's numpy
Generator supplies the uniforms, one ``rng.random(c)`` batch per round,
so sampled index sets follow the reference's stream.

Every strategy of the reference runs here: column sampling with "l2n",
"unf" and "ort", and row sampling (``rows=True``, ICRS) with "unf", "ort"
and "ls" -- one further ``rng.random(w)`` batch per round for the row draw.
Row-sharded multi-GPU runs cover the column path only (row draws are global
over all m rows).
"""

from __future__ import annotations

import dataclasses

import numpy as np

from .errors import DegenerateDistributionError, ParameterError
from .sampling import ctsvd_sample_count, ltsvd_sample_count

STRATEGIES = ("l2n", "unf", "ort", "ls")
LAST_STATS = {}  # engine statistics of the most recent isma_run (diagnostics)
LAST_DRAWS = None  # per-round (indices, counts) of the last run when engine.RECORD_DRAWS
CRITERIA = ("modes", "subspace")


@dataclasses.dataclass(frozen=True)
class IsmaConfig:
    """Parameters of an iterative run (isma.py:59-119); r defaults to 3k."""

    k: int
    r: int | None = None
    epsilon: float = 0.7
    delta: float = 0.6
    tau: float = 0.99
    strategy: str = "unf"
    rows: bool = False
    criterion: str = "modes"
    seed: int = 0
    finalize: bool = True
    c: int | None = None
    w: int | None = None

    def __post_init__(self):
        if self.k < 1:
            raise ParameterError("k must be >= 1")
        r = 3 * self.k if self.r is None else self.r
        if r < self.k:
            raise ParameterError(f"r={r} must be >= k={self.k}")
        if not self.epsilon > 0:
            raise ParameterError("epsilon must be > 0")
        if not 0 < self.delta < 1:
            raise ParameterError("delta must lie strictly between 0 and 1")
        if not 0 <= self.tau <= 1:
            raise ParameterError("tau must lie in [0, 1]")
        strategy = str(self.strategy).lower()
        if strategy not in STRATEGIES:
            raise ParameterError(f"strategy must be one of {STRATEGIES}")
        criterion = str(self.criterion).lower()
        if criterion not in CRITERIA:
            raise ParameterError(f"criterion must be one of {CRITERIA}")
        if strategy == "ls" and not self.rows:
            raise ParameterError("strategy 'ls' samples rows; set rows=True")
        if strategy == "l2n" and self.rows:
            raise ParameterError("strategy 'l2n' is column-only; rows must be False")
        for name, val in (("c", self.c), ("w", self.w)):
            if val is not None and val < 1:
                raise ParameterError(f"{name} override must be >= 1")
        object.__setattr__(self, "r", r)
        object.__setattr__(self, "strategy", strategy)
        object.__setattr__(self, "criterion", criterion)

    def column_budget(self):
        if self.c is not None:
            return int(self.c)
        return ltsvd_sample_count(self.k, self.epsilon, self.delta)

    def row_budget(self):
        if self.w is not None:
            return int(self.w)
        return ctsvd_sample_count(self.k, self.epsilon, self.delta)


@dataclasses.dataclass(frozen=True)
class IterationTrace:
    """Diagnostics of one update round (isma.py:122-141)."""

    iteration: int
    columns_sampled: int
    rows_sampled: int
    remaining: int
    cosines: np.ndarray
    wall_time: float

    def __post_init__(self):
        cos = np.asarray(self.cosines, dtype=np.float64)
        if cos.size and (cos.min() < -1.0 or cos.max() > 1.0):
            raise ParameterError("cosines must lie in [-1, 1]")
        object.__setattr__(self, "cosines", cos)


def _validate_shape(a):
    from .device import ColMat

    if isinstance(a, ColMat):
        if a.m == 0 or a.ncols == 0:
            raise ParameterError("matrix must have at least one row and column")
        return a, a.m, a.ncols
    shape = getattr(a, "shape", None)
    if shape is None:
        a = np.asarray(a, dtype=np.float64)
        shape = a.shape
    if len(shape) != 2:
        raise ParameterError(f"expected a 2-D matrix, got ndim={len(shape)}")
    if shape[0] == 0 or shape[1] == 0:
        raise ParameterError("matrix must have at least one row and column")
    return a, int(shape[0]), int(shape[1])


def isma_run(a, config, rng=None, keep=None, *, device=None, return_device=False,
             use_graphs=True, comm=None, m_total=None, residency="auto", precision="fp64"):
    """Run the full iteration (isma.py:225-303) on the GPU.

    ``a`` may be a numpy array (copied host->device), a CUDA torch tensor
    or a ``device.ColMat`` (used in place).  Returns ``(TruncatedFactor,
    list[IterationTrace])`` exactly as the reference.

    ``residency`` ("auto" | "device" | "host"): where a HOST matrix lives
    during the run.  "host" keeps it in page-locked host memory read by the
    kernels over PCIe -- the multi-pass streamed ISMA: one pass
    for the norms, each round's sampled columns copied into HBM, one pass for
    finalize (and one per round for "ort") -- for matrices larger than HBM.
    Results are bit-identical to the device-resident run.  "auto" picks
    "host" when the matrix would not leave headroom on the device.

    ``precision`` ("fp64" | "mixed"): "mixed" (BASELINE config 4) runs the
    products that read a float32-stored A -- the sampled Gram D^T D and
    finalize's A^T U -- on the tcgen05 tensor cores in 3xTF32 with fp32
    accumulation (relative error ~2e-6 per product; north_star tolerance
    sigma 1e-4, angles 1e-3); index sets are unchanged (the norms and draws
    are exact).  Ignored for float64 storage.

    Row-sharded multi-GPU (parallel.py): pass ``comm=parallel.Comm()`` and
    this rank's row block ``a`` = A[r0:r1] with r0, r1 = shard_rows(m_total,
    world, rank); every rank must use an identically seeded generator.  The
    returned factor is the full (gathered) one on every rank.
    """
    import torch

    from .device import ColMat, HostResident, get_ctx, upload_matrix
    from .parallel import Comm, shard_rows

    a, m, n = _validate_shape(a)
    comm = comm if comm is not None else Comm()
    row_offset = 0
    if comm.active:
        if m_total is None:
            raise ParameterError("row-sharded isma_run needs m_total")
        r0, r1 = shard_rows(int(m_total), comm.world, comm.rank)
        if r1 - r0 != m:
            raise ParameterError(f"rank {comm.rank} holds {m} rows, expected {r1 - r0}")
        row_offset, m = r0, int(m_total)
    k = config.k
    if k > min(m, n):
        raise ParameterError(f"k={k} exceeds min(m, n)={min(m, n)}")
    keep = k if keep is None else int(keep)
    if not 1 <= keep <= config.r:
        raise ParameterError(f"keep={keep} outside 1..r={config.r}")
    if rng is None:
        rng = np.random.default_rng(config.seed)
    ctx = get_ctx(device)
    if precision not in ("fp64", "mixed"):
        raise ParameterError("precision must be 'fp64' or 'mixed'")
    if residency not in ("auto", "device", "host"):
        raise ParameterError("residency must be 'auto', 'device' or 'host'")
    on_host = not isinstance(a, ColMat) and not (isinstance(a, torch.Tensor) and a.is_cuda)
    if on_host and residency == "auto":
        # device storage keeps float32 as float32 (to_device_colmajor)
        dt = getattr(a, "dtype", None)
        itemsize = 4 if dt in (np.float32, torch.float32) else 8
        nbytes = int(np.prod(getattr(a, "shape", (0,)))) * itemsize
        free, _ = torch.cuda.mem_get_info(ctx.device)
        residency = "host" if nbytes > 0.7 * free else "device"
    if on_host and residency == "host":
        # multi-pass streamed ISMA, also row-sharded: each rank
        # streams its own row block from its page-locked host memory
        if comm.active and config.strategy == "ort":
            raise ParameterError("strategy 'ort' with a host-resident row-sharded matrix is not "
                                 "supported (its C = U^T A must be reduced over ranks before "
                                 "the residual pass)")
        with HostResident(a) as A:
            return _run_engine(ctx, A, config, rng, k, keep, use_graphs, comm, row_offset, m,
                               return_device, precision)
    A = upload_matrix(a, ctx.device)
    return _run_engine(ctx, A, config, rng, k, keep, use_graphs, comm, row_offset, m,
                       return_device, precision)


def _run_engine(ctx, A, config, rng, k, keep, use_graphs, comm, row_offset, m, return_device,
                precision="fp64"):
    from .engine import get_engine
    from .matcore import TruncatedFactor

    eng = get_engine(ctx, A, k=k, r=config.r, c=config.column_budget(),
                     criterion=config.criterion, use_graphs=use_graphs, comm=comm,
                     row_offset=row_offset, m_total=m if comm.active else None,
                     w=config.row_budget() if config.rows else 0, precision=precision)
    traces, v = eng.run(rng, strategy=config.strategy, tau=config.tau,
                        finalize=config.finalize, keep=keep, trace_cls=IterationTrace)
    u, s, vv = eng.result(keep, v)
    eng.A = None  # the cached engine must not keep the caller's matrix alive
    factor = TruncatedFactor(u, s, vv)
    global LAST_STATS, LAST_DRAWS
    LAST_STATS = eng.stats
    LAST_DRAWS = eng.draw_log  # per-round (indices, counts) when engine.RECORD_DRAWS
    if return_device:
        return factor, traces, eng
    return factor, traces


def get_update(a, s, u_prev, dist, c, w, rows, rng, r):
    """One sampling round (isma.py:144-178) on the GPU.

    Draws ``c`` indices from ``dist`` (one ``rng.random(c)`` batch) and
    factors the distinct sampled columns D.  rows=False: through the Gram
    matrix D^T D.  rows=True (ICRS): ``w`` rows are drawn (one
    ``rng.random(w)`` batch) from D's squared row norms, or from the leverage
    scores of ``u_prev`` when it is a non-empty factor, and the eigensolve
    runs on Y^T Y of the dedup-scaled row block Y; the left vectors are lifted
    through D either way.  Returns ``(factor, remaining, g, h)``; an empty
    candidate set returns ``(None, s, 0, 0)``.
    """
    import torch

    from .device import ColMat, dptr, get_ctx, to_device_colmajor
    from .engine import MODE_ROWS, MODE_WEIGHTS
    from .matcore import TruncatedFactor

    s = np.asarray(s, dtype=np.int64)
    if s.size == 0:
        return None, s, 0, 0
    a, m, n = _validate_shape(a)
    if rows and int(w) < 1:
        raise ParameterError("sample count must be >= 1")
    ctx = get_ctx()
    A = to_device_colmajor(a, ctx.device)
    dev = ctx.device
    w_dev = torch.as_tensor(dist.weights, dtype=torch.float64, device=dev)
    npos = dist.size
    u = np.asarray(rng.random(int(c)), dtype=np.float64)
    uni = torch.as_tensor(u, device=dev)
    g_cap = min(int(c), npos)
    pos = torch.empty(g_cap, dtype=torch.int32, device=dev)
    cnt = torch.empty(g_cap, dtype=torch.int64, device=dev)
    ctx.draw(MODE_WEIGHTS, w_dev, None, npos, uni, int(c), pos, cnt)
    g, _, status = ctx.read_info(3)
    picked = dist.indices[pos[:g].cpu().numpy().astype(np.int64)]
    idx = torch.as_tensor(picked.astype(np.int32), device=dev)
    remaining = np.setdiff1d(s, picked, assume_unique=True)
    G = torch.empty(g * g, dtype=torch.float64, device=dev)
    h = 0
    if not rows:
        ctx.tn(g, g, 1.0, A, A, dptr(G), g, xcols=idx, ycols=idx)
    else:
        q = torch.empty(m, dtype=torch.float64, device=dev)
        if u_prev is None or u_prev.is_empty:
            ctx.rownorms2(A, g, q, cols=idx)                    # row_norm_distribution(d)
        else:
            up = np.asarray(u_prev.u, dtype=np.float64)
            if up.ndim != 2 or up.shape[0] != m:
                raise ParameterError("u_prev must have the same row count as a")
            U = to_device_colmajor(np.asfortranarray(up), dev)
            ctx.rownorms2(U, up.shape[1], q, div=float(up.shape[1]))  # leverage_distribution
        if not bool((q.sum() > 0).item()):
            raise DegenerateDistributionError("all row weights are zero")
        wu = torch.as_tensor(np.asarray(rng.random(int(w)), dtype=np.float64), device=dev)
        h_cap = min(int(w), m)
        ridx = torch.empty(h_cap, dtype=torch.int32, device=dev)
        rcnt = torch.empty(h_cap, dtype=torch.int64, device=dev)
        rp = torch.empty(h_cap, dtype=torch.float64, device=dev)
        ctx.draw(MODE_ROWS, q, None, m, wu, int(w), ridx, rcnt, p_out=rp)
        h, _, rstatus = ctx.read_info(3)
        if rstatus == 2:
            raise DegenerateDistributionError("all row weights are zero")
        Y = ColMat.zeros(h, g, dev)
        ctx.gather_scale_rows(A, idx, g, ridx, rcnt, rp, int(w), h, ctx.info[0:1], Y)
        ctx.tn(g, g, 1.0, Y, Y, dptr(G), g)                     # gram_spectrum(y)
    sig = torch.empty(g, dtype=torch.float64, device=dev)
    T = torch.empty(g * int(r), dtype=torch.float64, device=dev)
    info = torch.zeros(4, dtype=torch.int64, device=dev)
    ctx.gram_eigh_any(G, g, int(r), sig, T, info)
    keep = int(info[1].item())
    if keep == 0:
        return TruncatedFactor.empty(m), remaining, g, h
    U = ColMat.zeros(m, keep, dev)
    ctx.nn(g, keep, 1.0, A, dptr(T), g, U, xcols=idx)
    ctx.fix_signs(U, keep)
    return TruncatedFactor(U.to_numpy(), sig[:keep].cpu().numpy()), remaining, g, h


def convergence_cosines(prev, next_, k, criterion):
    """Cosines between successive top-k approximations (isma.py:181-201),
    computed on the GPU."""
    import torch

    from .device import ColMat, dptr, get_ctx, to_device_colmajor

    if criterion not in CRITERIA:
        raise ParameterError(f"criterion must be one of {CRITERIA}")
    kk = min(k, prev.nmodes, next_.nmodes)
    xi = np.zeros(k)
    if kk == 0:
        return xi
    ctx = get_ctx()
    P = to_device_colmajor(np.asfortranarray(prev.u[:, :kk]), ctx.device)
    Q = to_device_colmajor(np.asfortranarray(next_.u[:, :kk]), ctx.device)
    if criterion == "modes":
        out = torch.zeros(k, dtype=torch.float64, device=ctx.device)
        ctx.coldots(P, Q, k, kk, True, out)
        return out.cpu().numpy()
    C = torch.empty(kk * kk, dtype=torch.float64, device=ctx.device)
    ctx.tn(kk, kk, 1.0, P, Q, dptr(C), kk)
    sv = torch.empty(kk, dtype=torch.float64, device=ctx.device)
    ctx.svd_small(dptr(C), kk, kk, kk, None, 1, sv, None, 1)
    xi[:kk] = sv.cpu().numpy()
    return np.clip(xi, 0.0, 1.0)
