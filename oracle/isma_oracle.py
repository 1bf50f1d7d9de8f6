"""CPU oracle for the ISMA column-sampling path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy/scipy, the arithmetic of the reference
package ``podsketch`` 0.1.0 (``/root/reference/pkg/src/podsketch``) for the
hot path named in BASELINE.json: the column-norm pass, the inverse-CDF draw,
Gram/eigh + lift, BLOCK MERGE, convergence cosines, finalize, the Wedin
quality check and the one-pass incremental driver.  Every function cites the
reference lines it follows.  The restatement performs the same numpy/LAPACK
operations in the same order as the reference, so on the same machine it is
bit-identical to the reference (pinned by ``tests/test_oracle_pins.py``
against ``tests/golden/*.npz`` produced by ``tests/golden/make_golden.py``,
which imports the reference itself).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg / ``--impl reference`` arm may import this module.  The product package
``paper_1905_05107_b200`` never imports it; it runs on the CUDA library only.

Third-party arithmetic the reference relies on (not vendored in
/root/reference): numpy 2.3.5 (einsum, cumsum, searchsorted, unique, PCG64),
scipy 1.18.1 -> OpenBLAS 0.3.30 LAPACK (dgeqrf/dorgqr via scipy.linalg.qr,
dgesdd/dgesvd via scipy.linalg.svd, dsyevr via scipy.linalg.eigh).
"""

from __future__ import annotations

import math
import time

import numpy as np
import scipy.linalg as sla

# matcore.py:20, matcore.py:26, merge.py:34
SIGMA_ZERO_RTOL = 1e-14
GRAM_DUST_RTOL = 1e-12
LEAK_TOL = 1e-8


class OracleParamError(ValueError):
    """Raised where the reference raises ParameterError."""


class OracleDegenerate(ValueError):
    """Raised where the reference raises DegenerateDistributionError."""


# --------------------------------------------------------------------------
# L1 primitives
# --------------------------------------------------------------------------

def dense_f64(a):
    """matcore.py:29-60 -- F-order float64 copy/view, 2-D, non-empty, finite."""
    x = np.array(a, dtype=np.float64, order="F", copy=None)
    if x.ndim != 2:
        raise OracleParamError("expected a 2-D matrix")
    if x.size == 0:
        raise OracleParamError("empty matrix")
    if not np.isfinite(x).all():
        raise OracleParamError("matrix contains non-finite entries")
    return x


def canon_signs(u, v=None):
    """matcore.py:148-165 -- largest-|entry| of each u column made positive
    (first occurrence on ties); v columns flipped alongside."""
    u = np.array(u, order="F")
    flip = np.zeros(u.shape[1], dtype=bool)
    if u.shape[1]:
        hero = np.abs(u).argmax(axis=0)
        flip = u[hero, np.arange(u.shape[1])] < 0
        u[:, flip] *= -1.0
    if v is not None:
        v = np.array(v, order="F")
        v[:, flip] *= -1.0
    return u, v


def lapack_svd(x):
    """matcore.py:178-184 -- gesdd, falling back to gesvd."""
    try:
        return sla.svd(x, full_matrices=False, lapack_driver="gesdd")
    except sla.LinAlgError:
        return sla.svd(x, full_matrices=False, lapack_driver="gesvd")


def householder_qr(x):
    """matcore.py:200-210 (thin_qr) -- economic Householder QR."""
    if x.shape[0] < x.shape[1]:
        raise OracleParamError("thin_qr requires rows >= cols")
    return sla.qr(x, mode="economic")


# --------------------------------------------------------------------------
# L2 sampling
# --------------------------------------------------------------------------

def column_norms2(a):
    """isma.py:260 and sampling.py:136 -- einsum squared column norms."""
    return np.einsum("ij,ij->j", a, a)


def einsum_lane_state(a, state=None):
    """numpy's einsum("ij,ij->j") order (einsum_sumprod.c.src,
    sum_of_products_contig_contig_outstride0_two at the x86-64 SSE2 baseline:
    two lanes, separately rounded mul and add) over the 8-row blocks of the
    row segment `a` (rows a multiple of 8), continuing the lane state
    (2, n) of the rows above.  Vectorised over columns; the GPU's chained
    norm pass (pod_colnorms2_chain) hands the same state between row shards."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if m % 8:
        raise OracleParamError("a non-final segment needs a multiple of 8 rows")
    st = np.zeros((2, n)) if state is None else np.array(state, dtype=np.float64)
    a0, a1 = st[0], st[1]
    for i in range(0, m, 8):
        for lane_hi in (6, 4, 2, 0):
            x0, x1 = a[i + lane_hi], a[i + lane_hi + 1]
            a0 = x0 * x0 + a0
            a1 = x1 * x1 + a1
    return np.stack([a0, a1])


def einsum_lane_finish(a_tail, state):
    """The m % 8 tail of einsum's loop (lane pairs, zero filled) and acc0 + acc1."""
    a_tail = np.asarray(a_tail, dtype=np.float64)
    a0, a1 = np.array(state[0]), np.array(state[1])
    t = a_tail.shape[0]
    for i in range(0, t, 2):
        a0 = a_tail[i] * a_tail[i] + a0
        nxt = a_tail[i + 1] * a_tail[i + 1] if i + 1 < t else np.zeros_like(a0)
        a1 = nxt + a1
    return a0 + a1


def pairwise_sum(x):
    """numpy's pairwise summation of a contiguous float64 vector
    (loops_utils.h.src: blocks <= 128 with 8 accumulators, split at n/2
    rounded down to a multiple of 8), as ndarray.sum() does it."""
    x = [float(v) for v in np.asarray(x, dtype=np.float64)]

    def pw(lo, n):
        if n < 8:
            res = 0.0
            for i in range(n):
                res = res + x[lo + i]
            return res
        if n <= 128:
            r = x[lo:lo + 8]
            i = 8
            while i < n - n % 8:
                for j in range(8):
                    r[j] = r[j] + x[lo + i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res = res + x[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return pw(lo, n2) + pw(lo + n2, n - n2)

    return 0.0 + pw(0, len(x)) if x else 0.0


def normalized_weights(raw):
    """sampling.py:55-65 (from_weights) followed by sampling.py:34-53
    (__post_init__): raw/sum, then renormalised by the new sum."""
    raw = np.asarray(raw, dtype=np.float64)
    total = raw.sum()
    if not total > 0.0:
        raise OracleDegenerate("all weights are zero")
    w = raw / total
    total2 = w.sum()
    if abs(total2 - 1.0) > 1e-12:
        raise OracleParamError("weights must sum to 1")
    return w / total2


def uniform_weights(count):
    """sampling.py:150-155 then the __post_init__ renormalisation."""
    w = np.full(count, 1.0 / count)
    return w / w.sum()


def cdf_draw(candidates, weights, uniforms):
    """sampling.py:204-222 -- sequential cumsum, CDF pinned to 1.0 from the
    last positive weight, searchsorted(side='right'), unique with counts."""
    cum = np.cumsum(weights)
    last = np.nonzero(weights)[0][-1]
    cum[last:] = 1.0
    picked = np.asarray(candidates, dtype=np.int64)[
        np.searchsorted(cum, uniforms, side="right")
    ]
    uniq, counts = np.unique(picked, return_counts=True)
    return uniq.astype(np.int64), counts.astype(np.int64)


def residual_weights(a, u, candidates, degenerate_rtol=1e-14):
    """sampling.py:158-187 -- squared residuals of the candidate columns after
    projection on u, normalised (raw/total, then __post_init__ renormalises);
    None when their total is <= degenerate_rtol ||A||_F^2 (the caller then
    samples uniformly, isma.py:216-220)."""
    cols = a[:, candidates]
    if u.shape[1] == 0:
        return normalized_weights(column_norms2(cols))
    resid = cols - u @ (u.T @ cols)
    res2 = np.einsum("ij,ij->j", resid, resid)
    total = res2.sum()
    if total <= degenerate_rtol * np.einsum("ij,ij->", a, a):
        return None
    w = res2 / total
    return w / w.sum()


def row_weights(d):
    """sampling.py:143-147 -- rows of the sampled block by squared norm."""
    return normalized_weights(np.einsum("ij,ij->i", d, d))


def leverage_weights(u):
    """sampling.py:190-201 -- leverage scores ||u_i||^2 / k, normalised."""
    return normalized_weights(np.einsum("ij,ij->i", u, u) / u.shape[1])


def scaled_rows(d, uniq, counts, weights, w):
    """sampling.py:225-258 (_scale_factors + scale_sampled_rows, dedup) --
    Y = d[uniq] * sqrt(t_i / (w q_i))."""
    f = np.sqrt(counts / (w * weights[uniq]))
    return np.asfortranarray(d[uniq, :] * f[:, None])


def orthonormalize(u):
    """isma.py:244-254 -- Q R = u, U_R = SVD(R), canonical signs of Q U_R."""
    q0, rr = householder_qr(u)
    ur, _, _ = lapack_svd(rr)
    q, _ = canon_signs(q0 @ ur)
    return q


def margin_to_cdf_boundary(weights, uniforms):
    """Smallest |u - cum| over draws and CDF breakpoints (tie-risk monitor,
    SURVEY.md section 8c)."""
    cum = np.cumsum(weights)
    last = np.nonzero(weights)[0][-1]
    cum[last:] = 1.0
    pos = np.searchsorted(cum, uniforms, side="right")
    lo = np.where(pos > 0, cum[np.maximum(pos - 1, 0)], 0.0)
    hi = cum[np.minimum(pos, cum.size - 1)]
    return float(np.min(np.minimum(np.abs(uniforms - lo), np.abs(hi - uniforms))))


def ltsvd_count(k, epsilon, delta):
    """sampling.py:270-276 -- ceil(4k (1 + sqrt(8 ln(1/delta)))^2 / eps^2)."""
    return int(math.ceil(4.0 * k * (1.0 + math.sqrt(8.0 * math.log(1.0 / delta))) ** 2
                         / epsilon ** 2))


# --------------------------------------------------------------------------
# L3 kernels
# --------------------------------------------------------------------------

def gram_eig(d):
    """baselines.py:35-48 -- eigh of D^T D, descending, clipped, eigenvalue
    dust (<= 1e-12 lambda_1) zeroed, sqrt."""
    lam, vec = sla.eigh(d.T @ d)
    lam = np.clip(lam[::-1], 0.0, None)
    if lam.size:
        lam[lam <= GRAM_DUST_RTOL * max(lam[0], np.finfo(float).tiny)] = 0.0
    return np.sqrt(lam), np.asfortranarray(vec[:, ::-1])


def lift(d, sigma, v, r):
    """baselines.py:51-65 -- U = D V[:, :keep] / sigma, keep = min(r, rank),
    rank = #sigma > 1e-14 sigma_1; then canonical signs."""
    if sigma.size == 0 or sigma[0] <= 0.0:
        return np.zeros((d.shape[0], 0)), np.zeros(0)
    keep = min(r, int(np.count_nonzero(sigma > SIGMA_ZERO_RTOL * sigma[0])))
    u = d @ v[:, :keep]
    u /= sigma[:keep]
    u, _ = canon_signs(u)
    return u, sigma[:keep].copy()


def scaled_cols(a, uniq, counts, p, c, dedup=True):
    """sampling.py:225-245 (_scale_factors + scale_sampled_columns) -- dedup:
    D = a[:, uniq] * sqrt(t_i / (c p_i)); else one column per draw times
    1 / sqrt(c p_i).  ``p`` holds the weights of ``uniq``."""
    if dedup:
        f, idx = np.sqrt(counts / (c * p)), uniq
    else:
        f = 1.0 / np.sqrt(c * np.repeat(p, counts))
        idx = np.repeat(uniq, counts)
    return np.asfortranarray(a[:, idx] * f)


def scaled_rows_any(d, uniq, counts, p, w, dedup=True):
    """sampling.py:248-258 for both dedup settings (``p``: weights of uniq)."""
    if dedup:
        f, idx = np.sqrt(counts / (w * p)), uniq
    else:
        f = 1.0 / np.sqrt(w * np.repeat(p, counts))
        idx = np.repeat(uniq, counts)
    return np.asfortranarray(d[idx, :] * f[:, None])


def ltsvd(a, cand, weights, k, c, rng, dedup=True):
    """baselines.py:68-109 -- one column draw, scaled sample, Gram eigh,
    lift of min(k, rank) modes.  Returns (u, sigma, draw)."""
    uniq, cnt = cdf_draw(cand, weights, rng.random(int(c)))
    p = weights[np.searchsorted(cand, uniq)]
    d = scaled_cols(a, uniq, cnt, p, c, dedup)
    sig, v = gram_eig(d)
    u, s = lift(d, sig, v, k)
    return u, s, (uniq, cnt)


def ctsvd(a, cand, weights, k, c, w, epsilon, rng, dedup=True):
    """baselines.py:112-142 -- column draw, row draw from the sample's row
    norms, Gram eigh of the row sample, energy filter gamma = eps/(100k),
    lift through the column sample.  Returns (u, sigma)."""
    uniq, cnt = cdf_draw(cand, weights, rng.random(int(c)))
    p = weights[np.searchsorted(cand, uniq)]
    dc = scaled_cols(a, uniq, cnt, p, c, dedup)
    q = row_weights(dc)
    ridx, rcnt = cdf_draw(np.arange(dc.shape[0]), q, rng.random(int(w)))
    dw = scaled_rows_any(dc, ridx, rcnt, q[ridx], w, dedup)
    sig, v = gram_eig(dw)
    gamma = epsilon / (100.0 * k)
    frob2 = float(np.sum(sig * sig))
    passing = int(np.count_nonzero(sig * sig >= gamma * frob2))
    return lift(dc, sig, v, min(k, passing))


def dense_svd(a):
    """matcore.py:178-197 -- thin SVD (gesdd, gesvd fallback), canonical
    signs.  Returns (u, sigma, v)."""
    u, s, vt = lapack_svd(dense_f64(a))
    u, v = canon_signs(u, vt.T)
    return u, s, v


def pod_via_gram(a, k):
    """matcore.py:213-241 -- top-k eigenpairs of A^T A (dsyevr subset),
    descending, clipped, dust dropped, u = A v / sigma, canonical signs.
    Returns (u, sigma, v)."""
    a = dense_f64(a)
    n = a.shape[1]
    lam, v = sla.eigh(a.T @ a, subset_by_index=(n - k, n - 1))
    lam = np.clip(lam[::-1], 0.0, None)
    v = v[:, ::-1]
    sigma = np.sqrt(lam)
    keep = lam > GRAM_DUST_RTOL * max(lam[0], np.finfo(float).tiny)
    sigma, v = sigma[keep], v[:, keep]
    u = (a @ v) / sigma
    u, v = canon_signs(u, v)
    return u, sigma, v


def merge(u1, s1, u2, s2, r):
    """merge.py:37-91 -- BLOCK MERGE at rank r (no right vectors)."""
    u1, s1 = u1[:, :r], s1[:r]
    u2, s2 = u2[:, :r], s2[:r]
    if s1.size == 0:
        return u2.copy(), s2.copy()
    if s2.size == 0:
        return u1.copy(), s1.copy()
    if u1.shape[0] != u2.shape[0]:
        raise OracleParamError("factors live in different row spaces")
    l1, l2 = s1.size, s2.size
    mm = u1.T @ u2
    q, rr = sla.qr(u2 - u1 @ mm, mode="economic", overwrite_a=True)
    leak = np.abs(u1.T @ q).max()
    if leak > LEAK_TOL:
        m2 = u1.T @ q
        q, r2 = sla.qr(q - u1 @ m2, mode="economic", overwrite_a=True)
        mm = mm + m2 @ rr
        rr = r2 @ rr
    e = np.zeros((l1 + l2, l1 + l2), order="F")
    e[:l1, :l1] = np.diag(s1)
    e[:l1, l1:] = mm * s2
    e[l1:, l1:] = rr * s2
    ue, se, _ = lapack_svd(e)
    keep = min(r, int(np.count_nonzero(se > SIGMA_ZERO_RTOL * max(se[0], 1e-300))))
    u = np.hstack([u1, q]) @ ue[:, :keep]
    u, _ = canon_signs(u)
    return u, se[:keep].copy()


def cosines(u_prev, u_next, k, criterion):
    """isma.py:181-201 -- per-mode |dot| or subspace singular values, length
    k, missing modes 0, clipped to [0, 1]."""
    kk = min(k, u_prev.shape[1], u_next.shape[1])
    xi = np.zeros(k)
    if kk:
        a, b = u_prev[:, :kk], u_next[:, :kk]
        if criterion == "modes":
            xi[:kk] = np.abs(np.einsum("ij,ij->j", a, b))
        else:
            xi[:kk] = np.linalg.svd(a.T @ b, compute_uv=False)
    return np.clip(xi, 0.0, 1.0)


def finalize(a, u):
    """isma.py:295-301 -- Q,R = QR(A^T U); SVD(R); rotate; canonical signs."""
    q, rr = householder_qr(a.T @ u)
    ur, sr, vrt = lapack_svd(rr)
    u_new, v_new = canon_signs(u @ vrt.T, q @ ur)
    return u_new, sr, v_new


# --------------------------------------------------------------------------
# L4 driver
# --------------------------------------------------------------------------

def run(a, k, *, r=None, c, tau, strategy="l2n", criterion="modes", seed=0,
        rng=None, do_finalize=True, keep=None, monitor=False, max_rounds=None,
        rows=False, w=None):
    """isma.py:225-303: column sampling (strategies l2n / unf / ort) or,
    with rows=True and a row budget w, ICRS row sampling (unf / ort / ls).
    Returns a dict with u, sigma, v (or None), and a per-round trace list of
    dicts (iteration, unique, counts, remaining, cosines, wall_time[, rows,
    row_counts][, margin]) plus phase timings.  ``max_rounds`` stops after
    that many update rounds (a bounded CPU-timing sample only)."""
    if strategy not in (("unf", "ort", "ls") if rows else ("l2n", "unf", "ort")):
        raise OracleParamError("strategy not valid for this sampling mode")
    if rows and (w is None or int(w) < 1):
        raise OracleParamError("row sampling needs a row budget w >= 1")
    a = dense_f64(a)
    m, n = a.shape
    r = 3 * k if r is None else r
    if k > min(m, n):
        raise OracleParamError("k exceeds min(m, n)")
    keep = k if keep is None else int(keep)
    if not 1 <= keep <= r:
        raise OracleParamError("keep outside 1..r")
    if rng is None:
        rng = np.random.default_rng(seed)
    t_start = time.perf_counter()
    norms2 = column_norms2(a)
    t_norm = time.perf_counter() - t_start
    trace = []

    def one_round(s, weights, u_prev=None):
        t0 = time.perf_counter()
        uni = rng.random(int(c))
        idx, counts = cdf_draw(s, weights, uni)
        d = np.asfortranarray(a[:, idx])
        rest = np.setdiff1d(s, idx, assume_unique=True)
        info = {"unique": idx, "counts": counts, "remaining": rest.size, "t0": t0}
        if not rows:
            sig, v = gram_eig(d)
        else:                                                   # isma.py:168-176
            q = row_weights(d) if u_prev is None or u_prev.shape[1] == 0 \
                else leverage_weights(u_prev)
            ridx, rcnt = cdf_draw(np.arange(m), q, rng.random(int(w)))
            sig, v = gram_eig(scaled_rows(d, ridx, rcnt, q, int(w)))
            info.update(rows=ridx, row_counts=rcnt)
        u2, s2 = lift(d, sig, v, r)
        if monitor:
            info["margin"] = margin_to_cdf_boundary(weights, uni)
        return u2, s2, rest, info

    s = np.arange(n)
    u, sig, s, info = one_round(s, normalized_weights(norms2))
    if rows and sig.size:
        u = orthonormalize(u)                                   # isma.py:267-269
    info.update(iteration=0, cosines=np.zeros(0),
                wall_time=time.perf_counter() - info.pop("t0"))
    trace.append(info)
    xi = np.zeros(k)
    it = 0
    while s.size and (it == 0 or bool(np.any(xi < tau))):
        if max_rounds is not None and it >= max_rounds:
            break
        it += 1
        if strategy == "l2n":
            try:
                wts = normalized_weights(norms2[s])
            except OracleDegenerate:
                break
        elif strategy == "ort":
            wts = residual_weights(a, u, s)
            if wts is None:
                wts = uniform_weights(s.size)
        else:
            wts = uniform_weights(s.size)
        u_rows = None
        if rows and strategy == "ls" and sig.size:
            # factor.truncate(k) (matcore.py:118-128): a C-order copy when it cuts
            u_rows = u if k >= u.shape[1] else u[:, :k].copy()
        u2, s2, s, info = one_round(s, wts, u_rows)
        um, sm = merge(u, sig, u2, s2, r)
        xi = cosines(u, um, k, criterion)
        u, sig = um, sm
        info.update(iteration=it, cosines=xi.copy(),
                    wall_time=time.perf_counter() - info.pop("t0"))
        trace.append(info)
    v = None
    t0 = time.perf_counter()
    if do_finalize and sig.size:
        u, sig, v = finalize(a, u)
    t_fin = time.perf_counter() - t0
    if keep < sig.size:
        u, sig = u[:, :keep].copy(), sig[:keep].copy()
        v = None if v is None else v[:, :keep].copy()
    return {"u": u, "sigma": sig, "v": v, "trace": trace,
            "timings": {"norms": t_norm, "finalize": t_fin,
                        "total": time.perf_counter() - t_start}}


def wedin(a, u, sigma, v, k):
    """quality.py:82-118 -- residual norms, gap estimate, measure."""
    a = np.asarray(a)
    uk, vk, sk = u[:, :k], v[:, :k], sigma[:k]
    rn = float(np.linalg.norm(a @ vk - uk * sk))
    sn = float(np.linalg.norm(a.T @ uk - vk * sk))
    om = float(min(abs(sigma[k - 1] - sigma[k]), sigma[k - 1]))
    degen = bool(om <= SIGMA_ZERO_RTOL * max(sigma[0], 1e-300))
    meas = math.inf if degen else math.hypot(rn, sn) / om
    return {"r_norm": rn, "s_norm": sn, "omega_hat": om, "measure": meas,
            "ceiling": math.sqrt(2.0 * k), "degenerate": degen}


def principal_angle_sines(u1, u2):
    """tests/oracles.py:100-111 semantics -- sines of the principal angles
    between the column spans (accurate near zero), ascending, in radians."""
    q1 = np.linalg.qr(np.asarray(u1, dtype=np.float64))[0]
    q2 = np.linalg.qr(np.asarray(u2, dtype=np.float64))[0]
    s = np.linalg.svd(q2 - q1 @ (q1.T @ q2), compute_uv=False)
    return np.arcsin(np.sort(np.clip(s, 0.0, 1.0)))


def incremental(blocks, k, *, r=None, c, tau, strategy="l2n", criterion="modes",
                seed=0, rows=False, w=None):
    """ooc.py:105-148 -- one-pass fold: per column block an ISMA run with
    finalize off and keep=r sharing ONE generator, then a rank-r merge into
    the accumulator; final truncation to k."""
    r = 3 * k if r is None else r
    rng = np.random.default_rng(seed)
    acc_u = acc_s = None
    trace = []
    for blk in blocks:
        kk = min(k, min(blk.shape))
        out = run(blk, kk, r=r, c=c, tau=tau, strategy=strategy,
                  criterion=criterion, rng=rng, do_finalize=False, keep=r, rows=rows, w=w)
        trace.extend(out["trace"])
        if acc_u is None:
            acc_u, acc_s = out["u"], out["sigma"]
        else:
            acc_u, acc_s = merge(acc_u, acc_s, out["u"], out["sigma"], r)
    if acc_u is None:
        raise OracleParamError("reader produced no blocks")
    return {"u": acc_u[:, :k].copy(), "sigma": acc_s[:k].copy(), "trace": trace}


def column_blocks(a, t):
    """ooc.py:61-66 -- block i covers columns [i n // t, (i+1) n // t)."""
    n = a.shape[1]
    return [np.asfortranarray(a[:, (i * n) // t:((i + 1) * n) // t]) for i in range(t)]
