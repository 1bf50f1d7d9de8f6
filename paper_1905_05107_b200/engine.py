"""Device-resident ISMA engine (column-sampling path).

One ``IsmaEngine`` owns every buffer of a run on one GPU.  The data matrix
A stays in HBM (column-major, ld = m); the running factor lives in one of
two "stacks" S0/S1 of 2r columns each: columns [0, r) hold the current
basis U (zero-padded beyond its l modes), columns [r, r + l2) receive the
merge's orthogonal complement Q, so the merged basis [U1 Q] U_E is one
GEMM over a contiguous operand (no hstack copy, merge.py:86).

Per round (isma.py:276-293) the host issues:
  draw (pod_draw)  -> Gram of A[:, idx] (TN, gathered)  -> eigh (Jacobi)
  -> lift A[:, idx] T (NN, gathered)                     [get_update]
  -> M = U1^T U2 -> W = U2 - U1 M -> CholeskyQR passes   [block_merge]
  -> leak test / second projection -> E-SVD -> [U1 Q] T
  -> cosines                                             [convergence]
and reads back a handful of scalars (g, |S|, keep, CholQR defect, leak,
cosines): the round's only host synchronisation points.
"""

from __future__ import annotations

import time

import numpy as np
import torch

from .device import ColMat, dptr
from .errors import DegenerateDistributionError

REORTH_TOL = 1e-8          # merge.py:34
CHOLQR_STOP_DEFECT = 1e-4  # input defect below which one more CholQR pass is exact to eps

MODE_L2N, MODE_UNIFORM, MODE_WEIGHTS = 0, 1, 2


class MergeWorkspace:
    """Buffers + steps of BLOCK MERGE at rank r for m-row factors: the two
    basis stacks, the update slot, the residual block and the small
    r x r matrices.  Used by the ISMA engine, block_merge and the
    out-of-core driver."""

    def __init__(self, ctx, m, r, *, k=1, criterion="modes", upd_cap=None):
        self.ctx = ctx
        self.m, self.r, self.k = int(m), int(r), int(k)
        self.criterion = criterion
        dev = ctx.device
        f64 = dict(dtype=torch.float64, device=dev)
        r = self.r
        self.S = [ColMat.zeros(self.m, 2 * r, dev), ColMat.zeros(self.m, 2 * r, dev)]
        self.Uupd = ColMat.zeros(self.m, r, dev)
        self.W = ColMat.zeros(self.m, r, dev)
        self.sig_upd = torch.zeros(max(r, upd_cap or 0), **f64)
        sq = r * r
        self.M = torch.zeros(sq, **f64)
        self.C = torch.zeros(sq, **f64)
        self.Gq = torch.zeros(sq, **f64)
        self.Rinv = torch.zeros(sq, **f64)
        self.Rk = torch.zeros(sq, **f64)
        self.Rt = torch.zeros(sq, **f64)
        self.Rt2 = torch.zeros(sq, **f64)
        self.Rtmp = torch.zeros(sq, **f64)
        self.Tm = torch.zeros(2 * r * r, **f64)
        self.sig = [torch.zeros(r, **f64), torch.zeros(r, **f64)]
        self.xi = torch.zeros(max(self.k, 1), **f64)
        self.Ck = torch.zeros(max(self.k, 1) ** 2, **f64)
        self.cur = 0
        self.l = 0
        self.stats = {"cholqr_passes": 0, "reorth": 0, "rounds": 0}

    def load_factor(self, which, u, sigma):
        """Host factor -> stack `which` (cols 0..l) or the update slot."""
        l = int(sigma.shape[0])
        ut = torch.as_tensor(np.ascontiguousarray(np.asarray(u, dtype=np.float64).T))
        if which == "upd":
            self.Uupd.t[:l, :self.m].copy_(ut)
            self.sig_upd[:l].copy_(torch.as_tensor(sigma, dtype=torch.float64))
        else:
            self.S[which].t[:l, :self.m].copy_(ut)
            self.sig[which][:l].copy_(torch.as_tensor(sigma, dtype=torch.float64))
        return l

    # ---------------------------------------------------------- pieces ---
    def cholqr(self, W, l, dest, Rout):
        """Orthonormalise the m x l block W into dest (Q) with W = Q Rout.
        CholeskyQR2 with column scaling; more passes while a pass's input
        was not already orthonormal to CHOLQR_STOP_DEFECT."""
        ctx, r = self.ctx, self.r
        src = W
        for pas in range(6):
            ctx.tn(l, l, 1.0, src, src, dptr(self.Gq), r)
            ctx.cholqr_factor(dptr(self.Gq), r, l, src.m, dptr(self.Rinv), r, dptr(self.Rk), r)
            defect, attempts, _, _ = ctx.read_dinfo(4)
            if src is dest and l <= 64:
                out = dest
            else:
                out = dest if src is not dest else W
            ctx.nn(l, l, 1.0, src, dptr(self.Rinv), r, out)
            if pas == 0:
                Rout.copy_(self.Rk)
            else:
                ctx.small_gemm(l, l, l, 1.0, dptr(self.Rk), r, 0, dptr(Rout), r, 0.0,
                               dptr(self.Rtmp), r)
                Rout.copy_(self.Rtmp)
            self.stats["cholqr_passes"] += 1
            src = out
            if pas >= 1 and defect <= CHOLQR_STOP_DEFECT and attempts == 0:
                break
        if src is not dest:
            dest.t[dest.col0:dest.col0 + l, :dest.m].copy_(src.t[src.col0:src.col0 + l, :src.m])
        return dest

    def merge(self, l1, l2):
        """block_merge (merge.py:37-91) of the current factor (stack cur,
        l1 modes) with the update in Uupd (l2 modes) into the other stack."""
        ctx, r = self.ctx, self.r
        S, Snext = self.S[self.cur], self.S[1 - self.cur]
        if l2 == 0:  # empty update: identity (merge.py:57-58)
            return self.cur, l1
        if l1 == 0:  # empty accumulator: the update is the merge (merge.py:55-56)
            Snext.t[:l2, :self.m].copy_(self.Uupd.t[:l2, :self.m])
            self.sig[1 - self.cur][:l2].copy_(self.sig_upd[:l2])
            return 1 - self.cur, l2
        U1 = S.cols(0, l1)
        U2 = self.Uupd.cols(0, l2)
        ctx.tn(l1, l2, 1.0, U1, U2, dptr(self.M), r)                       # merge.py:65
        ctx.nn(l1, l2, -1.0, U1, dptr(self.M), r, self.W, beta=1.0, Z=U2)  # merge.py:69
        Q = S.cols(r, r + l2)
        self.cholqr(self.W.cols(0, l2), l2, Q, self.Rt)                    # merge.py:70
        ctx.tn(l1, l2, 1.0, U1, Q, dptr(self.C), r)                        # merge.py:72
        ctx.maxabs(dptr(self.C), r, l1, l2, dptr(ctx.dinfo, 8))
        leak = ctx.read_dinfo(9)[8]
        if leak > REORTH_TOL:                                              # merge.py:73-79
            self.stats["reorth"] += 1
            ctx.nn(l1, l2, -1.0, U1, dptr(self.C), r, self.W, beta=1.0, Z=Q)
            self.cholqr(self.W.cols(0, l2), l2, Q, self.Rt2)
            ctx.small_gemm(l1, l2, l2, 1.0, dptr(self.C), r, 0, dptr(self.Rt), r, 1.0,
                           dptr(self.M), r)
            ctx.small_gemm(l2, l2, l2, 1.0, dptr(self.Rt2), r, 0, dptr(self.Rt), r, 0.0,
                           dptr(self.Rtmp), r)
            self.Rt.copy_(self.Rtmp)
        nxt = 1 - self.cur
        ctx.merge_core(dptr(self.sig[self.cur]), l1, dptr(self.M), r, dptr(self.Rt), r,
                       dptr(self.sig_upd), l2, r, r, dptr(self.Tm), 2 * r, r,
                       dptr(self.sig[nxt]))                               # merge.py:80-85
        keep, sweeps = ctx.read_info(2)
        self.stats.setdefault("merge_sweeps", []).append(sweeps)
        ctx.nn(r + l2, keep, 1.0, S, dptr(self.Tm), 2 * r, Snext.cols(0, keep))  # merge.py:86-88
        return nxt, keep

    def cosines(self, old, l_old, new, l_new):
        """convergence_cosines (isma.py:181-201)."""
        ctx, k = self.ctx, self.k
        kk = min(k, l_old, l_new)
        P, Qn = self.S[old].cols(0, max(kk, 1)), self.S[new].cols(0, max(kk, 1))
        if self.criterion == "modes":
            ctx.coldots(P, Qn, k, kk, True, self.xi)
            return self.xi[:k].cpu().numpy().copy()
        xi = np.zeros(k)
        if kk:
            ctx.tn(kk, kk, 1.0, P, Qn, dptr(self.Ck), kk)
            sv = torch.empty(kk, dtype=torch.float64, device=ctx.device)
            ctx.svd_small(dptr(self.Ck), kk, kk, kk, None, 1, sv, None, 1)
            xi[:kk] = sv.cpu().numpy()
        return np.clip(xi, 0.0, 1.0)

class IsmaEngine(MergeWorkspace):
    def __init__(self, ctx, A, *, k, r, c, criterion="modes"):
        self.A = A
        self.n = A.ncols
        self.c = int(c)
        gcap = min(self.c, A.ncols)
        super().__init__(ctx, A.m, r, k=k, criterion=criterion, upd_cap=gcap)
        dev = ctx.device
        f64 = dict(dtype=torch.float64, device=dev)
        n, r, g = self.n, self.r, gcap
        self.gcap = g
        self.norms2 = torch.empty(n, **f64)
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)
        self.live = torch.ones(n, dtype=torch.uint8, device=dev)
        self.uni = torch.empty(self.c, **f64)
        self.h_uni = torch.empty(self.c, dtype=torch.float64).pin_memory()
        self.idx = torch.empty(g, dtype=torch.int32, device=dev)
        self.cnt = torch.empty(g, dtype=torch.int64, device=dev)
        self.G = torch.empty(g * g, **f64)
        self.Tl = torch.empty(g * r, **f64)
        self.npos = 0

    def norm_pass(self):
        """Fused validate + column norms (matcore.py:54, isma.py:260)."""
        self.ctx.colnorms2(self.A, self.norms2, self.nonfinite)
        flag = int(self.nonfinite.item())
        if flag:
            from .errors import ParameterError

            raise ParameterError("matrix contains non-finite entries")
        self.npos = int((self.norms2 > 0).sum().item())
        if self.npos == 0:
            raise DegenerateDistributionError("all candidate column weights are zero")

    def draw(self, mode, rng):
        u = np.asarray(rng.random(int(self.c)), dtype=np.float64)  # one batch (sampling.py:213)
        self.h_uni.numpy()[:] = u
        self.uni.copy_(self.h_uni, non_blocking=True)
        self.ctx.draw(mode, self.norms2 if mode == MODE_L2N else None, self.live, self.n, self.uni,
                      self.c, self.idx, self.cnt)
        g, rem, status = self.ctx.read_info(3)
        return g, rem, status

    def update(self, mode, rng, dest):
        """get_update (isma.py:144-178), column path: returns (g, |S|, keep)."""
        g, rem, status = self.draw(mode, rng)
        if status != 0:
            raise RuntimeError(f"pod_draw status {status}")
        ctx, A = self.ctx, self.A
        ctx.tn(g, g, 1.0, A, A, dptr(self.G), g, xcols=self.idx, ycols=self.idx)
        ctx.gram_eigh(dptr(self.G), g, g, self.r, self.sig_upd, dptr(self.Tl), g)
        rank, keep, sweeps = ctx.read_info(3)
        self.stats.setdefault("eigh_sweeps", []).append(sweeps)
        if keep > 0:
            ctx.nn(g, keep, 1.0, A, dptr(self.Tl), g, dest, xcols=self.idx)
        return g, rem, keep

    def finalize(self):
        """isma.py:295-301: Q, R = QR(A^T U); SVD(R); U V_R, Q U_R; signs."""
        ctx, r, n, l = self.ctx, self.r, self.n, self.l
        dev = ctx.device
        U = self.S[self.cur].cols(0, l)
        Cm = ColMat.zeros(n, l, dev)
        ctx.tn(n, l, 1.0, self.A, U, Cm.ptr, n)                            # A^T U
        Qc = ColMat.zeros(n, l, dev)
        Rc = torch.zeros(r * r, dtype=torch.float64, device=dev)
        self.cholqr(Cm, l, Qc, Rc)
        Ur = torch.zeros(l * l, dtype=torch.float64, device=dev)
        Vr = torch.zeros(l * l, dtype=torch.float64, device=dev)
        sr = torch.zeros(l, dtype=torch.float64, device=dev)
        ctx.svd_small(dptr(Rc), r, l, l, dptr(Ur), l, sr, dptr(Vr), l)     # _svd(rr)
        nxt = 1 - self.cur
        Unew = self.S[nxt].cols(0, l)
        ctx.nn(l, l, 1.0, U, dptr(Vr), l, Unew)                            # u @ vrt.T
        Vnew = ColMat.zeros(n, l, dev)
        ctx.nn(l, l, 1.0, Qc, dptr(Ur), l, Vnew)                           # q @ ur
        ctx.fix_signs(Unew, l, Vnew, n)
        self.sig[nxt][:l].copy_(sr)
        self.cur = nxt
        return Vnew

    # ------------------------------------------------------------ driver ---
    def run(self, rng, *, strategy, tau, finalize, keep, trace_cls):
        """isma_run main loop (isma.py:258-303) on the device."""
        self.norm_pass()
        traces = []
        t0 = time.perf_counter()
        g, rem, l = self.update(MODE_L2N, rng, self.S[self.cur])
        self.npos -= g
        self.sig[self.cur][:l].copy_(self.sig_upd[:l])
        self.l = l
        traces.append(trace_cls(0, g, 0, rem, np.zeros(0), time.perf_counter() - t0))
        xi = np.zeros(self.k)
        it = 0
        mode = MODE_L2N if strategy == "l2n" else MODE_UNIFORM
        while rem and (it == 0 or bool(np.any(xi < tau))):
            it += 1
            t0 = time.perf_counter()
            if mode == MODE_L2N and self.npos <= 0:
                break  # l2n over only zero-norm columns (isma.py:211-215, 280-281)
            g, rem, l2 = self.update(mode, rng, self.Uupd)
            if mode == MODE_L2N:
                self.npos -= g
            old, l_old = self.cur, self.l
            nxt, l_new = self.merge(l_old, l2)
            xi = self.cosines(old, l_old, nxt, l_new)
            self.cur, self.l = nxt, l_new
            self.stats["rounds"] += 1
            traces.append(trace_cls(it, g, 0, rem, xi.copy(), time.perf_counter() - t0))
        v = None
        if finalize and self.l:
            v = self.finalize()
        elif self.l:
            self.ctx.fix_signs(self.S[self.cur].cols(0, self.l), self.l)
        return traces, v

    def result(self, keep, v=None):
        l = min(self.l, keep)
        u = self.S[self.cur].to_numpy(l) if l else np.zeros((self.m, 0))
        s = self.sig[self.cur][:l].cpu().numpy().copy()
        vv = None if v is None else (v.to_numpy(l) if l else np.zeros((self.n, 0)))
        return u, s, vv
