"""Device-resident ISMA engine (column sampling and ICRS row sampling).

Layout in HBM (one engine per run and GPU):
  A          m x n column-major, ld = m (the data matrix, read in place)
  S0, S1     m x 2r "stacks": columns [0, r) hold the current basis U (zero
             beyond its l modes), columns [r, 2r) receive the merge's
             orthogonal complement Q, so the merged basis [U1 Q] U_E is ONE
             GEMM over a contiguous operand (no hstack, merge.py:86)
  Uupd, W    m x r: the lifted update U2 and the projection residual
  small      r x r matrices (M, C, Grams, R factors), 2r x r rotation T

Every kernel of a round runs at CAPACITY (g = min(c, n) sampled columns,
l = r modes) on zero-padded operands: padded sample slots carry gather
index -1 (a zero column), padded modes are zero columns with sigma = 0.
Zero columns add only zero singular values and never pass the reference's
rank cuts, so results equal the reference's on the active part.  Data-
dependent branches of the reference -- the number of CholeskyQR passes
and the second projection of merge.py:73-79 -- are device-side gates
(int32 flags) read by the kernels themselves.  A round is therefore a
static launch sequence with no host synchronisation: the host uploads the
round's uniforms, launches (or replays a captured CUDA graph), and reads
back one small record (g, |S|, ranks, keep) plus the k cosines.

Per round (isma.py:276-293):
  draw -> Gram of A[:, idx] (TN, gathered) -> eigh (pivoted Cholesky +
  Jacobi) -> lift A[:, idx] T (NN, gathered)                 [get_update]
  M = U1^T U2 -> W = U2 - U1 M -> CholeskyQR2 (+ <= 2 gated passes)
  -> leak gate -> gated second projection -> E-SVD (Jacobi)
  -> [U1 Q] T                                                [block_merge]
  -> cosines                                                 [convergence]
With rows=True the update draws rows (row norms or leverage), builds the
dedup-scaled row block Y and eigensolves Y^T Y (isma.py:168-176).
"""

from __future__ import annotations

import time

import numpy as np
import torch

from . import _lib
from .device import ColMat, dptr
from .errors import DegenerateDistributionError, ParameterError

REORTH_TOL = 1e-8  # merge.py:34
# CTAs of the pipelined update's GEMMs (which run beside the merge chain on
# the side stream); 0 = no cap.  POD_UPDATE_GRID_CAP overrides.
# (measured: caps of 148-200 CTAs and forking the update at the round start
# instead of after the merge's GEMM phase are within noise or slower)
UPDATE_GRID_CAP = int(__import__("os").environ.get("POD_UPDATE_GRID_CAP", "0"))
#: CTA cap for the merge's GEMM phase in pipelined rounds: the side stream's
#: eigensolve holds an 8-CTA cluster plus the pivoted-Cholesky CTA, so the
#: one-wave GEMM grids (2 CTAs per SM) are sized for the remaining SMs
#: instead of spilling a partial second wave (config 2: 57.1 -> 55.2 ms).
#: Default 2 * (SMs - 9); POD_MERGE_GRID_CAP overrides (0 = no cap).
MERGE_GRID_CAP_ENV = __import__("os").environ.get("POD_MERGE_GRID_CAP")


def merge_grid_cap(device):
    if MERGE_GRID_CAP_ENV is not None:
        return int(MERGE_GRID_CAP_ENV)
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    return max(2 * (sms - 9), 0)
CHOLQR_PASSES = 4  # passes 0-1 always (CholeskyQR2); passes 2..3 gated on the previous pass

MODE_L2N, MODE_UNIFORM, MODE_WEIGHTS, MODE_ORT, MODE_ROWS = 0, 1, 2, 3, 4
ORT_DEGENERATE_RTOL = 1e-14  # sampling.py:158 degenerate_rtol

# round record slots (int64)
REC_G, REC_REM, REC_STATUS, REC_RANK, REC_KEEP_UPD, REC_EIGH_SWEEPS, REC_KEEP, REC_MERGE_SWEEPS = \
    range(8)
REC_H, REC_HREM, REC_HSTATUS = 8, 9, 10  # row draw (ICRS): distinct rows, -, status
REC_LEN = 11  # rec[0]: merge record; rec[1 + b]: update record of buffer b
UPDATE_FIELDS = (REC_G, REC_REM, REC_STATUS, REC_RANK, REC_KEEP_UPD, REC_EIGH_SWEEPS, REC_H,
                 REC_HREM, REC_HSTATUS)

# gate slots (int32)
G_QR = 0            # main CholeskyQR passes: slots 0..4
G_LEAK = 5          # merge.py:73 second projection
G_RQR = 6           # second-projection CholeskyQR passes: slots 6..10
G_FQR = 11          # finalize CholeskyQR passes: 11..15
N_GATES = 16

DINFO_BREAKDOWN = 8  # POD_DINFO_BREAKDOWN (include/podsketch_b200.h)

#: precision="mixed": finalize's A^T U runs on the tcgen05 kernel; the sampled
#: Gram too only with POD_TC_GRAM=1 -- measured at config 4 (r02): 2.0 s with
#: it vs 1.46 s without (the pipelined Gram's long 192-KB-smem CTAs crowd the
#: merge chain off the SMs), so the Gram stays on fp64 DMMA by default
TC_GRAM = __import__("os").environ.get("POD_TC_GRAM", "0") == "1"
#: speculative merge core: the E-SVD starts on the first CholeskyQR's R while
#: the leak check (U1^T Q, merge.py:72) runs beside it; a gated re-run covers
#: the rounds whose second projection fires.  POD_SPEC_CORE=0 disables.
SPEC_CORE = __import__("os").environ.get("POD_SPEC_CORE", "1") != "0"
#: largest E (2r columns) the core runs speculatively for.  Measured
#: (tools/spec_probe.py): config 2 (120) 51.9 -> 49.7 ms; config 3 (300)
#: neutral (the side-stream update chain sets the round there); config 4
#: (384): U1^T Q sits at ~1e-8, next to the threshold, the check fires in
#: 4-19 of 34 rounds and every fire re-runs a 5-7 ms core (1.53 -> 2.05 s)
SPEC_MAX_N = 256
#: CTA cap of the speculative leak check's GEMM (full grid: its CTAs crowd the
#: E-SVD's cluster -- config 2 57.8 ms; 8: the check outlasts the core, 66 ms;
#: 32-64: 51.2-51.4 ms vs 52.3 serial)
LEAK_GRID_CAP = int(__import__("os").environ.get("POD_LEAK_GRID_CAP", "64"))

#: the merge's second projection (merge.py:73-79) factors its nearly
#: orthonormal W2 with one CholeskyQR pass, the second only when the first
#: reports a defect > 1e-4 or a shift.  POD_SECOND_PROJ_ONE_PASS=0: always two.
SECOND_PROJ_ONE_PASS = __import__("os").environ.get("POD_SECOND_PROJ_ONE_PASS", "1") != "0"

#: the merge's CholeskyQR2 (merge.py:70) skips its second m x r apply: the
#: pass-1 factor's R^-1 stays a small r x r matrix ("fold") that multiplies
#: the leak matrix U1^T Q (merge.py:72) and the lower half of the rotation
#: (merge.py:86-88) instead -- [U1 Q1 R^-1] T = [U1 Q1] [T_top; R^-1 T_bot].
#: Q is materialized (gated) only when a further CholeskyQR pass or the
#: second projection needs it.  POD_FOLD_QR=0 disables.
FOLD_QR = __import__("os").environ.get("POD_FOLD_QR", "1") != "0"

#: out-of-place CholeskyQR applies Q = W R^-1 skip the zero half of the upper
#: triangular R^-1: column chunk [c0, c1) multiplies only W's first c1
#: columns (bitwise equal to the full product; tools/trmm_split_probe.py:
#: l = 150 split at 80: 1.92 -> 1.48 ms, l = 192 in 64-wide chunks: 3.11 ->
#: 2.12 ms at m = 1M; l <= 96 loses).  POD_TRI_APPLY=0 disables.
TRI_APPLY = __import__("os").environ.get("POD_TRI_APPLY", "1") != "0"


def tri_apply_bounds(l):
    """Column chunk boundaries of the triangular apply for width l."""
    if not TRI_APPLY or l < 120:
        return [0, l]
    if l <= 160:
        return [0, 80, l]
    b = list(range(0, l, 64))
    if l - b[-1] < 32:  # fold a thin last chunk into its neighbour
        b.pop()
    return b + [l]


#: row-sharded rounds over NCCL are captured into CUDA graphs like the
#: single-GPU rounds (POD_SHARDED_GRAPHS=0: eager launches)
SHARDED_GRAPHS = __import__("os").environ.get("POD_SHARDED_GRAPHS", "1") != "0"

#: with the folded pass, the leak GEMM U1^T Q1 (merge.py:72) no longer waits
#: for the pass-1 factor: it runs on its own stream beside that single-CTA
#: kernel (non-speculative, unsharded merges).  POD_EARLY_LEAK=0 disables.
EARLY_LEAK = __import__("os").environ.get("POD_EARLY_LEAK", "1") != "0"

#: NN GEMMs whose output a CholeskyQR pass consumes next form its Gram in
#: their epilogue (pod_gemm_nn_gram, q <= 64) instead of a TN pass over the
#: output.  POD_NN_GRAM=0 disables.
NN_GRAM = __import__("os").environ.get("POD_NN_GRAM", "1") != "0"

#: POD_FUSED_COSINES=1: the merge's rotation GEMM also forms the convergence
#: cosines (criterion "modes") in its epilogue (pod_gemm_nn_dots) instead of
#: the separate coldots pass.  Off by default -- measured slower (config 2
#: 49.13 -> 49.37 ms, config 3 2.905 -> 2.942 s): the epilogue re-reads
#: U_old's k columns from L2 on the rotation's critical path and loads only
#: the first column group's CTAs, which costs more than the 2-kernel pass.
FUSED_COSINES = __import__("os").environ.get("POD_FUSED_COSINES", "0") == "1"

#: debug/parity switch: when set, every run copies each round's drawn index
#: set and counts (the draw slot's idx/cnt, still intact when the round's
#: record is read) to the host -> IsmaEngine.draw_log, isma.LAST_DRAWS.
#: Costs one small synchronous D2H per round; off for timed runs.
RECORD_DRAWS = False


#: update slots of the ISMA engine: round t merges slot t % 3 while its side
#: stream finishes update(t+1) (eigensolve + lift, slot (t+1) % 3) and starts
#: update(t+2) (draw + Gram, slot (t+2) % 3)
NSLOT = 3

#: widest in-place Q <- Q R^-1 the NN kernel takes (pod_gemm_nn_f64)
NN_INPLACE_MAX_Q = 192


class MergeWorkspace:
    """Buffers and launch sequences of BLOCK MERGE at rank r for m-row
    factors (used by the ISMA engine, block_merge and the one-pass
    incremental driver)."""

    def __init__(self, ctx, m, r, *, k=1, criterion="modes", upd_cap=None, comm=None,
                 row_offset=0, nupd=1):
        from .parallel import Comm

        self.ctx = ctx
        self.comm = comm if comm is not None else Comm()
        self.row_offset = int(row_offset)
        self.m, self.r, self.k = int(m), int(r), int(k)
        self.criterion = criterion
        dev = ctx.device
        f64 = dict(dtype=torch.float64, device=dev)
        r = self.r
        self.S = [ColMat.zeros(self.m, 2 * r, dev), ColMat.zeros(self.m, 2 * r, dev)]
        # update slots (three for the cross-round pipeline of the ISMA engine)
        self.Uupd_b = [ColMat.zeros(self.m, r, dev) for _ in range(nupd)]
        self.sig_upd_b = [torch.zeros(max(r, upd_cap or 0), **f64) for _ in range(nupd)]
        self.Uupd, self.sig_upd = self.Uupd_b[0], self.sig_upd_b[0]
        self.W = ColMat.zeros(self.m, r, dev)
        sq = r * r
        self.M = torch.zeros(sq, **f64)
        self.C = torch.zeros(sq, **f64)
        self.Gq = torch.zeros(sq, **f64)
        self.Rinv = torch.zeros(sq, **f64)
        self.Rk = torch.zeros(sq, **f64)
        self.Rt = torch.zeros(sq, **f64)
        self.Rt2 = torch.zeros(sq, **f64)
        self.Rtmp = torch.zeros(sq, **f64)
        # folded CholeskyQR pass (FOLD_QR): the unapplied R^-1, the raw leak
        # matrix U1^T Q1 and an identity to reset the fold with
        self.Rfold = torch.eye(r, **f64).reshape(-1).contiguous()
        self.Ident = torch.eye(r, **f64).reshape(-1).contiguous()
        self.C1 = torch.zeros(sq, **f64)
        self.Tm = torch.zeros(2 * r * r, **f64)
        self.sig = [torch.zeros(r, **f64), torch.zeros(r, **f64)]
        kk = max(self.k, 1)
        self.xi = torch.zeros(kk, **f64)
        self.Ck = torch.zeros(kk * kk, **f64)
        self.gates = torch.ones(N_GATES, dtype=torch.int32, device=dev)
        self.rec = torch.zeros((1 + nupd, REC_LEN), dtype=torch.int64, device=dev)
        self.h_rec = torch.zeros((1 + nupd, REC_LEN), dtype=torch.int64).pin_memory()
        self.h_xi = torch.zeros(kk, dtype=torch.float64).pin_memory()
        # sticky CholeskyQR breakdown flag (dinfo[POD_DINFO_BREAKDOWN]), read with the record
        self.h_breakdown = torch.zeros(1, dtype=torch.float64).pin_memory()
        self.leak = torch.zeros(1, **f64)
        self._spec = None
        self._leak_stream = None
        self._qscratch = {}
        self.cur = 0
        self.l = 0
        self.stats = {"rounds": 0}

    # ------------------------------------------------------------ helpers --
    def gate(self, i):
        return self.gates[i:i + 1]

    def load_factor(self, which, u, sigma):
        """Host factor -> stack `which` (cols 0..l) or the update slot; the
        padding columns and sigmas are zeroed."""
        l = int(sigma.shape[0])
        ut = torch.as_tensor(np.ascontiguousarray(np.asarray(u, dtype=np.float64).T))
        if which == "upd":
            self.Uupd.t[:self.r, :self.m].zero_()
            self.Uupd.t[:l, :self.m].copy_(ut)
            self.sig_upd.zero_()
            self.sig_upd[:l].copy_(torch.as_tensor(sigma, dtype=torch.float64))
        else:
            self.S[which].t[:self.r, :self.m].zero_()
            self.S[which].t[:l, :self.m].copy_(ut)
            self.sig[which].zero_()
            self.sig[which][:l].copy_(torch.as_tensor(sigma, dtype=torch.float64))
        return l

    # ------------------------------------------------------- launch pieces --
    def cholqr_ops(self, Wsrc, Q, l, Rout, gate_base, first_gate=None, sharded=True,
                   gram_ready=False, fold=False, after_gram1=None):
        """Q = orthonormal factor of Wsrc (m x l) with Wsrc = Q Rout (the
        Householder QR of merge.py:70/76, matcore.py:209 replaced by
        CholeskyQR passes).  Passes 0 and 1 (CholeskyQR2) run when first_gate
        is null or set -- pass 0 into a scratch block, pass 1 from it into Q,
        so both GEMMs are out of place (column-group parallel); further
        passes run in place when the previous pass asked for them (slot
        gate_base + p).  gram_ready: self.Gq already holds Wsrc^T Wsrc (from
        the producing GEMM's Gram epilogue); pass 0's apply forms pass 1's
        Gram the same way when the shape allows (nn_gram).  fold: pass 0
        writes Q directly and pass 1 only factors -- its R^-1 is left in
        self.Rfold for the caller to apply to the small matrices (FOLD_QR);
        `materialize_q` turns Q into the true factor when someone needs it."""
        ctx, r = self.ctx, self.r
        assert not fold or (first_gate is None and l == r)
        g0 = first_gate
        tmp = self._scratch_like(Q)
        src = Wsrc
        # the running R: pass 0 writes it, later passes fold R_p R into it
        # inside the factor kernel (pod_cholqr_factor2)
        rk = None if l <= 64 else dptr(self.Rk)
        fuse = NN_GRAM and ctx.nn_gram_ok(l, l)
        have_gram = gram_ready
        # second projection (first_gate set, merge.py:76): W2 = Q - U1 C is
        # orthonormal to ~1e-8, where ONE CholeskyQR pass is already exact to
        # working precision (error ~ kappa^2 u) -- pass 0 writes Q directly and
        # pass 1 runs (in place) only when pass 0's scaled Gram was off the
        # identity by more than 1e-4 or needed a shift, like passes >= 2
        one = first_gate is not None and SECOND_PROJ_ONE_PASS
        for p in range(2):  # CholeskyQR2: Wsrc -> tmp -> Q
            dst = (Q if (one or fold) else tmp) if p == 0 else Q
            gp = g0 if (p == 0 or not one) else self.gate(gate_base + 1)
            if not have_gram:
                ctx.tn(l, l, 1.0, src, src, dptr(self.Gq), r, gate=gp, tag="tn_cholqr_gram")
            if sharded:
                self.comm.allreduce_sum_(self.Gq)
            if p == 1 and after_gram1 is not None:
                after_gram1()
            ctx.cholqr_factor_acc(dptr(self.Gq), r, l, src.m, dptr(self.Rinv), r,
                                  dptr(Rout) if p == 0 else rk, r,
                                  None if p == 0 else dptr(Rout), r,
                                  gate_in=gp, gate_out=self.gate(gate_base + p + 1),
                                  first_pass=1 if (p == 0 and not one) else 0)
            if p == 1 and fold:  # the apply is folded into the small matrices
                ctx.small_copy(l, l, dptr(self.Rinv), r, dptr(self.Rfold), r)
                break
            if p == 1 and one and l > NN_INPLACE_MAX_Q:  # in place through the scratch block
                self.apply_upper(src, self.Rinv, l, tmp, gate=gp)
                ctx.small_copy(Q.m, l, tmp.ptr, tmp.ld, Q.ptr, Q.ld, gate=gp)
            elif p == 0 and fuse:  # the apply also forms pass 1's Gram
                ctx.nn_gram(l, l, 1.0, src, dptr(self.Rinv), r, dst, dptr(self.Gq), r, gate=gp,
                            tag="nn_cholqr_apply")
                have_gram = True
            else:
                self.apply_upper(src, self.Rinv, l, dst, gate=gp)
                have_gram = False
            src = dst
        for p in range(2, CHOLQR_PASSES):
            gp = self.gate(gate_base + p)
            if fold and p == 2:
                self.materialize_q(Q, gp)
            ctx.tn(l, l, 1.0, Q, Q, dptr(self.Gq), r, gate=gp, tag="tn_cholqr_gram")
            if sharded:
                self.comm.allreduce_sum_(self.Gq)
            ctx.cholqr_factor_acc(dptr(self.Gq), r, l, Q.m, dptr(self.Rinv), r, rk, r,
                                  dptr(Rout), r, gate_in=gp,
                                  gate_out=self.gate(gate_base + p + 1), first_pass=0)
            if l <= NN_INPLACE_MAX_Q:
                ctx.nn(l, l, 1.0, Q, dptr(self.Rinv), r, Q, gate=gp, tag="nn_cholqr_apply")
            else:  # wider than the in-place NN kernel: through the scratch block
                self.apply_upper(Q, self.Rinv, l, tmp, gate=gp)
                ctx.small_copy(Q.m, l, tmp.ptr, tmp.ld, Q.ptr, Q.ld, gate=gp)

    def apply_upper(self, src, T, l, dst, gate=None):
        """dst = src T for an upper triangular l x l T (leading dimension r),
        src and dst distinct blocks."""
        b = tri_apply_bounds(l)
        for c0, c1 in zip(b[:-1], b[1:]):
            self.ctx.nn(c1, c1 - c0, 1.0, src.cols(0, c1), dptr(T, c0 * self.r), self.r,
                        dst.cols(c0, c1), gate=gate, tag="nn_cholqr_apply")

    def materialize_q(self, Q, gate):
        """Folded CholeskyQR (FOLD_QR): Q <- Q Rfold, Rfold <- I, when `gate`
        is set (a further pass or the second projection reads the true Q)."""
        ctx, r = self.ctx, self.r
        if r <= NN_INPLACE_MAX_Q:
            ctx.nn(r, r, 1.0, Q, dptr(self.Rfold), r, Q, gate=gate, tag="nn_cholqr_apply")
        else:
            tmp = self._scratch_like(Q)
            self.apply_upper(Q, self.Rfold, r, tmp, gate=gate)
            ctx.small_copy(Q.m, r, tmp.ptr, tmp.ld, Q.ptr, Q.ld, gate=gate)
        ctx.small_copy(r, r, dptr(self.Ident), r, dptr(self.Rfold), r, gate=gate)

    def _scratch_like(self, Q):
        """m x r scratch block for the first CholeskyQR pass (one per row count)."""
        key = Q.m
        buf = self._qscratch.get(key)
        if buf is None:
            buf = ColMat.zeros(Q.m, self.r, self.ctx.device)
            self._qscratch[key] = buf
        return buf

    def merge_ops(self, cur, ub=0, before_core=None, cos_out=None):
        """block_merge (merge.py:37-91) of stack `cur` (U1, sig[cur]) with
        update slot `ub` (Uupd, sig_upd) into stack 1 - cur, at capacity r.
        `before_core` is issued after the GEMM phase, before the E-SVD.
        cos_out: the rotation also writes the raw convergence cosines
        u_old_j . u_new_j, j < k (isma.py:195-198, criterion "modes")."""
        ctx, r = self.ctx, self.r
        S, Snext = self.S[cur], self.S[1 - cur]
        U1 = S.cols(0, r)
        U2 = self.Uupd_b[ub].cols(0, r)
        sig_upd = self.sig_upd_b[ub]
        Q = S.cols(r, 2 * r)
        core = (dptr(self.sig[cur]), r, dptr(self.M), r, dptr(self.Rt), r, dptr(sig_upd), r, r, r,
                dptr(self.Tm), 2 * r, r, dptr(self.sig[1 - cur]))
        info = self.rec[0, REC_KEEP:]
        ctx.tn(r, r, 1.0, U1, U2, dptr(self.M), r, tag="tn_merge_proj")       # merge.py:65
        self.comm.allreduce_sum_(self.M)
        spec = self.speculative_core()
        early = FOLD_QR and EARLY_LEAK and not spec and not self.comm.active
        hook = None
        if early:
            if self._leak_stream is None:
                self._leak_stream = torch.cuda.Stream(ctx.device)

            def hook():  # Q1 and its Gram are out: U1^T Q1 beside the pass-1 factor
                ev = torch.cuda.Event()
                ev.record(torch.cuda.current_stream(ctx.device))
                self._leak_stream.wait_event(ev)
                ctx.ws_suffix = "_leak"
                try:
                    with torch.cuda.stream(self._leak_stream):
                        ctx.tn(r, r, 1.0, U1, Q, dptr(self.C1), r, tag="tn_merge_leak")
                finally:
                    ctx.ws_suffix = ""
        if NN_GRAM and ctx.nn_gram_ok(r, r):  # the residual's Gram in the same pass
            ctx.nn_gram(r, r, -1.0, U1, dptr(self.M), r, self.W, dptr(self.Gq), r, beta=1.0,
                        Z=U2, tag="nn_merge_resid")                          # merge.py:69
            self.cholqr_ops(self.W, Q, r, self.Rt, G_QR, gram_ready=True,
                            fold=FOLD_QR, after_gram1=hook)                  # merge.py:70
        else:
            ctx.nn(r, r, -1.0, U1, dptr(self.M), r, self.W, beta=1.0, Z=U2,
                   tag="nn_merge_resid")                                     # merge.py:69
            self.cholqr_ops(self.W, Q, r, self.Rt, G_QR, fold=FOLD_QR,
                            after_gram1=hook)                                # merge.py:70
        if spec:
            # the E-SVD on the first-pass (M, R) starts now; the leak check
            # (merge.py:72-73) runs beside it on its own stream, and the
            # gated second projection re-runs the core only when it fired
            main = torch.cuda.current_stream(ctx.device)
            ev = torch.cuda.Event()
            ev.record(main)
            if before_core is not None:
                before_core()
            ctx.merge_core(*core, info=info)                                 # merge.py:80-85
            self._leak_stream.wait_event(ev)
            ctx.ws_suffix = "_leak"
            lib = _lib.load()
            lib.pod_set_grid_cap(LEAK_GRID_CAP)
            try:
                with torch.cuda.stream(self._leak_stream):
                    self.leak_check_ops(U1, Q)
            finally:
                lib.pod_set_grid_cap(0)
                ctx.ws_suffix = ""
            main.wait_stream(self._leak_stream)
        elif early:
            torch.cuda.current_stream(ctx.device).wait_stream(self._leak_stream)
            # a further CholeskyQR pass materialized Q after the early product
            self.leak_check_ops(U1, Q, tn_gate=self.gate(G_QR + 2))
        else:
            self.leak_check_ops(U1, Q)
        gl = self.gate(G_LEAK)                                               # merge.py:73-79
        if FOLD_QR:
            self.materialize_q(Q, gl)
        ctx.nn(r, r, -1.0, U1, dptr(self.C), r, self.W, beta=1.0, Z=Q, gate=gl,
               tag="nn_merge_resid")
        self.cholqr_ops(self.W, Q, r, self.Rt2, G_RQR, first_gate=gl)
        ctx.small_gemm(r, r, r, 1.0, dptr(self.C), r, 0, dptr(self.Rt), r, 1.0, dptr(self.M), r,
                       gate=gl)
        ctx.small_gemm(r, r, r, 1.0, dptr(self.Rt2), r, 0, dptr(self.Rt), r, 0.0,
                       dptr(self.Rtmp), r, gate=gl)
        ctx.small_copy(r, r, dptr(self.Rtmp), r, dptr(self.Rt), r, gate=gl)
        if spec:
            ctx.merge_core_gated(*core, info, gl)
        else:
            if before_core is not None:
                before_core()
            ctx.merge_core(*core, info=info)                                 # merge.py:80-85
        if FOLD_QR:  # T_bot <- Rfold T_bot: the rotation reads Q1, not Q1 R^-1
            tbot = dptr(self.Tm, r)
            ctx.small_gemm(r, r, r, 1.0, dptr(self.Rfold), r, 0, tbot, 2 * r, 0.0,
                           dptr(self.Rtmp), r)
            ctx.small_copy(r, r, dptr(self.Rtmp), r, tbot, 2 * r)
        if cos_out is not None:  # rotation + cosines in one pass (isma.py:195-198)
            ctx.nn_dots(2 * r, r, 1.0, S, dptr(self.Tm), 2 * r, Snext.cols(0, r), self.k, cos_out,
                        tag="nn_merge_rotate")                               # merge.py:86-88
        else:
            ctx.nn(2 * r, r, 1.0, S, dptr(self.Tm), 2 * r, Snext.cols(0, r),
                   tag="nn_merge_rotate")                                    # merge.py:86-88

    def leak_check_ops(self, U1, Q, tn_gate=None):
        """C = U1^T Q and the gate max|C| > REORTH_TOL (merge.py:72-73)."""
        ctx, r = self.ctx, self.r
        if FOLD_QR:  # Q holds Q1: U1^T Q = (U1^T Q1) Rfold
            ctx.tn(r, r, 1.0, U1, Q, dptr(self.C1), r, gate=tn_gate, tag="tn_merge_leak")
            self.comm.allreduce_sum_(self.C1)
            ctx.small_gemm(r, r, r, 1.0, dptr(self.C1), r, 0, dptr(self.Rfold), r, 0.0,
                           dptr(self.C), r)
        else:
            ctx.tn(r, r, 1.0, U1, Q, dptr(self.C), r, tag="tn_merge_leak")
            self.comm.allreduce_sum_(self.C)
        ctx.maxabs(dptr(self.C), r, r, r, dptr(self.leak), thr=REORTH_TOL,
                   gate_out=self.gate(G_LEAK))

    def speculative_core(self):
        """Whether the merge core runs speculatively beside the leak check:
        single shard (no collective on the side stream), a single-cluster
        E-SVD (pod_merge_core_gatable) of at most SPEC_MAX_N columns,
        POD_SPEC_CORE not 0."""
        if self._spec is None:
            self._spec = (SPEC_CORE and not self.comm.active and 2 * self.r <= SPEC_MAX_N
                          and bool(_lib.load().pod_merge_core_gatable(self.r, self.r)))
            if self._spec:
                self._leak_stream = torch.cuda.Stream(self.ctx.device)
        return self._spec

    def fused_cosines(self):
        """Whether the merge's rotation forms the cosines (criterion modes)."""
        return FUSED_COSINES and self.criterion == "modes" and 1 <= self.k <= self.r

    def cosines_ops(self, old, new, fused=False):
        """convergence_cosines (isma.py:181-201) into self.xi (length k);
        padded (missing) modes are zero columns and contribute 0.  fused:
        the rotation already wrote the raw dots (only the shard sum is left)."""
        ctx, k = self.ctx, self.k
        P, Qn = self.S[old].cols(0, k), self.S[new].cols(0, k)
        if self.criterion == "modes":
            if not fused:
                ctx.coldots(P, Qn, k, k, False, self.xi)  # raw dots; |.| and clip on the host
            self.comm.allreduce_sum_(self.xi)
        else:
            ctx.tn(k, k, 1.0, P, Qn, dptr(self.Ck), k, tag="tn_cosines")
            self.comm.allreduce_sum_(self.Ck)
            ctx.svd_small(dptr(self.Ck), k, k, k, None, 1, self.xi, None, 1)

    def readback(self):
        self.h_rec.copy_(self.rec, non_blocking=True)
        self.h_xi.copy_(self.xi, non_blocking=True)
        self.h_breakdown.copy_(self.ctx.dinfo[DINFO_BREAKDOWN:DINFO_BREAKDOWN + 1],
                               non_blocking=True)

    def clear_breakdown(self):
        self.ctx.dinfo[DINFO_BREAKDOWN:DINFO_BREAKDOWN + 1].zero_()

    def read_record(self, ub=0):
        """(record, cosines): merge fields from rec[0], update fields of
        buffer `ub` from rec[1 + ub]."""
        torch.cuda.current_stream(self.ctx.device).synchronize()
        if self.h_breakdown[0] != 0.0:
            # every shifted CholeskyQR retry broke down: the factor is unusable
            # (LAPACK's Householder QR cannot fail; report it like a LAPACK error)
            self.clear_breakdown()
            raise np.linalg.LinAlgError("CholeskyQR breakdown: the merge residual could not be "
                                        "factored after 8 shifted retries")
        hr = self.h_rec.tolist()
        rec = [int(x) for x in hr[0]]
        for i in UPDATE_FIELDS:
            rec[i] = int(hr[1 + ub][i])
        xi = np.clip(np.abs(self.h_xi.numpy().astype(np.float64)), 0.0, 1.0)
        return rec, xi

    def fix_signs_ops(self, U, l, V=None, n=0):
        """fix_signs (matcore.py:148-165) of a row-sharded basis: per-shard
        arg-max, allgather, deterministic global choice, local flip."""
        ctx = self.ctx
        if not self.comm.active:
            ctx.fix_signs(U, l, V, n)
            return
        dev = ctx.device
        val = torch.empty(l, dtype=torch.float64, device=dev)
        row = torch.empty(l, dtype=torch.int64, device=dev)
        sign = torch.empty(l, dtype=torch.float64, device=dev)
        ctx.colargmax(U, l, self.row_offset, val, row, sign)
        from .parallel import combine_signs

        g = combine_signs(self.comm.allgather(val), self.comm.allgather(row),
                          self.comm.allgather(sign))
        sign.copy_(g)
        ctx.scale_cols(U, l, sign)
        if V is not None:
            ctx.scale_cols(V, l, sign)

    def gather_rows(self, U, l, m_total):
        """Full m_total x l host copy of a row-sharded basis."""
        from .parallel import gather_row_shards

        return gather_row_shards(U.t[U.col0:U.col0 + l, :U.m], m_total, self.comm)

    def merge_now(self, cur):
        """Standalone merge (block_merge): returns (next stack, keep)."""
        self.merge_ops(cur)
        self.readback()
        rec, _ = self.read_record(0)
        return 1 - cur, rec[REC_KEEP]


class IsmaEngine(MergeWorkspace):
    """The ISMA loop on one GPU (or one row shard).

    Cross-round pipeline: an update (draw, Gram, eigensolve, lift) only
    depends on the candidate set, not on the merges, so each captured round
    graph runs merge(t) + cosines(t) on the main stream and, on a side stream
    forked at the start of the round, the eigensolve and lift of update(t+1)
    and the draw and Gram of update(t+2) -- three update slots in rotation.
    The uniforms of round t+2 are staged speculatively before round t runs;
    when the loop stops, the generator is rolled back to its state before the
    first batch of a round that never ran, so it is consumed exactly as by
    the reference (numpy Generators; other generator objects run without the
    pipeline)."""

    def __init__(self, ctx, A, *, k, r, c, criterion="modes", use_graphs=True, comm=None,
                 row_offset=0, m_total=None, w=0, precision="fp64"):
        self.A = A
        # precision="mixed" (BASELINE config 4): the A-reading TN products of a
        # float32-stored A -- the sampled Gram and finalize's A^T U -- run on
        # the tcgen05 tensor cores in 3xTF32 (pod_gemm_tn_tf32x3); every other
        # product stays fp64 DMMA
        self.mixed = (precision == "mixed" and A.code == 1 and A.ld % 4 == 0
                      and A.m % 4 == 0 and A.t.is_cuda)
        self.n = A.ncols
        self.c = int(c)
        gcap = min(self.c, A.ncols)
        # beyond the hand-written eigensolver's order the library one runs
        # (Ctx.gram_eigh_any): it synchronises, so such runs are eager and
        # unpipelined (the reference's default budget for k >= 28)
        self.big_gram = gcap > int(_lib.load().pod_gram_eigh_max_g())
        if self.big_gram:
            use_graphs = False
        super().__init__(ctx, A.m, r, k=k, criterion=criterion, upd_cap=gcap, comm=comm,
                         row_offset=row_offset, nupd=NSLOT)
        self.m_total = A.m if m_total is None else int(m_total)
        dev = ctx.device
        f64 = dict(dtype=torch.float64, device=dev)
        n, r, g = self.n, self.r, gcap
        self.gcap = g
        self.norms2 = torch.empty(n, **f64)
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)
        self.live = torch.ones(n, dtype=torch.uint8, device=dev)
        self.uni = [torch.empty(self.c, **f64) for _ in range(NSLOT)]
        self.h_uni = [torch.empty(self.c, dtype=torch.float64).pin_memory() for _ in range(NSLOT)]
        self.idx = [torch.empty(g, dtype=torch.int32, device=dev) for _ in range(NSLOT)]
        self.cnt = [torch.empty(g, dtype=torch.int64, device=dev) for _ in range(NSLOT)]
        self.G = [torch.empty(g * g, **f64) for _ in range(NSLOT)]
        self.Tl = [torch.empty(g * r, **f64) for _ in range(NSLOT)]
        self.npos = 0
        self.use_graphs = use_graphs
        self.graphs = {}
        self.graph_launches = {}
        self.graph_epoch = -1
        self.side = torch.cuda.Stream(dev)
        self.merge_cap = merge_grid_cap(dev)
        self.ort = None  # (C = U^T A, residual norms) buffers of the "ort" strategy
        self.frob2 = 0.0
        # host-resident A (page-locked, mapped): the norm pass, ort's U^T A and
        # finalize's A^T U stream it over PCIe; each round copies its sampled
        # columns into an HBM block D (multi-pass streamed ISMA)
        self.host_A = not A.t.is_cuda
        self.draw_log = None
        self._hbuf = None
        self.D = [ColMat.zeros(A.m, g, dev, dtype=A.t.dtype) for _ in range(len(self.Uupd_b))] \
            if self.host_A else None
        # row sampling (ICRS, isma.py:168-176): w row draws per round over the m rows
        self.w = int(w)
        if self.w:
            if self.comm.active:
                raise NotImplementedError("row sampling is not row-sharded")
            m = self.m
            self.hcap = min(self.w, m)
            self.rowq = torch.empty(m, **f64)
            self.uniw = [torch.empty(self.w, **f64) for _ in range(2)]
            self.h_uniw = [torch.empty(self.w, dtype=torch.float64).pin_memory()
                           for _ in range(2)]
            self.ridx = [torch.empty(self.hcap, dtype=torch.int32, device=dev) for _ in range(2)]
            self.rcnt = [torch.empty(self.hcap, dtype=torch.int64, device=dev) for _ in range(2)]
            self.rp = [torch.empty(self.hcap, **f64) for _ in range(2)]
            self.Y = [ColMat.zeros(self.hcap, g, dev) for _ in range(2)]
            self.levdiv = torch.ones(1, **f64)
            self.h_levdiv = torch.ones(1, dtype=torch.float64).pin_memory()

    def reset(self):
        """Per-run state (the captured graphs and buffers are reused)."""
        self.live.fill_(1)
        self.cur = 0
        self.l = 0
        self.npos = 0
        self.stats = {"rounds": 0}

    # ------------------------------------------------------------ pieces --
    def norm_pass(self):
        """Fused validate + column norms (matcore.py:54, isma.py:260)."""
        self.clear_breakdown()
        comm = self.comm
        if comm.active:
            # chained einsum-order pass over the row shards (parallel.py)
            st_in = st_out = None
            if comm.rank > 0:
                st_in = comm.recv(torch.empty(2 * self.n, dtype=torch.float64,
                                              device=self.ctx.device), comm.rank - 1)
            last = comm.rank == comm.world - 1
            if not last:
                st_out = torch.empty(2 * self.n, dtype=torch.float64, device=self.ctx.device)
            self.nonfinite.zero_()
            self.ctx.colnorms2_chain(self.A, st_in, st_out, last, self.norms2, self.nonfinite)
            if not last:
                comm.send(st_out, comm.rank + 1)
            comm.broadcast_(self.norms2, comm.world - 1)
        else:
            self.ctx.colnorms2(self.A, self.norms2, self.nonfinite)
        self.comm.allreduce_max_(self.nonfinite)
        flag = int(self.nonfinite.item())
        if flag:
            raise ParameterError("matrix contains non-finite entries")
        self.npos = int((self.norms2 > 0).sum().item())
        self.frob2 = float(self.norms2.double().sum().item())  # ||A||_F^2 (sampling.py:182)
        if self.npos == 0:
            raise DegenerateDistributionError("all candidate column weights are zero")

    def ort_weights_ops(self, cur):
        """residual_distribution (sampling.py:158-187) against the current
        basis: C = U^T A (TN) and ||a_j - U c_j||^2 (fused DMMA pass)."""
        ctx, A, r, n = self.ctx, self.A, self.r, self.n
        if self.ort is None:
            dev = ctx.device
            self.ort = (torch.zeros(r * n, dtype=torch.float64, device=dev),
                        torch.zeros(n, dtype=torch.float64, device=dev))
        C, res2 = self.ort
        U = self.S[cur].cols(0, r)
        if self.host_A:  # one PCIe pass: DMA column chunks, both products per chunk
            def chunk(Ach, j0, j1):
                ctx.tn(r, j1 - j0, 1.0, U, Ach, dptr(C, j0 * r), r, tag="tn_ort_UtA")
                ctx.resid_colnorms2(Ach, j1 - j0, U, r, dptr(C, j0 * r), r, res2[j0:j1])
            self._stream_columns(chunk)
            return res2
        ctx.tn(r, n, 1.0, U, A, dptr(C), r, tag="tn_ort_UtA")
        self.comm.allreduce_sum_(C)
        ctx.resid_colnorms2(A, n, U, r, dptr(C), r, res2)
        self.comm.allreduce_sum_(res2)
        return res2

    def _stream_columns(self, fn):
        """Host-resident A: column chunks (~1 GB) DMA-copied into two HBM
        buffers on a copy stream, each consumed by fn(chunk, j0, j1) on the
        current stream while the next one is in flight -- one PCIe pass with
        copy engines instead of kernel reads that a tiled product would
        repeat per output tile."""
        A, ctx = self.A, self.ctx
        dev = ctx.device
        m, n, es = A.m, self.n, A.esize
        per = max(1, min(n, (1 << 30) // (m * es)))
        if self._hbuf is None or self._hbuf[0].ncols < per:
            self._hbuf = [ColMat.zeros(m, per, dev, dtype=A.t.dtype) for _ in range(2)]
            self._copy_stream = torch.cuda.Stream(dev)
            self._ev_ready = [torch.cuda.Event() for _ in range(2)]
            self._ev_free = [torch.cuda.Event() for _ in range(2)]
        main = torch.cuda.current_stream(dev)
        cs = self._copy_stream
        cs.wait_stream(main)
        for i, j0 in enumerate(range(0, n, per)):
            j1 = min(n, j0 + per)
            b = i % 2
            buf = self._hbuf[b]
            if i >= 2:
                cs.wait_event(self._ev_free[b])  # chunk i - 2 consumed this buffer
            with torch.cuda.stream(cs):
                buf.t[:j1 - j0, :m].copy_(A.t[j0:j1, :m], non_blocking=True)
                self._ev_ready[b].record(cs)
            main.wait_event(self._ev_ready[b])
            fn(ColMat(buf.t, m, j1 - j0), j0, j1)
            self._ev_free[b].record(main)

    def update_ops(self, mode, b, dest, cur=None, rowsrc=None):
        """get_update (isma.py:144-178) at capacity into update slot b (its
        own draw/Gram/eigensolver scratch).  rowsrc None: column path (Gram
        of the gathered columns D).  rowsrc "norms"/"lev": ICRS -- w rows
        drawn from D's squared row norms or from the leverage of the current
        top-k basis (stack `cur`), the dedup-scaled row block Y and Y^T Y."""
        self.draw_gram_ops(mode, b, cur=cur, rowsrc=rowsrc)
        self.eigh_lift_ops(b, dest)

    def draw_gram_ops(self, mode, b, cur=None, rowsrc=None):
        """First half of get_update: the draw (isma.py:158-164) and the
        sampled Gram (baselines.py:43) or, for ICRS, the row draw and Y^T Y."""
        ctx, A, g = self.ctx, self.A, self.gcap
        self.uni[b].copy_(self.h_uni[b], non_blocking=True)
        weights, thr = None, 0.0
        if mode == MODE_L2N:
            weights = self.norms2
        elif mode == MODE_ORT:
            weights = self.ort_weights_ops(cur)
            thr = ORT_DEGENERATE_RTOL * self.frob2
        ctx.draw(mode, weights, self.live, self.n, self.uni[b], self.c, self.idx[b], self.cnt[b],
                 info=self.rec[1 + b, REC_G:], thr=thr)
        # the sampled block D: gathered inside the GEMM loaders from A in HBM,
        # or -- A host-resident -- copied once over PCIe into HBM (isma.py:163)
        if self.host_A:
            ctx.gather_cols(A, self.idx[b], g, self.D[b])
            src, cols = self.D[b], None
        else:
            src, cols = A, self.idx[b]
        if rowsrc is None:
            if self.mixed and TC_GRAM:                                       # tensor cores
                ctx.tn_tf32x3(g, g, 1.0, src, src, dptr(self.G[b]), g, xcols=cols, ycols=cols,
                              tag="tc_gram_gather")
            else:
                ctx.tn(g, g, 1.0, src, src, dptr(self.G[b]), g, xcols=cols, ycols=cols,
                       tag="tn_gram_gather")                                 # baselines.py:43
            self.comm.allreduce_sum_(self.G[b])
            return
        self.uniw[b].copy_(self.h_uniw[b], non_blocking=True)
        if rowsrc == "lev":                                                  # sampling.py:190-201
            self.levdiv.copy_(self.h_levdiv, non_blocking=True)
            ctx.rownorms2(self.S[cur], self.k, self.rowq, div_dev=self.levdiv)
        else:                                                                # sampling.py:143-147
            ctx.rownorms2(src, g, self.rowq, cols=cols)
        hinfo = self.rec[1 + b, REC_H:]
        ctx.draw(MODE_ROWS, self.rowq, None, self.m, self.uniw[b], self.w, self.ridx[b],
                 self.rcnt[b], info=hinfo, p_out=self.rp[b])
        ctx.gather_scale_rows(src, cols, g, self.ridx[b], self.rcnt[b], self.rp[b],
                              self.w, self.hcap, hinfo, self.Y[b])          # sampling.py:248-258
        ctx.tn(g, g, 1.0, self.Y[b], self.Y[b], dptr(self.G[b]), g, tag="tn_gram_rows")

    def eigh_lift_ops(self, b, dest):
        """Second half of get_update: eigensolve of slot b's Gram
        (baselines.py:44-48) and the lift through D (baselines.py:62-63)."""
        self.eigh_ops(b)
        self.lift_ops(b, dest)

    def eigh_ops(self, b):
        g, r = self.gcap, self.r
        self.ctx.gram_eigh_any(self.G[b], g, r, self.sig_upd_b[b], self.Tl[b],
                               self.rec[1 + b, REC_RANK:])                   # baselines.py:44-48

    def lift_ops(self, b, dest):
        g, r = self.gcap, self.r
        src, cols = (self.D[b], None) if self.host_A else (self.A, self.idx[b])
        self.ctx.nn(g, r, 1.0, src, dptr(self.Tl[b]), g, dest, xcols=cols,
                    tag="nn_lift_gather")                                    # baselines.py:62-63

    def side_ops(self, fn, join=True):
        """fn() on the side stream with its own workspaces (forked from the
        current stream; joined back when `join`)."""
        main = torch.cuda.current_stream(self.ctx.device)
        self.side.wait_stream(main)
        self.ctx.ws_suffix = "_upd"
        lib = _lib.load()
        lib.pod_set_grid_cap(UPDATE_GRID_CAP)  # leave SMs to the concurrent merge
        try:
            with torch.cuda.stream(self.side):
                fn()
        finally:
            lib.pod_set_grid_cap(0)
            self.ctx.ws_suffix = ""
        if join:
            main.wait_stream(self.side)

    def round_ops(self, mode, cur, ub, pipelined, rowsrc=None):
        """Round t: merge(t) with update slot ub (+ cosines, readback).
        pipelined: the side stream, forked at the start of the round, runs
        the eigensolve of update(t+1) (a few SMs, beside the merge's GEMM
        phase); once that GEMM phase is done it lifts update(t+1) and draws
        and forms the Gram of update(t+2) -- GEMMs that then share the GPU
        with the merge's latency-bound E-SVD instead of its GEMMs.  The update
        chain thus has a whole round to run in, and only the merge chain is
        on the critical path."""
        if pipelined:
            u1, u2 = (ub + 1) % NSLOT, (ub + 2) % NSLOT
            self.side_ops(lambda: self.eigh_ops(u1), join=False)
            lib = _lib.load()
            lib.pod_set_grid_cap(self.merge_cap)

            def before_core():
                lib.pod_set_grid_cap(0)
                self.side_ops(lambda: (self.lift_ops(u1, self.Uupd_b[u1].cols(0, self.r)),
                                       self.draw_gram_ops(mode, u2)), join=False)

            fc = self.fused_cosines()
            try:
                self.merge_ops(cur, ub, before_core=before_core,
                               cos_out=self.xi if fc else None)
            finally:
                lib.pod_set_grid_cap(0)
            self.cosines_ops(cur, 1 - cur, fused=fc)
            torch.cuda.current_stream(self.ctx.device).wait_stream(self.side)
            self.readback()
            return
        self.update_ops(mode, ub, self.Uupd_b[ub].cols(0, self.r), cur=cur, rowsrc=rowsrc)
        fc = self.fused_cosines()
        self.merge_ops(cur, ub, cos_out=self.xi if fc else None)
        self.cosines_ops(cur, 1 - cur, fused=fc)
        self.readback()

    def sharded_graphs(self):
        """Row-sharded rounds replay as CUDA graphs when the collectives are
        NCCL's (stream-ordered, capturable: every rank captures the same
        launch sequence); gloo's host-mediated collectives cannot be captured
        and run eagerly.  POD_SHARDED_GRAPHS=0 disables."""
        return SHARDED_GRAPHS and self.comm.backend == "nccl"

    def launch_round(self, mode, cur, ub, pipelined, rowsrc=None):
        if (not self.use_graphs or self.ctx.prof is not None
                or (self.comm.active and not self.sharded_graphs())):
            self.round_ops(mode, cur, ub, pipelined, rowsrc)
            return
        # graphs bake the matrix pointer into their launches: one set per A buffer
        key = (self.A.ptr.value, self.A.code, mode, cur, ub, pipelined, rowsrc)
        if self.graphs and (self.graph_epoch != self.ctx.ws_epoch or len(self.graphs) > 64):
            self.graphs.clear()  # a workspace was reallocated since these were captured
        gr = self.graphs.get(key)
        if gr is None:
            dev = self.ctx.device
            # eager warm-up (grows every workspace) on a side stream, state restored
            keep = (self.live, self.rec, self.S[0].t, self.S[1].t, self.sig[0], self.sig[1],
                    *(u.t for u in self.Uupd_b), *self.sig_upd_b, *self.G, *self.Tl, *self.idx,
                    *self.cnt)
            saved = [t.clone() for t in keep]
            st = torch.cuda.Stream(dev)
            st.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(st):
                self.round_ops(mode, cur, ub, pipelined, rowsrc)
            torch.cuda.current_stream(dev).wait_stream(st)
            torch.cuda.synchronize(dev)
            for dst, src in zip(keep, saved):
                dst.copy_(src)
            torch.cuda.synchronize(dev)
            if self.graph_epoch != self.ctx.ws_epoch:
                self.graphs.clear()  # the warm-up grew a workspace other graphs captured
            gr = torch.cuda.CUDAGraph()
            l0 = self.ctx.launches
            # thread_local: the OOC read-ahead thread may touch CUDA (pinned
            # allocation, H2D copies) while a round is being captured
            with torch.cuda.graph(gr, stream=st, capture_error_mode="thread_local"):
                self.round_ops(mode, cur, ub, pipelined, rowsrc)
            self.graph_launches[key] = self.ctx.launches - l0
            self.graphs[key] = gr
            self.graph_epoch = self.ctx.ws_epoch
            torch.cuda.synchronize(dev)
        gr.replay()
        self.ctx.launches += self.graph_launches[key]

    def finalize(self):
        """isma.py:295-301: Q, R = QR(A^T U); SVD(R); U V_R, Q U_R; signs."""
        ctx, r, n = self.ctx, self.r, self.n
        dev = ctx.device
        U = self.S[self.cur].cols(0, r)
        Cm = ColMat.zeros(n, r, dev)
        if self.host_A:                                                      # A^T U, streamed
            self._stream_columns(lambda Ach, j0, j1: ctx.tn(
                j1 - j0, r, 1.0, Ach, U, dptr(Cm.t[0], j0), n, tag="tn_finalize_AtU"))
        elif self.mixed:                                    # A^T U on the tensor cores
            m = U.m
            hi = torch.empty(m * r, dtype=torch.float32, device=dev)
            lo = torch.empty(m * r, dtype=torch.float32, device=dev)
            ctx.split_tf32(U, r, hi, lo)
            ctx.tn_tf32x3(n, r, 1.0, self.A, ColMat(hi.view(r, m), m, r), Cm.ptr, n, Ylo=lo,
                          tag="tc_finalize_AtU")
            del hi, lo
        else:
            ctx.tn(n, r, 1.0, self.A, U, Cm.ptr, n, tag="tn_finalize_AtU")  # A^T U
        self.comm.allreduce_sum_(Cm.t)
        Qc = ColMat.zeros(n, r, dev)
        Rc = torch.zeros(r * r, dtype=torch.float64, device=dev)
        self.cholqr_ops(Cm, Qc, r, Rc, G_FQR, sharded=False)  # A^T U is replicated
        Ur = torch.zeros(r * r, dtype=torch.float64, device=dev)
        Vr = torch.zeros(r * r, dtype=torch.float64, device=dev)
        sr = torch.zeros(r, dtype=torch.float64, device=dev)
        ctx.svd_small(dptr(Rc), r, r, r, dptr(Ur), r, sr, dptr(Vr), r)       # _svd(rr)
        nxt = 1 - self.cur
        Unew = self.S[nxt].cols(0, r)
        ctx.nn(r, r, 1.0, U, dptr(Vr), r, Unew, tag="nn_finalize_rot")      # u @ vrt.T
        Vnew = ColMat.zeros(n, r, dev)
        ctx.nn(r, r, 1.0, Qc, dptr(Ur), r, Vnew, tag="nn_finalize_rot")     # q @ ur
        self.fix_signs_ops(Unew, r, Vnew, n)
        self.sig[nxt].copy_(sr)
        self.cur = nxt
        return Vnew

    # ------------------------------------------------------------ driver ---
    def _stage_uniforms(self, rng, b, rows=False):
        """One rng.random(c) batch for the column draw (sampling.py:213); with
        rows, then one rng.random(w) batch for the row draw (isma.py:173)."""
        u = np.asarray(rng.random(int(self.c)), dtype=np.float64)
        if u.shape != (self.c,):
            raise ParameterError("generator returned a batch of the wrong shape")
        self.h_uni[b].numpy()[:] = u
        if rows:
            # the reference raises on a zero row distribution AFTER the column
            # batch and BEFORE the row batch (isma.py:162-173, sampling.py:62-64)
            bg = getattr(rng, "bit_generator", None)
            self._state_before_rows = bg.state if bg is not None else None
            u = np.asarray(rng.random(int(self.w)), dtype=np.float64)
            if u.shape != (self.w,):
                raise ParameterError("generator returned a batch of the wrong shape")
            self.h_uniw[b].numpy()[:] = u

    def _log_draw(self, b, rec):
        """RECORD_DRAWS: the index set and counts drawn into slot b this round."""
        if self.draw_log is None:
            return
        g = rec[REC_G]
        entry = (self.idx[b][:g].cpu().numpy().astype(np.int64),
                 self.cnt[b][:g].cpu().numpy().astype(np.int64))
        if self.w:  # ICRS: the round's row draw too (isma.py:168-173)
            h = rec[REC_H]
            entry += (self.ridx[b][:h].cpu().numpy().astype(np.int64),
                      self.rcnt[b][:h].cpu().numpy().astype(np.int64))
        self.draw_log.append(entry)

    def _check_rows(self, rec, rng, state):
        """A zero row distribution raises (sampling.py:62-64) after the column
        batch and before the row batch is drawn in the reference: put the
        generator back between the two batches, then raise."""
        if rec[REC_HSTATUS] == 2:
            mid = getattr(self, "_state_before_rows", None)
            if state is not None and mid is not None:
                rng.bit_generator.state = mid
            raise DegenerateDistributionError("all row weights are zero")

    def _orthonormalize_ops(self, cur, l):
        """isma.py:267-269 / orthonormalize (isma.py:244-254): Q0 R = U
        (CholeskyQR into the stack's Q half), U_R = SVD(R), U <- fix_signs(Q0
        U_R); sigma is kept."""
        ctx, r = self.ctx, self.r
        S = self.S[cur]
        U, Q0 = S.cols(0, l), S.cols(r, r + l)
        self.cholqr_ops(U, Q0, l, self.Rt, G_QR)
        ctx.svd_small(dptr(self.Rt), r, l, l, dptr(self.Rt2), r, self.sig_upd_b[1][:l], None, 1)
        ctx.nn(l, l, 1.0, Q0, dptr(self.Rt2), r, U, tag="nn_orthonormalize")
        self.fix_signs_ops(U, l)

    def run(self, rng, *, strategy, tau, finalize, keep, trace_cls):
        """isma_run main loop (isma.py:258-303) on the device."""
        self.norm_pass()
        traces = []
        t0 = time.perf_counter()
        cur = self.cur
        r = self.r
        # the pipeline stages uniforms two rounds ahead; only generators whose
        # state can be rolled back support that
        bitgen = getattr(rng, "bit_generator", None)
        mode = {"l2n": MODE_L2N, "ort": MODE_ORT}.get(strategy, MODE_UNIFORM)
        rows = self.w > 0
        # ort's distribution depends on the merged basis, and so does the
        # leverage-driven row draw: no pipelining for either (nor for ICRS).
        # Row-sharded runs pipeline too: every rank issues its collectives in
        # the same program order (update Gram after the merge's GEMM-phase
        # reductions), which the backend serialises on its own stream.
        pipelined = bitgen is not None and mode != MODE_ORT and not rows and not self.big_gram
        state = bitgen.state if (rows and bitgen is not None) else None
        self._stage_uniforms(rng, 0, rows)
        # generator state before each speculatively staged batch (round -> state)
        spec = {}
        ran = 0  # rounds launched
        if pipelined:
            # rounds 1 and 2 are staged speculatively so that update(1) and the
            # draw + Gram of update(2) run on the side stream beside the
            # bootstrap's eigensolve (they only need draw(0)'s candidate set)
            spec[1] = bitgen.state
            self._stage_uniforms(rng, 1)                                     # round 1
            spec[2] = bitgen.state
            self._stage_uniforms(rng, 2)                                     # round 2
            self.draw_gram_ops(MODE_L2N, 0)                                  # bootstrap draw + Gram
            self.side_ops(lambda: (self.update_ops(mode, 1, self.Uupd_b[1].cols(0, r)),
                                   self.draw_gram_ops(mode, 2)), join=False)
            self.eigh_lift_ops(0, self.S[cur].cols(0, r))                    # bootstrap eigh + lift
        else:
            self.update_ops(MODE_L2N, 0, self.S[cur].cols(0, r),             # bootstrap
                            rowsrc="norms" if rows else None)
        self.sig[cur].copy_(self.sig_upd_b[0][:r])
        self.readback()
        rec, _ = self.read_record(0)
        self.draw_log = [] if RECORD_DRAWS else None
        self._log_draw(0, rec)
        if pipelined:
            torch.cuda.current_stream(self.ctx.device).wait_stream(self.side)
        if rows:
            self._check_rows(rec, rng, state)
        g, rem, keep0, h = rec[REC_G], rec[REC_REM], rec[REC_KEEP_UPD], rec[REC_H]
        self.npos -= g
        self.sig[cur][keep0:].zero_()  # the basis carries keep0 modes; zero sigma padding
        self.l = keep0
        if rows and keep0:
            self._orthonormalize_ops(cur, keep0)                             # isma.py:267-269
        traces.append(trace_cls(0, g, h if rows else 0, rem, np.zeros(0),
                                time.perf_counter() - t0))
        xi = np.zeros(self.k)
        it = 0
        ub = 1
        if pipelined:
            # round t's graph draws update(t + 2) from uniform slot (t + 2) % 3.
            # Its batch is staged while round t - 1 still runs (right after
            # that round's launch, below), so between two rounds the host only
            # reads the record and launches; the slot's last reader, round
            # t - 3, has completed by then.  Round 1's batch goes in now (the
            # bootstrap's record read synchronized the device).
            spec[3] = bitgen.state
            self._stage_uniforms(rng, 0)                                     # round 3
        while rem and (it == 0 or bool(np.any(xi < tau))):
            it += 1
            t0 = time.perf_counter()
            if mode == MODE_L2N and self.npos <= 0:
                break  # l2n over only zero-norm columns (isma.py:211-215, 280-281)
            rowsrc = None
            if pipelined:
                ub = it % NSLOT
            else:
                if rows:
                    state = bitgen.state if bitgen is not None else None
                    rowsrc = "lev" if (strategy == "ls" and self.l) else "norms"  # isma.py:283-284
                    self.h_levdiv[0] = float(min(self.k, self.l))
                self._stage_uniforms(rng, ub, rows)
            self.launch_round(mode, cur, ub, pipelined, rowsrc)
            ran = it
            if pipelined:  # the next round's batch, while this round runs
                spec[it + 3] = bitgen.state
                self._stage_uniforms(rng, (it + 3) % NSLOT)                  # round it + 3
            rec, xi = self.read_record(ub)
            self._log_draw(ub, rec)
            if rows:
                self._check_rows(rec, rng, state)
            g, rem = rec[REC_G], rec[REC_REM]
            if mode == MODE_L2N:
                self.npos -= g
            cur = 1 - cur
            self.l = rec[REC_KEEP]
            self.stats["rounds"] += 1
            self.stats.setdefault("eigh_sweeps", []).append(rec[REC_EIGH_SWEEPS])
            self.stats.setdefault("merge_sweeps", []).append(rec[REC_MERGE_SWEEPS])
            traces.append(trace_cls(it, g, rec[REC_H] if rows else 0, rem, xi.copy(),
                                    time.perf_counter() - t0))
        if pipelined and spec:
            # undo the speculative batches of the rounds never run
            first = min((u for u in spec if u > ran), default=None)
            if first is not None:
                bitgen.state = spec[first]
        self.cur = cur
        v = None
        if finalize and self.l:
            v = self.finalize()
        elif self.l:
            self.fix_signs_ops(self.S[self.cur].cols(0, self.l), self.l)
        return traces, v

    def result(self, keep, v=None):
        if float(self.ctx.dinfo[DINFO_BREAKDOWN].item()) != 0.0:  # finalize's CholeskyQR
            self.clear_breakdown()
            raise np.linalg.LinAlgError("CholeskyQR breakdown in finalize (QR of A^T U)")
        l = min(self.l, keep)
        u = self.gather_rows(self.S[self.cur], l, self.m_total) if l else np.zeros((self.m_total, 0))
        s = self.sig[self.cur][:l].cpu().numpy().copy()
        vv = None if v is None else (v.to_numpy(l) if l else np.zeros((self.n, 0)))
        return u, s, vv


def eng_input_is_staged(A):
    from .device import _STAGING

    return any(A.t is b.t for b in _STAGING.values())


_ENGINE_CACHE = {}
ENGINE_CACHE_SIZE = 2  # per device: e.g. the two block widths of a column-block stream


def get_engine(ctx, A, *, k, r, c, criterion, use_graphs, comm=None, row_offset=0, m_total=None,
               w=0, precision="fp64"):
    """Reuse an engine (buffers + captured round graphs) of an earlier run
    when the matrix shape and configuration match (LRU, two per device).
    The graphs are kept per matrix buffer (they bake its pointer in) and read
    A and the staged uniforms at replay time, so a reused engine is valid for
    new contents of a buffer it has seen."""
    world = 1 if comm is None else comm.world
    key = (A.m, A.ncols, A.ld, A.code, A.t.is_cuda, int(k), int(r), int(c), criterion,
           bool(use_graphs),
           ctx.device.index, world, bool(comm is not None and comm.active), int(row_offset),
           m_total, int(w), precision)
    lru = _ENGINE_CACHE.setdefault(ctx.device.index, [])
    for i, eng in enumerate(lru):
        if eng.key == key:
            lru.append(lru.pop(i))  # most recently used last
            eng.A = A
            eng.reset()
            return eng
    while len(lru) >= ENGINE_CACHE_SIZE:
        lru.pop(0)
    try:
        eng = IsmaEngine(ctx, A, k=k, r=r, c=c, criterion=criterion, use_graphs=use_graphs,
                         comm=comm, row_offset=row_offset, m_total=m_total, w=w,
                         precision=precision)
    except torch.OutOfMemoryError:
        lru.clear()  # cached engines hold their buffers: drop them and retry once
        from .device import release_staging

        if eng_input_is_staged(A):
            pass  # the run's own matrix lives in the staging buffer: keep it
        else:
            release_staging()
        torch.cuda.empty_cache()
        eng = IsmaEngine(ctx, A, k=k, r=r, c=c, criterion=criterion, use_graphs=use_graphs,
                         comm=comm, row_offset=row_offset, m_total=m_total, w=w,
                         precision=precision)
    eng.key = key
    lru.append(eng)
    return eng
