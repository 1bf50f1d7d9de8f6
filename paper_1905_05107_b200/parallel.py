"""Row-sharded data parallelism for the ISMA path.

A is partitioned by ROWS over the ranks of one node (contiguous, balanced
ranges); every m-length operand (sampled columns, U1, U2, Q, the merged U)
follows the same row partition, every r/g/n-sized object is replicated.
The reference algorithm exchanges data only through a few small reductions
per round, which become collectives here:

  norms           a chained pass: rank p continues numpy's einsum lane state
                  (2 n doubles) from rank p - 1 and hands it on (send/recv),
                  the last rank's norms are broadcast -- the sharded norms
                  equal the single-GPU and numpy ones bit for bit, so the
                  draws are the reference's on any rank count
  draw            recomputed on every rank from the identical reduced norms
                  and the identically seeded generator (no broadcast)
  Gram D^T D      allreduce(sum) g x g, then the eigensolver is replicated
  M = U1^T U2     allreduce(sum) r x r
  CholeskyQR      allreduce(sum) of every pass's r x r Gram
  leak U1^T Q     allreduce(sum) r x r (the leak gate is then identical)
  cosines         allreduce(sum) of the k raw dots (or k x k for subspace)
  fix_signs       allgather of (max |u|, global row, sign) per column and a
                  deterministic combination (largest |u|, lowest row on ties)
  finalize A^T U  allreduce(sum) n x r; the n x r QR and r x r SVD replicated

Collectives go through ``torch.distributed`` (NCCL over NVLink on the GPU
box, gloo in the CPU tests); every reduced buffer is bitwise identical on all
ranks, so all data-dependent decisions (index sets, gates, keep counts, the
tau test) agree across ranks by construction.
"""

from __future__ import annotations

import torch


#: inner shard boundaries are multiples of this (numpy's einsum works in
#: 8-row blocks, so a chained norm segment must start on a block boundary)
ROW_ALIGN = 8


def shard_rows(m, world, rank):
    """Contiguous balanced row range [r0, r1) of `rank` (like ooc.py:61-66),
    inner boundaries rounded down to a multiple of ROW_ALIGN."""
    def bound(k):
        if k >= world:
            return m
        return ((k * m) // world) // ROW_ALIGN * ROW_ALIGN
    return bound(rank), bound(rank + 1)


class Comm:
    """Collectives over the default process group (no-ops for one rank).

    force (or POD_COMM_FORCE=1): a single-rank group still takes the sharded
    code path and issues its collectives -- the way to drive the NCCL calls,
    and their capture into the round graphs, on a one-GPU box."""

    def __init__(self, group=None, force=None):
        import os

        import torch.distributed as dist

        self.dist = dist
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0
        if force is None:
            force = os.environ.get("POD_COMM_FORCE", "0") == "1"
        self.force = bool(force) and dist.is_available() and dist.is_initialized()

    @property
    def active(self):
        return self.world > 1 or self.force

    @property
    def backend(self):
        return self.dist.get_backend(self.group) if self.dist.is_initialized() else None

    def allreduce_sum_(self, t):
        if self.active:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def allreduce_max_(self, t):
        if self.active:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t

    def _host_p2p(self, t):
        # gloo's point-to-point ops take host tensors only (NCCL takes device ones)
        return t.is_cuda and self.dist.get_backend(self.group) == "gloo"

    def send(self, t, dst):
        self.dist.send(t.cpu() if self._host_p2p(t) else t, dst, group=self.group)

    def recv(self, t, src):
        if self._host_p2p(t):
            h = torch.empty(t.shape, dtype=t.dtype)
            self.dist.recv(h, src, group=self.group)
            t.copy_(h)
        else:
            self.dist.recv(t, src, group=self.group)
        return t

    def broadcast_(self, t, src):
        if self.active:
            self.dist.broadcast(t, src, group=self.group)
        return t

    def allgather(self, t):
        """Stack of every rank's tensor along a new leading axis."""
        if not self.active:
            return t.unsqueeze(0)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return torch.stack(out, 0)


def combine_signs(vals, rows, signs):
    """Global fix_signs decision from per-shard candidates.

    vals/rows/signs: (world, l) -- each shard's max |u| per column, its global
    row and the sign there.  Returns the (l,) sign vector of the entry with
    the largest |u|, the lowest global row winning ties (np.argmax's first
    occurrence, matcore.py:159-161).  Deterministic and identical on every
    rank.
    """
    world, l = vals.shape
    best = torch.full((l,), -1.0, dtype=vals.dtype, device=vals.device)
    brow = torch.full((l,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=vals.device)
    bsign = torch.ones((l,), dtype=signs.dtype, device=signs.device)
    for w in range(world):
        v, r, s = vals[w], rows[w], signs[w]
        take = (v > best) | ((v == best) & (r < brow))
        best = torch.where(take, v, best)
        brow = torch.where(take, r, brow)
        bsign = torch.where(take, s, bsign)
    return bsign


def gather_row_shards(local, m_total, comm):
    """Full (m_total, l) numpy array from each rank's (l, m_local) row block
    (rows follow ``shard_rows``); identical on every rank."""
    import numpy as np

    l, m_local = local.shape
    if not comm.active:
        if local.is_cuda:
            from .device import d2h_colmajor

            return d2h_colmajor(local)
        return np.asfortranarray(local.cpu().numpy().T)
    mmax = max(shard_rows(m_total, comm.world, w)[1] - shard_rows(m_total, comm.world, w)[0]
               for w in range(comm.world))
    pad = torch.zeros((l, mmax), dtype=local.dtype, device=local.device)
    pad[:, :m_local].copy_(local)
    parts = comm.allgather(pad).cpu().numpy()  # (world, l, mmax)
    out = np.empty((m_total, l), dtype=parts.dtype)
    for w in range(comm.world):
        r0, r1 = shard_rows(m_total, comm.world, w)
        out[r0:r1] = parts[w][:, :r1 - r0].T
    return np.asfortranarray(out)
