"""World-size-2 gloo tests (CPU) of the row-sharded collective protocol
(parallel.py): partial reductions over row shards, the global sign
convention, and the row gather."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import isma_oracle as orc
from paper_1905_05107_b200.parallel import Comm, combine_signs, gather_row_shards, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(Comm())))
    finally:
        dist.destroy_process_group()


def run_world(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [out[r] for r in range(world)]


def test_shard_rows_partition():
    for m in (1, 7, 100, 262144):
        for w in (1, 2, 3, 8):
            bounds = [shard_rows(m, w, r) for r in range(w)]
            assert bounds[0][0] == 0 and bounds[-1][1] == m
            assert all(b[1] == c[0] for b, c in zip(bounds, bounds[1:]))


def _gram_and_signs(comm):
    rng = np.random.default_rng(0)
    a = rng.standard_normal((101, 7))
    a[40, 3] = -9.0  # global max of column 3 on rank 0's shard (negative)
    a[77, 3] = 9.0   # tie on rank 1's shard: the lower row (40) must win
    r0, r1 = shard_rows(101, comm.world, comm.rank)
    loc = torch.as_tensor(a[r0:r1])
    g = loc.T @ loc
    comm.allreduce_sum_(g)
    absl = loc.abs()
    val, arg = absl.max(0)
    # first occurrence on ties inside the shard
    arg = torch.tensor([int(np.argmax(absl[:, j].numpy())) for j in range(7)])
    sign = torch.where(loc[arg, torch.arange(7)] < 0, -1.0, 1.0).double()
    s = combine_signs(comm.allgather(val.double()), comm.allgather(arg + r0), comm.allgather(sign))
    full = gather_row_shards(loc.T.contiguous(), 101, comm)
    return g.numpy(), s.numpy(), full


def test_partial_grams_signs_and_gather_over_two_ranks():
    res = run_world(_gram_and_signs, 2)
    rng = np.random.default_rng(0)
    a = rng.standard_normal((101, 7))
    a[40, 3] = -9.0
    a[77, 3] = 9.0
    _, flip = orc.canon_signs(a, np.eye(7))
    want = np.where(np.diag(flip) < 0, -1.0, 1.0)
    for g, s, full in res:
        np.testing.assert_allclose(g, a.T @ a, rtol=1e-13)
        np.testing.assert_array_equal(s, want)
        np.testing.assert_array_equal(full, a)
    # every rank holds bitwise identical reductions (identical decisions)
    assert np.array_equal(res[0][0], res[1][0])


def test_config2_generator_is_shard_invariant():
    from paper_1905_05107_b200 import workloads

    full = workloads.config2_torch(3, side=96, n=25)
    m = 96 * 96
    for world in (2, 3):
        parts = [workloads.config2_torch(3, side=96, n=25, rows=shard_rows(m, world, r))
                 for r in range(world)]
        assert torch.equal(full, torch.cat(parts, 1))


def _chained_norms(comm):
    """The engine's sharded norm protocol (engine.IsmaEngine.norm_pass): rank p
    continues numpy's einsum lane state from rank p - 1 (recv), hands it on
    (send), the last rank's norms are broadcast -- here with the oracle's
    restatement of the lane order standing in for pod_colnorms2_chain."""
    rng = np.random.default_rng(3)
    m, n = 1003, 9
    a = np.asfortranarray(rng.standard_normal((m, n)))
    r0, r1 = shard_rows(m, comm.world, comm.rank)
    seg = a[r0:r1]
    st = None
    if comm.rank > 0:
        st = comm.recv(torch.empty(2 * n, dtype=torch.float64), comm.rank - 1).numpy().reshape(2, n)
    last = comm.rank == comm.world - 1
    body = seg.shape[0] - (seg.shape[0] % 8 if last else 0)
    st = orc.einsum_lane_state(seg[:body], st)
    norms = torch.zeros(n, dtype=torch.float64)
    if last:
        norms = torch.as_tensor(orc.einsum_lane_finish(seg[body:], st))
    else:
        comm.send(torch.as_tensor(st.reshape(-1).copy()), comm.rank + 1)
    comm.broadcast_(norms, comm.world - 1)
    return norms.numpy(), np.einsum("ij,ij->j", a, a)


@pytest.mark.parametrize("world", [2, 3])
def test_chained_norm_pass_over_ranks_equals_numpy(world):
    for got, ref in run_world(_chained_norms, world=world):
        assert np.array_equal(got, ref)


def _forced_single_rank(comm):
    """Comm(force=True) on a one-rank group: the sharded path's collectives
    are issued (identity results) instead of short-circuited."""
    forced = Comm(force=True)
    t = torch.arange(6, dtype=torch.float64)
    out = {
        "plain_active": comm.active,
        "forced_active": forced.active,
        "backend": forced.backend,
        "sum": forced.allreduce_sum_(t.clone()).tolist(),
        "max": forced.allreduce_max_(t.clone()).tolist(),
        "bcast": forced.broadcast_(t.clone(), 0).tolist(),
        "gather_shape": list(forced.allgather(t).shape),
    }
    rows = gather_row_shards(torch.arange(12, dtype=torch.float64).reshape(3, 4), 4, forced)
    out["rows"] = rows.tolist()
    return out


def test_forced_single_rank_group_issues_collectives():
    res = run_world(_forced_single_rank, world=1)[0]
    assert res["plain_active"] is False and res["forced_active"] is True
    assert res["backend"] == "gloo"
    assert res["sum"] == res["max"] == res["bcast"] == [0.0, 1.0, 2.0, 3.0, 4.0, 5.0]
    assert res["gather_shape"] == [1, 6]
    assert res["rows"] == np.arange(12.0).reshape(3, 4).T.tolist()


def test_comm_without_process_group_is_inactive_even_when_forced():
    c = Comm(force=True)
    assert not c.active and c.world == 1 and c.backend is None


def test_triangular_apply_chunks_cover_the_width():
    """engine.tri_apply_bounds: contiguous chunks from 0 to l; single call
    below 120 columns, [0, 80, l] to 160, 64-wide chunks beyond with no thin
    tail."""
    from paper_1905_05107_b200.engine import tri_apply_bounds

    for l in list(range(1, 300)) + [384, 512, 1000]:
        b = tri_apply_bounds(l)
        assert b[0] == 0 and b[-1] == l and all(x < y for x, y in zip(b[:-1], b[1:]))
        if l < 120:
            assert b == [0, l]
        elif l <= 160:
            assert b == [0, 80, l]
        else:
            assert all(y - x == 64 for x, y in zip(b[:-2], b[1:-1]))
            assert 32 <= b[-1] - b[-2] < 96
