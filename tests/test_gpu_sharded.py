"""Row-sharded isma_run on real kernels: two processes share the GPU and
exchange through gloo (host-mediated collectives; no kernel waits on another
rank), checked against the unsharded single-process run."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402
from parity_util import ANGLE_TOL_RAD, SIGMA_RTOL, principal_angles_sin, sigma_relerr  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, crit, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import paper_1905_05107_b200 as pod
    from paper_1905_05107_b200 import workloads
    from paper_1905_05107_b200.parallel import Comm, shard_rows

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = workloads.config1(seed=0)
        r0, r1 = shard_rows(a.shape[0], world, rank)
        cfg = pod.IsmaConfig(k=10, r=30, c=50, tau=0.999, strategy="l2n", criterion=crit, seed=7)
        f, tr = pod.isma_run(np.asfortranarray(a[r0:r1]), cfg, comm=Comm(), m_total=a.shape[0])
        q.put((rank, (f.u, f.sigma, f.v, [t.remaining for t in tr])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("crit", ["modes", "subspace"])
def test_two_rank_row_sharded_run_matches_single_gpu(crit):
    import paper_1905_05107_b200 as pod
    from paper_1905_05107_b200 import workloads

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, crit, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = workloads.config1(seed=0)
    cfg = pod.IsmaConfig(k=10, r=30, c=50, tau=0.999, strategy="l2n", criterion=crit, seed=7)
    f, tr = pod.isma_run(a, cfg)
    for rank in (0, 1):
        u, s, v, rem = res[rank]
        assert rem == [t.remaining for t in tr]
        assert sigma_relerr(s, f.sigma) <= SIGMA_RTOL
        assert principal_angles_sin(u, f.u).max() <= ANGLE_TOL_RAD
        assert principal_angles_sin(v, f.v).max() <= ANGLE_TOL_RAD
    np.testing.assert_array_equal(res[0][1], res[1][1])  # identical on every rank


def _host_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import paper_1905_05107_b200 as pod
    from paper_1905_05107_b200 import workloads
    from paper_1905_05107_b200.parallel import Comm, shard_rows

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = 60_000
        r0, r1 = shard_rows(m, world, rank)
        blk = workloads.config5_host(seed=3, m=m, n=900, rows=(r0, r1), device="cuda")
        cfg = pod.IsmaConfig(k=16, r=48, c=64, tau=1 - 1e-8, strategy="l2n", seed=5)
        f, tr = pod.isma_run(blk.T, cfg, comm=Comm(), m_total=m, residency="host")
        q.put((rank, (f.u, f.sigma, f.v, [t.remaining for t in tr])))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_resident_config5_matches_oracle():
    """Config 5's layout on two ranks: each rank's row block of the fp32
    matrix stays in its page-locked host memory (residency="host"), the norm
    pass is chained over the ranks, rounds gather sampled columns from host
    memory; identical bookkeeping and factors to the CPU oracle."""
    from oracle import isma_oracle as orc
    from paper_1905_05107_b200 import workloads

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_host_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = workloads.config5_host(seed=3, m=60_000, n=900, device="cuda").numpy().T
    o = orc.run(a.astype(np.float64), 16, r=48, c=64, tau=1 - 1e-8, strategy="l2n", seed=5)
    for rank in (0, 1):
        u, s, v, rem = res[rank]
        assert rem == [t["remaining"] for t in o["trace"]]
        assert sigma_relerr(s, o["sigma"]) <= SIGMA_RTOL
        assert principal_angles_sin(u, o["u"]).max() <= ANGLE_TOL_RAD
        assert principal_angles_sin(v, o["v"]).max() <= ANGLE_TOL_RAD


# ---- NCCL on the one GPU: a single-rank group on the sharded code path -----
_NCCL_SCRIPT = r"""
import os, sys
sys.path.insert(0, {root!r})
os.environ["MASTER_ADDR"] = "127.0.0.1"
os.environ["MASTER_PORT"] = {port!r}
import numpy as np, torch
import torch.distributed as dist
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import engine, workloads
from paper_1905_05107_b200.parallel import Comm

torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
try:
    comm = Comm(force=True)
    assert comm.active and comm.backend == "nccl"
    a = workloads.config1(seed=0)
    cfg = pod.IsmaConfig(k=10, r=30, c=50, tau=0.999, strategy="l2n", criterion={crit!r}, seed=7)
    f, tr = pod.isma_run(np.asfortranarray(a), cfg, comm=comm, m_total=a.shape[0])
    engs = [e for lru in engine._ENGINE_CACHE.values() for e in lru]
    graphs = sum(len(getattr(e, "graphs", ())) for e in engs)
    np.savez({out!r}, u=f.u, sigma=f.sigma, v=f.v, remaining=[t.remaining for t in tr],
             graphs=graphs, expect_graphs=int(engine.SHARDED_GRAPHS))
finally:
    dist.destroy_process_group()
"""


@pytest.mark.parametrize("crit", ["modes", "subspace"])
def test_single_rank_nccl_group_runs_sharded_path_with_captured_rounds(tmp_path, crit):
    """The row-sharded code path with its collectives carried by NCCL (a
    one-rank group, Comm(force=True)): norms chain + broadcast, every
    allreduce of the round (Gram, M, CholeskyQR Grams, leak, cosines) inside
    the captured round graphs, the fix_signs allgather and finalize's
    allreduce -- against the oracle, like the unsharded run."""
    import subprocess
    import sys

    from oracle import isma_oracle as orc
    from paper_1905_05107_b200 import workloads

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "nccl1.npz")
    subprocess.run([sys.executable, "-c",
                    _NCCL_SCRIPT.format(root=root, port=str(_port()), crit=crit, out=out)],
                   check=True, timeout=600)
    g = np.load(out)
    a = workloads.config1(seed=0)
    o = orc.run(a, 10, r=30, c=50, tau=0.999, strategy="l2n", criterion=crit, seed=7)
    assert list(g["remaining"]) == [t["remaining"] for t in o["trace"]]
    assert sigma_relerr(g["sigma"], o["sigma"]) <= SIGMA_RTOL
    assert principal_angles_sin(g["u"], o["u"]).max() <= ANGLE_TOL_RAD
    assert principal_angles_sin(g["v"], o["v"]).max() <= ANGLE_TOL_RAD
    if int(g["expect_graphs"]):
        assert int(g["graphs"]) > 0, "sharded NCCL rounds were not graph-captured"
