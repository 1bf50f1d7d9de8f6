"""Speculative merge core (engine.SPEC_CORE): the E-SVD of merge.py:80-85
starts on the first CholeskyQR's (M, R) while the leak check of
merge.py:72-73 runs beside it; a re-run gated on that check covers the
rounds whose second projection fires.

* pod_merge_core_gated with gate 1 == pod_merge_core bit for bit; gate 0
  touches nothing;
* ISMA runs give bit-identical factors with the core speculative and
  serial, in rounds where the leak check never fires and with it forced to
  fire every round (REORTH_TOL = 0).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1905_05107_b200 as pod  # noqa: E402
from paper_1905_05107_b200 import _lib, engine, workloads  # noqa: E402
from paper_1905_05107_b200.device import dptr, get_ctx  # noqa: E402


def _core_inputs(l, rng, dev):
    f = dict(dtype=torch.float64, device=dev)
    sig1 = torch.as_tensor(np.sort(rng.random(l) + 0.1)[::-1].copy(), **f)
    sig2 = torch.as_tensor(np.sort(rng.random(l) + 0.1)[::-1].copy(), **f)
    M = torch.as_tensor(rng.standard_normal(l * l) * 0.3, **f)
    R = np.triu(rng.standard_normal((l, l)) * 0.2 + np.eye(l))
    R = torch.as_tensor(np.asfortranarray(R).T.reshape(-1).copy(), **f)
    return sig1, M, R, sig2


@pytest.mark.parametrize("l", [16, 60, 150])
def test_gated_core_equals_core_and_gate0_is_noop(l):
    lib = _lib.load()
    assert lib.pod_merge_core_gatable(l, l) == 1
    ctx = get_ctx()
    dev = ctx.device
    rng = np.random.default_rng(l)
    sig1, M, R, sig2 = _core_inputs(l, rng, dev)
    outs = []
    for gate_val in (None, 1, 0):
        T = torch.full((2 * l * l,), 7.0, dtype=torch.float64, device=dev)
        sn = torch.full((l,), 7.0, dtype=torch.float64, device=dev)
        info = torch.full((4,), 7, dtype=torch.int64, device=dev)
        args = (dptr(sig1), l, dptr(M), l, dptr(R), l, dptr(sig2), l, l, l, dptr(T), 2 * l, l,
                dptr(sn))
        if gate_val is None:
            ctx.merge_core(*args, info=info)
        else:
            gate = torch.full((1,), gate_val, dtype=torch.int32, device=dev)
            ctx.merge_core_gated(*args, info, gate)
        torch.cuda.synchronize()
        outs.append((T.cpu().numpy(), sn.cpu().numpy(), info.cpu().numpy()))
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    assert (outs[2][0] == 7.0).all() and (outs[2][1] == 7.0).all() and (outs[2][2] == 7).all()
    assert outs[0][2][0] >= 1


def test_gatable_sizes():
    lib = _lib.load()
    assert lib.pod_merge_core_gatable(1, 1) == 1
    assert lib.pod_merge_core_gatable(0, 5) == 0
    assert lib.pod_merge_core_gatable(400, 400) == 0  # the grid solver: not gatable
    with pytest.raises(Exception):
        ctx = get_ctx()
        z = torch.zeros(8, dtype=torch.float64, device=ctx.device)
        g = torch.ones(1, dtype=torch.int32, device=ctx.device)
        _lib.call("pod_merge_core_gated", dptr(z), 400, dptr(z), 400, dptr(z), 400, dptr(z),
                  400, 400, 400, dptr(z), 800, 400, dptr(z), dptr(z), dptr(g), ctx.stream)


def _run(a, cfg, spec, force_leak, monkeypatch):
    monkeypatch.setattr(engine, "SPEC_CORE", spec)
    if force_leak:
        monkeypatch.setattr(engine, "REORTH_TOL", 0.0)
    engine._ENGINE_CACHE.clear()
    f, trace = pod.isma_run(a, cfg)
    engine._ENGINE_CACHE.clear()
    return f, trace


@pytest.mark.parametrize("force_leak", [False, True])
@pytest.mark.parametrize("strategy", ["l2n", "unf"])
def test_isma_speculative_core_bit_identical(strategy, force_leak, monkeypatch):
    a = workloads.config2(seed=4, side=64, n=400)
    cfg = pod.IsmaConfig(k=10, r=30, c=50, tau=1 - 1e-8, strategy=strategy, seed=3)
    f0, t0 = _run(a, cfg, False, force_leak, monkeypatch)
    f1, t1 = _run(a, cfg, True, force_leak, monkeypatch)
    assert np.array_equal(f0.sigma, f1.sigma)
    assert np.array_equal(f0.u, f1.u)
    assert len(t0) == len(t1)
