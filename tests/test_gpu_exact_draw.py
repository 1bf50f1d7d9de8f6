"""Sampled index sets are the reference's BY CONSTRUCTION (exact_sums.cu):

* pod_colnorms2 == np.einsum("ij,ij->j") bit for bit (f64 and f32 storage,
  16-byte aligned bulk path and unaligned plain path, chained row segments);
* pod_draw's normalised weights and CDF == numpy's from_weights /
  __post_init__ / cumsum bit for bit, so idx/counts == the reference's;
* every golden case recorded from the reference itself: the GPU engine's
  per-round drawn index sets and counts (engine.RECORD_DRAWS) equal the
  reference's recorded draws, round by round.
"""

import numpy as np
import pytest
from podtest_util import load_golden, make_low_rank

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1905_05107_b200 as pod  # noqa: E402
from oracle import isma_oracle as orc  # noqa: E402
from paper_1905_05107_b200 import _lib, engine, workloads  # noqa: E402
from paper_1905_05107_b200.device import ColMat, _ptr, get_ctx, to_device_colmajor  # noqa: E402

GOLDEN_CASES = ["cfg1_l2n_modes", "cfg1_unf_subspace", "cfg1_l2n_nofinal_keep11",
                "rank3_unf", "rank3_l2n", "exhaustive_40x18", "cfg2proxy_l2n", "cfg1_ort_modes",
                "rank3_ort_fallback", "rank3_unf_rows", "rank3_ort_rows", "rank3_ls_rows",
                "cfg1_ls_rows", "cfg1_unf_rows_subspace"]


def _golden_matrix(name):
    if name == "rank3_ort_fallback":
        return make_low_rank(60, 30, 3, np.random.default_rng(10))
    if name.startswith("cfg1"):
        return workloads.config1(seed=0)
    if name.startswith("rank3"):
        return make_low_rank(100, 60, 3, np.random.default_rng(7))
    if name == "exhaustive_40x18":
        return np.random.default_rng(13).standard_normal((40, 18))
    if name == "cfg2proxy_l2n":
        return workloads.config2(seed=1, side=64, n=300)
    raise KeyError(name)


@pytest.fixture
def record_draws():
    engine.RECORD_DRAWS = True
    yield
    engine.RECORD_DRAWS = False


def _gpu_norms(a, ld=None):
    ctx = get_ctx()
    if ld is None:
        A = to_device_colmajor(a, ctx.device)
    else:  # explicit (possibly odd) leading dimension: the unaligned plain path
        m, n = a.shape
        dt = torch.float32 if a.dtype == np.float32 else torch.float64
        t = torch.zeros((n, ld), dtype=dt, device=ctx.device)
        t[:, :m] = torch.as_tensor(np.ascontiguousarray(a.T))
        A = ColMat(t, m, n)
    out = torch.empty(a.shape[1], dtype=torch.float64, device=ctx.device)
    flag = torch.zeros(1, dtype=torch.int32, device=ctx.device)
    ctx.colnorms2(A, out, flag)
    return out.cpu().numpy(), int(flag.item())


@pytest.mark.parametrize("m", [1, 7, 8, 63, 64, 65, 1000, 4097, 65536, 262151])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_norms_equal_einsum_bitwise(m, dtype):
    rng = np.random.default_rng(m)
    n = 37
    a = np.asfortranarray((rng.standard_normal((m, n)) * rng.uniform(1e-3, 1e3, n)).astype(dtype))
    got, flag = _gpu_norms(a)
    a64 = a.astype(np.float64)
    assert flag == 0
    assert np.array_equal(got, np.einsum("ij,ij->j", a64, a64))
    got2, _ = _gpu_norms(a, ld=m + 1)  # unaligned leading dimension
    assert np.array_equal(got2, np.einsum("ij,ij->j", a64, a64))


def test_norms_many_columns_and_nonfinite():
    rng = np.random.default_rng(5)
    a = np.asfortranarray(rng.standard_normal((2056, 3001)))
    got, flag = _gpu_norms(a)
    assert flag == 0 and np.array_equal(got, np.einsum("ij,ij->j", a, a))
    a[1234, 2999] = np.nan
    _, flag = _gpu_norms(a)
    assert flag == 1
    b = np.full((80, 3), 1e200)  # overflow of finite entries is not "non-finite"
    got, flag = _gpu_norms(b)
    assert flag == 0 and np.isinf(got).all()


@pytest.mark.parametrize("splits", [[8], [64, 512], [1000, 2000, 3000]])
def test_chained_row_segments_equal_einsum(splits):
    """The row-sharded norm pass: segment states handed on equal one pass."""
    rng = np.random.default_rng(len(splits))
    m, n = 4003, 19
    a = np.asfortranarray(rng.standard_normal((m, n)))
    ctx = get_ctx()
    bounds = [0] + splits + [m]
    st = None
    out = torch.empty(n, dtype=torch.float64, device=ctx.device)
    flag = torch.zeros(1, dtype=torch.int32, device=ctx.device)
    for i in range(len(bounds) - 1):
        seg = to_device_colmajor(np.asfortranarray(a[bounds[i]:bounds[i + 1]]), ctx.device)
        last = i == len(bounds) - 2
        nxt = None if last else torch.empty(2 * n, dtype=torch.float64, device=ctx.device)
        ctx.colnorms2_chain(seg, st, nxt, last, out, flag)
        st = nxt
    assert np.array_equal(out.cpu().numpy(), np.einsum("ij,ij->j", a, a))


def _numpy_draw(mode, raw, live, uni):
    """The reference's arithmetic: candidates S (ascending), weights by
    from_weights/__post_init__ (or uniform), cumsum, pin, searchsorted."""
    s = np.nonzero(live)[0] if mode != 2 else np.arange(raw.size)
    if mode == 1:
        weights = pod.uniform_distribution(s).weights
    elif mode == 0:
        weights = pod.Distribution.from_weights(s, raw[s]).weights
    else:  # a Distribution's weights, used as they are (sampling.py:214)
        weights = raw
    cum = np.cumsum(weights)
    last = np.nonzero(weights)[0][-1]
    cum[last:] = 1.0
    picked = s[np.searchsorted(cum, uni, side="right")]
    uq, cnt = np.unique(picked, return_counts=True)
    return weights, cum, uq, cnt


@pytest.mark.parametrize("n", [1, 9, 130, 2000, 20000, 50003])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_draw_weights_cdf_and_indices_bitwise(n, mode):
    rng = np.random.default_rng(1000 + n + mode)
    ctx = get_ctx()
    dev = ctx.device
    lib = _lib.load()
    for trial in range(3):
        raw = rng.random(n) ** 4 * 10.0 ** rng.uniform(-3, 3)
        raw[rng.random(n) < 0.05] = 0.0
        live = (rng.random(n) < 0.7).astype(np.uint8) if mode != 2 else np.ones(n, np.uint8)
        if mode == 2:
            raw = pod.Distribution.from_weights(np.arange(n), raw + 1e-3).weights
        if live.sum() == 0:
            live[0] = 1
        if mode == 0 and raw[live.astype(bool)].sum() == 0:
            raw[np.nonzero(live)[0][0]] = 1.0
        c = 200
        uni = rng.random(c)
        w_ref, cum_ref, uq_ref, cnt_ref = _numpy_draw(mode, raw, live, uni)
        nb = (int(lib.pod_draw_exact_ws_bytes(n)) + 7) // 8 * 8
        ws = torch.zeros(nb, dtype=torch.uint8, device=dev)
        live_d = torch.as_tensor(live, device=dev)
        raw_d = torch.as_tensor(raw, device=dev)
        uni_d = torch.as_tensor(uni, device=dev)
        cap = min(c, n)
        idx = torch.empty(cap, dtype=torch.int32, device=dev)
        cnt = torch.empty(cap, dtype=torch.int64, device=dev)
        info = torch.zeros(4, dtype=torch.int64, device=dev)
        _lib.call("pod_draw_exact", mode, _ptr(raw_d), _ptr(live_d), n, _ptr(uni_d), c,
                  _ptr(idx), _ptr(cnt), cap, _ptr(ws), ws.numel(), _ptr(info), 0.0,
                  None, ctx.stream)
        g, rem, status = (int(x) for x in info[:3].cpu())
        assert status == 0
        s = w_ref.size
        wsd = ws.view(torch.float64)
        w_gpu = wsd[:s].cpu().numpy()
        cum_gpu = wsd[n:n + s].cpu().numpy()
        assert np.array_equal(w_gpu, w_ref)
        assert np.array_equal(cum_gpu, cum_ref)
        assert np.array_equal(idx[:g].cpu().numpy(), uq_ref)
        assert np.array_equal(cnt[:g].cpu().numpy(), cnt_ref)
        assert rem == s - g


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_engine_draws_equal_reference_draws(name, record_draws):
    """Each round's index set and counts drawn BY THE GPU == those the
    reference drew (recorded by tests/golden/make_golden.py)."""
    g = load_golden(name)
    k, r, c, fin, keep, w = (int(x) for x in g["meta"])
    cfg = pod.IsmaConfig(k=k, r=r, c=c, tau=float(g["tau"]), strategy=str(g["strategy"]),
                         criterion=str(g["criterion"]), seed=int(g["seed"]),
                         finalize=bool(fin), rows=w > 0, w=w or None)
    pod.isma_run(_golden_matrix(name), cfg, keep=None if keep < 0 else keep)
    log = pod.isma.LAST_DRAWS
    off = g["draw_off"]
    step = 2 if w > 0 else 1  # row cases record a column draw and a row draw per round
    ref = [(g["draw_idx"][off[i]:off[i + 1]], g["draw_cnt"][off[i]:off[i + 1]])
           for i in range(0, len(off) - 1, step)]
    assert len(log) == len(ref) == int(g["n_rounds"])
    for rnd, (entry, (ri, rc)) in enumerate(zip(log, ref)):
        assert np.array_equal(entry[0], ri), f"round {rnd}"
        assert np.array_equal(entry[1], rc), f"round {rnd}"
    if w > 0:  # ICRS: the row draws too (row norms / leverage in einsum order)
        rref = [(g["draw_idx"][off[i]:off[i + 1]], g["draw_cnt"][off[i]:off[i + 1]])
                for i in range(1, len(off) - 1, 2)]
        for rnd, (entry, (ri, rc)) in enumerate(zip(log, rref)):
            assert np.array_equal(entry[2], ri), f"row draw, round {rnd}"
            assert np.array_equal(entry[3], rc), f"row draw, round {rnd}"


@pytest.mark.parametrize("strategy", ["l2n", "unf"])
def test_engine_draws_equal_oracle_draws_pipelined_and_not(strategy, record_draws):
    """Pipelined (numpy Generator) and unpipelined (plain .random object)
    runs draw the oracle's index sets in every round."""
    a = workloads.config2(seed=3, side=48, n=700)

    class Plain:
        def __init__(self, seed):
            self.g = np.random.default_rng(seed)

        def random(self, k):
            return self.g.random(k)

    cfg = pod.IsmaConfig(k=8, r=24, c=40, tau=1 - 1e-8, strategy=strategy, seed=9)
    o = orc.run(a, 8, r=24, c=40, tau=1 - 1e-8, strategy=strategy, seed=9)
    for rng in (None, Plain(9)):
        pod.isma_run(a, cfg, rng=rng)
        log = pod.isma.LAST_DRAWS
        assert len(log) == len(o["trace"])
        for entry, t in zip(log, o["trace"]):
            assert np.array_equal(entry[0], t["unique"]) and np.array_equal(entry[1], t["counts"])
