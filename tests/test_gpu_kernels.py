"""Kernel-level parity on the B200: each C-ABI entry point against numpy /
the CPU oracle on seeded inputs (fp64: rtol stated per test)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from oracle import isma_oracle as orc  # noqa: E402
from paper_1905_05107_b200.device import ColMat, dptr, get_ctx, to_device_colmajor  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    return get_ctx()


def dev_mat(a, ctx):
    return to_device_colmajor(np.asfortranarray(a), ctx.device)


@pytest.mark.parametrize("m,n", [(1, 1), (7, 3), (2000, 500), (5000, 37), (262144 + 3, 5)])
def test_colnorms(ctx, m, n):
    a = np.random.default_rng(m + n).standard_normal((m, n))
    A = dev_mat(a, ctx)
    out = torch.empty(n, dtype=torch.float64, device=ctx.device)
    flag = torch.zeros(1, dtype=torch.int32, device=ctx.device)
    ctx.colnorms2(A, out, flag)
    ref = np.einsum("ij,ij->j", a, a)
    np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=1e-13)
    assert flag.item() == 0


def test_colnorms_nonfinite(ctx):
    a = np.ones((5000, 4))
    a[1234, 2] = np.nan
    A = dev_mat(a, ctx)
    out = torch.empty(4, dtype=torch.float64, device=ctx.device)
    flag = torch.zeros(1, dtype=torch.int32, device=ctx.device)
    ctx.colnorms2(A, out, flag)
    assert flag.item() == 1


def _draw(ctx, mode, weights, live, n, u):
    c = len(u)
    idx = torch.empty(c, dtype=torch.int32, device=ctx.device)
    cnt = torch.empty(c, dtype=torch.int64, device=ctx.device)
    wt = None if weights is None else torch.as_tensor(weights, dtype=torch.float64,
                                                      device=ctx.device)
    lv = None if live is None else torch.as_tensor(live, dtype=torch.uint8, device=ctx.device)
    ut = torch.as_tensor(np.asarray(u, dtype=np.float64), device=ctx.device)
    ctx.draw(mode, wt, lv, n, ut, c, idx, cnt)
    g, rem, st = ctx.read_info(3)
    return idx[:g].cpu().numpy(), cnt[:g].cpu().numpy(), rem, st, lv


def test_draw_inverse_cdf_known_answer(ctx):
    # reference tests/test_sampling.py:197-203 (positions 0,1,2 <-> indices 3,7,9)
    idx, cnt, _, st, _ = _draw(ctx, 2, [0.2, 0.3, 0.5], None, 3, [0.05, 0.21, 0.45, 0.51, 0.99])
    assert st == 0
    np.testing.assert_array_equal(idx, [0, 1, 2])
    np.testing.assert_array_equal(cnt, [1, 2, 2])


def test_draw_cdf_edge(ctx):
    # reference tests/test_sampling.py:236-242
    idx, _, _, _, _ = _draw(ctx, 2, [0.5, 0.5, 0.0], None, 3, [1.0 - 1e-16, 0.999999999])
    np.testing.assert_array_equal(idx, [1])


@pytest.mark.parametrize("n,c,mode", [(500, 50, 0), (2000, 100, 0), (2000, 100, 1),
                                      (20000, 200, 0), (7, 300, 1), (50000, 128, 0)])
def test_draw_matches_oracle_over_rounds(ctx, n, c, mode):
    rng = np.random.default_rng(n + c)
    norms2 = rng.random(n) ** 3
    norms2[rng.integers(0, n, size=n // 10)] = 0.0
    live = np.ones(n, dtype=np.uint8)
    lv_dev = torch.as_tensor(live, device=ctx.device)
    w_dev = torch.as_tensor(norms2, device=ctx.device)
    gen = np.random.default_rng(5)
    s = np.arange(n)
    idx_t = torch.empty(c, dtype=torch.int32, device=ctx.device)
    cnt_t = torch.empty(c, dtype=torch.int64, device=ctx.device)
    for rnd in range(6):
        if mode == 0:
            if not np.any(norms2[s] > 0):
                break
            w = orc.normalized_weights(norms2[s])
        else:
            w = orc.uniform_weights(s.size)
        u = gen.random(c)
        ref_idx, ref_cnt = orc.cdf_draw(s, w, u)
        ut = torch.as_tensor(u, device=ctx.device)
        ctx.draw(mode, w_dev if mode == 0 else None, lv_dev, n, ut, c, idx_t, cnt_t)
        g, rem, st = ctx.read_info(3)
        assert st == 0
        np.testing.assert_array_equal(idx_t[:g].cpu().numpy(), ref_idx)
        np.testing.assert_array_equal(cnt_t[:g].cpu().numpy(), ref_cnt)
        s = np.setdiff1d(s, ref_idx, assume_unique=True)
        assert rem == s.size
        if s.size == 0:
            break


def test_draw_degenerate_and_empty(ctx):
    _, _, rem, st, _ = _draw(ctx, 0, [0.0, 0.0, 0.0], [1, 1, 1], 3, [0.5])
    assert st == 2
    _, _, rem, st, _ = _draw(ctx, 1, None, [0, 0, 0], 3, [0.5])
    assert st == 1


@pytest.mark.parametrize("m,p,q", [(1, 1, 1), (37, 5, 3), (2000, 50, 50), (4097, 64, 65),
                                   (262144, 100, 100), (100003, 7, 130), (2000, 500, 30)])
def test_gemm_tn(ctx, m, p, q):
    rng = np.random.default_rng(m + p + q)
    x = rng.standard_normal((m, p))
    y = rng.standard_normal((m, q))
    X, Y = dev_mat(x, ctx), dev_mat(y, ctx)
    C = torch.empty(p * q, dtype=torch.float64, device=ctx.device)
    ctx.tn(p, q, 2.0, X, Y, dptr(C), p)
    got = C.cpu().numpy().reshape(q, p).T
    ref = 2.0 * x.T @ y
    np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())


@pytest.mark.parametrize("m,p", [(50001, 150), (7, 160), (20000, 161), (100000, 200), (3000, 240),
                                 (1000003, 150), (40000, 300), (60001, 192), (20000, 256),
                                 (5000, 100), (3000, 129), (200000, 128)])
def test_gemm_tn_symmetric_balanced(ctx, m, p):
    """Symmetric products on 80- and 64-wide tiles (config 3: r = 150,
    g = 200; config 4: 192, 256; config 2: g = 100): the diagonal tiles
    compute only their upper fragments and the K split weights tiles by
    their work -- exactly symmetric C, numpy's values, and the same with an
    index list holding -1 (zero) padding columns."""
    rng = np.random.default_rng(m + p)
    x = rng.standard_normal((m, p))
    X = dev_mat(x, ctx)
    C = torch.empty(p * p, dtype=torch.float64, device=ctx.device)
    ctx.tn(p, p, 1.0, X, X, dptr(C), p)
    got = C.cpu().numpy().reshape(p, p).T
    ref = x.T @ x
    np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-12 * np.abs(ref).max())
    assert np.array_equal(got, got.T)
    idx = np.arange(p, dtype=np.int32)
    idx[p - 3:] = -1
    it = torch.as_tensor(idx, device=ctx.device)
    ctx.tn(p, p, 1.0, X, X, dptr(C), p, xcols=it, ycols=it)
    got = C.cpu().numpy().reshape(p, p).T
    d = x.copy()
    d[:, p - 3:] = 0.0
    np.testing.assert_allclose(got, d.T @ d, rtol=1e-11, atol=1e-12 * np.abs(ref).max())
    assert np.array_equal(got, got.T)


def test_gemm_tn_gather(ctx):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((3001, 40))
    idx = np.array([1, 5, 6, 20, 39, 0], dtype=np.int32)
    A = dev_mat(a, ctx)
    it = torch.as_tensor(idx, device=ctx.device)
    g = idx.size
    C = torch.empty(g * g, dtype=torch.float64, device=ctx.device)
    ctx.tn(g, g, 1.0, A, A, dptr(C), g, xcols=it, ycols=it)
    d = a[:, idx]
    np.testing.assert_allclose(C.cpu().numpy().reshape(g, g).T, d.T @ d, rtol=1e-12)


@pytest.mark.parametrize("m,p,q", [(1, 1, 1), (129, 3, 5), (2000, 50, 30), (262144, 100, 60),
                                   (5000, 120, 60), (3000, 30, 190), (20000, 64, 128)])
def test_gemm_nn(ctx, m, p, q):
    rng = np.random.default_rng(m * 7 + p + q)
    x = rng.standard_normal((m, p))
    t = rng.standard_normal((p, q))
    z = rng.standard_normal((m, q))
    X, Z = dev_mat(x, ctx), dev_mat(z, ctx)
    T = torch.as_tensor(np.asfortranarray(t).T.copy().reshape(-1), device=ctx.device)
    Y = ColMat.zeros(m, q, ctx.device)
    ctx.nn(p, q, -1.5, X, dptr(T), p, Y, beta=0.5, Z=Z)
    ref = -1.5 * x @ t + 0.5 * z
    np.testing.assert_allclose(Y.to_numpy(), ref, rtol=1e-11, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("m,p,q", [(1, 1, 1), (100, 7, 7), (4099, 20, 20), (262144 + 5, 60, 60),
                                   (70001, 64, 64), (5000, 48, 40)])
@pytest.mark.parametrize("beta", [0.0, 0.5])
def test_gemm_nn_gram_epilogue(ctx, m, p, q, beta):
    """pod_gemm_nn_gram: Y as pod_gemm_nn and G = Y^T Y from the output
    tiles (exactly symmetric); a zero gate leaves Y and G untouched."""
    rng = np.random.default_rng(m + 3 * p + q)
    x = rng.standard_normal((m, p))
    t = rng.standard_normal((p, q))
    z = rng.standard_normal((m, q))
    X, Z = dev_mat(x, ctx), dev_mat(z, ctx)
    T = torch.as_tensor(np.asfortranarray(t).T.copy().reshape(-1), device=ctx.device)
    Y = ColMat.zeros(m, q, ctx.device)
    ldg = q + 3
    G = torch.full((q * ldg,), 7.0, dtype=torch.float64, device=ctx.device)
    assert ctx.nn_gram_ok(p, q)
    ctx.nn_gram(p, q, -1.5, X, dptr(T), p, Y, dptr(G), ldg, beta=beta, Z=Z if beta else None)
    ref = -1.5 * x @ t + beta * z
    y = Y.to_numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-11, atol=1e-12 * np.abs(ref).max())
    g = G.cpu().numpy().reshape(q, ldg).T[:q, :]  # column-major q x q, ld = ldg
    gref = y.T @ y
    np.testing.assert_allclose(g, gref, rtol=1e-12, atol=1e-13 * np.abs(gref).max())
    assert np.array_equal(g, g.T)
    gate = torch.zeros(1, dtype=torch.int32, device=ctx.device)
    Y.t.zero_()
    ctx.nn_gram(p, q, 1.0, X, dptr(T), p, Y, dptr(G), ldg, gate=gate)
    assert not Y.to_numpy().any() and np.array_equal(G.cpu().numpy().reshape(q, ldg).T[:q], g)


@pytest.mark.parametrize("m,p,q,k", [(77, 8, 8, 8), (1000, 60, 30, 10), (262144 + 3, 120, 60, 20),
                                     (100003, 300, 150, 50), (5001, 400, 200, 64)])
def test_gemm_nn_dots_rotation_cosines(ctx, m, p, q, k):
    """pod_gemm_nn_dots: the rotation Y = X T and the raw cosines
    dots[j] = Y[:, j] . X[:, j] (j < k) formed in its epilogue."""
    rng = np.random.default_rng(m + p + q + k)
    x = rng.standard_normal((m, p))
    t = rng.standard_normal((p, q))
    X = dev_mat(x, ctx)
    T = torch.as_tensor(np.asfortranarray(t).T.copy().reshape(-1), device=ctx.device)
    Y = ColMat.zeros(m, q, ctx.device)
    dots = torch.full((k,), 3.0, dtype=torch.float64, device=ctx.device)
    ctx.nn_dots(p, q, 0.75, X, dptr(T), p, Y, k, dots)
    ref = 0.75 * x @ t
    np.testing.assert_allclose(Y.to_numpy(), ref, rtol=1e-11, atol=1e-12 * np.abs(ref).max())
    y = Y.to_numpy()
    dref = np.einsum("ij,ij->j", y[:, :k], x[:, :k])
    np.testing.assert_allclose(dots.cpu().numpy(), dref, rtol=1e-11,
                               atol=1e-13 * np.sqrt((y[:, :k] ** 2).sum() * (x[:, :k] ** 2).sum()))


def test_gemm_nn_gram_shape_limits(ctx):
    assert not ctx.nn_gram_ok(60, 65) and not ctx.nn_gram_ok(30, 40) and ctx.nn_gram_ok(64, 64)


def test_gemm_nn_inplace_and_gather(ctx):
    rng = np.random.default_rng(11)
    a = rng.standard_normal((10000, 30))
    idx = np.array([3, 4, 29, 0], dtype=np.int32)
    t = rng.standard_normal((4, 8))
    A = dev_mat(a, ctx)
    T = torch.as_tensor(np.asfortranarray(t).T.copy().reshape(-1), device=ctx.device)
    Y = ColMat.zeros(10000, 8, ctx.device)
    ctx.nn(4, 8, 1.0, A, dptr(T), 4, Y, xcols=torch.as_tensor(idx, device=ctx.device))
    np.testing.assert_allclose(Y.to_numpy(), a[:, idx] @ t, rtol=1e-12, atol=1e-13)
    # in place: Y <- Y S
    s = rng.standard_normal((8, 8))
    Sd = torch.as_tensor(np.asfortranarray(s).T.copy().reshape(-1), device=ctx.device)
    before = Y.to_numpy()
    ctx.nn(8, 8, 1.0, Y, dptr(Sd), 8, Y)
    np.testing.assert_allclose(Y.to_numpy(), before @ s, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("g", [1, 2, 17, 50, 100, 160, 200])
def test_gram_eigh_matches_reference_semantics(ctx, g):
    rng = np.random.default_rng(g)
    d = rng.standard_normal((3 * g + 5, g)) * np.exp(-np.arange(g) / 8.0)
    G = d.T @ d
    r = max(1, (2 * g) // 3)
    Gd = torch.as_tensor(np.asfortranarray(G).T.copy().reshape(-1), device=ctx.device)
    sig = torch.empty(g, dtype=torch.float64, device=ctx.device)
    T = torch.empty(g * r, dtype=torch.float64, device=ctx.device)
    ctx.gram_eigh(dptr(Gd), g, g, r, sig, dptr(T), g)
    rank, keep, sweeps = ctx.read_info(3)
    s_ref, v_ref = orc.gram_eig(d)
    np.testing.assert_allclose(sig.cpu().numpy(), s_ref, rtol=1e-10, atol=1e-13 * s_ref[0])
    keep_ref = min(r, int(np.count_nonzero(s_ref > 1e-14 * s_ref[0])))
    assert keep == keep_ref
    Tn = T.cpu().numpy().reshape(r, g).T[:, :keep]
    u_gpu = d @ Tn
    u_ref = d @ v_ref[:, :keep] / s_ref[:keep]
    cos = np.abs(np.einsum("ij,ij->j", u_gpu, u_ref))
    assert np.all(cos > 1 - 1e-9)


def test_gram_eigh_dust_and_rank(ctx):
    # exactly rank-3 sample: dust eigenvalues zeroed (baselines.py:46-47)
    rng = np.random.default_rng(0)
    d = rng.standard_normal((100, 3)) @ rng.standard_normal((3, 20))
    G = d.T @ d
    Gd = torch.as_tensor(np.asfortranarray(G).T.copy().reshape(-1), device=ctx.device)
    sig = torch.empty(20, dtype=torch.float64, device=ctx.device)
    T = torch.empty(20 * 9, dtype=torch.float64, device=ctx.device)
    ctx.gram_eigh(dptr(Gd), 20, 20, 9, sig, dptr(T), 20)
    rank, keep, _ = ctx.read_info(3)
    assert rank == 3 and keep == 3
    assert np.all(sig.cpu().numpy()[3:] == 0.0)


@pytest.mark.parametrize("nr,nc", [(1, 1), (5, 5), (60, 60), (120, 120), (200, 30), (300, 150)])
def test_svd_small(ctx, nr, nc):
    rng = np.random.default_rng(nr + nc)
    a = rng.standard_normal((nr, nc)) * np.exp(-np.arange(nc) / 10.0)
    Ad = torch.as_tensor(np.asfortranarray(a).T.copy().reshape(-1), device=ctx.device)
    U = torch.empty(nr * nc, dtype=torch.float64, device=ctx.device)
    V = torch.empty(nc * nc, dtype=torch.float64, device=ctx.device)
    s = torch.empty(nc, dtype=torch.float64, device=ctx.device)
    ctx.svd_small(dptr(Ad), nr, nr, nc, dptr(U), nr, s, dptr(V), nc)
    s_ref = np.linalg.svd(a, compute_uv=False)
    np.testing.assert_allclose(s.cpu().numpy(), s_ref, rtol=1e-12, atol=1e-14 * s_ref[0])
    u = U.cpu().numpy().reshape(nc, nr).T
    v = V.cpu().numpy().reshape(nc, nc).T
    np.testing.assert_allclose((u * s.cpu().numpy()) @ v.T, a, atol=1e-13 * s_ref[0])
    assert np.abs(v.T @ v - np.eye(nc)).max() < 1e-13


@pytest.mark.parametrize("m,l,cond", [(1000, 10, 1e2), (50000, 60, 1e6), (3000, 130, 1e3),
                                      (20000, 60, 1e12), (200000, 150, 1e6), (5000, 158, 1e10),
                                      (4000, 105, 1e3), (3000, 159, 1e3), (30000, 192, 1e8), (3000, 230, 1e3),
                                      (3000, 231, 1e3)])
def test_cholqr_orthonormal(ctx, m, l, cond):
    from paper_1905_05107_b200.engine import G_QR, MergeWorkspace
    rng = np.random.default_rng(l)
    q0 = np.linalg.qr(rng.standard_normal((m, l)))[0]
    w = q0 * np.logspace(0, -np.log10(cond), l) @ np.linalg.qr(rng.standard_normal((l, l)))[0]
    ws = MergeWorkspace(ctx, m, l)
    W = dev_mat(w, ctx)
    Q = ColMat.zeros(m, l, ctx.device)
    R = torch.zeros(l * l, dtype=torch.float64, device=ctx.device)
    ws.cholqr_ops(W, Q, l, R, G_QR)
    q = Q.to_numpy()
    rr = R.cpu().numpy().reshape(l, l).T
    assert np.abs(q.T @ q - np.eye(l)).max() < 1e-12
    np.testing.assert_allclose(q @ rr, w, atol=1e-13 * np.abs(w).max())


_CQ_SCRIPT = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_1905_05107_b200.device import get_ctx, dptr
ctx = get_ctx()
rng = np.random.default_rng(4)
l = {l}
w = rng.standard_normal((3000, l)) * np.logspace(0, -5, l)
w[:, 7] = 0.0  # a dead column
g = w.T @ w
G = torch.as_tensor(np.asfortranarray(g).T.copy().reshape(-1), device=ctx.device)
Ri = torch.zeros(l * l, dtype=torch.float64, device=ctx.device)
R = torch.zeros(l * l, dtype=torch.float64, device=ctx.device)
ctx.cholqr_factor(dptr(G), l, l, 3000, dptr(Ri), l, dptr(R), l)
torch.cuda.synchronize()
np.save({out!r}, np.concatenate([R.cpu().numpy(), Ri.cpu().numpy()]))
"""


@pytest.mark.parametrize("l", [120, 150, 192, 230])
def test_cholqr_inplace_factor_bitwise_equals_global_path(tmp_path, l):
    """The shared-memory in-place factor (104 < l <= 158) reproduces the
    global-memory kernel bit for bit, dead column included."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        out = str(tmp_path / f"cq{flag}.npy")
        env = dict(os.environ, POD_CHOLQR_INPLACE=flag)
        subprocess.run([sys.executable, "-c", _CQ_SCRIPT.format(root=root, l=l, out=out)],
                       env=env, check=True)
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])
    rr = outs[0][:l * l].reshape(l, l).T
    ri = outs[0][l * l:].reshape(l, l).T
    live = np.ones(l, bool)
    live[7] = False
    np.testing.assert_allclose((ri @ rr)[np.ix_(live, live)], np.eye(l - 1), atol=1e-9)
    assert not rr[7].any() and not rr[:, 7].any() and not ri[7].any() and not ri[:, 7].any()


def test_fix_signs_and_coldots(ctx):
    rng = np.random.default_rng(2)
    u = rng.standard_normal((20000, 7))
    u[5, 3] = -100.0
    u[9, 3] = 100.0  # tie: first occurrence (row 5, negative) wins -> flip
    v = rng.standard_normal((50, 7))
    U, V = dev_mat(u, ctx), dev_mat(v, ctx)
    ctx.fix_signs(U, 7, V, 50)
    ru, rv = orc.canon_signs(u, v)
    np.testing.assert_array_equal(U.to_numpy(), ru)
    np.testing.assert_array_equal(V.to_numpy(), rv)
    out = torch.zeros(9, dtype=torch.float64, device=ctx.device)
    P = dev_mat(ru / np.linalg.norm(ru, axis=0), ctx)
    ctx.coldots(P, P, 9, 7, True, out)
    np.testing.assert_allclose(out.cpu().numpy(), [1.0] * 7 + [0.0, 0.0], atol=1e-15)
