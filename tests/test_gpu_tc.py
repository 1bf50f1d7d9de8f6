"""The tcgen05 (5th-generation tensor core, TMEM accumulator) 3xTF32 TN
product used by the mixed-precision path for float32-stored matrices
(BASELINE config 4): C = alpha X^T Y against the fp64 product of the same
fp32 values.  3xTF32 with fp32 accumulation over <= 8192-row chunks and an
fp64 chunk reduction: relative error (max |err| / max |C|) <= 1e-5 (measured 2-5e-6)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1905_05107_b200.device import ColMat, dptr, get_ctx  # noqa: E402

TOL = 1e-5


def _colmat(a, dev):
    """Column-major device copy with the leading dimension padded to a
    multiple of 4 (the 16-byte cp.async staging needs it)."""
    m, n = a.shape
    ld = (m + 3) // 4 * 4
    t = torch.zeros((n, ld), dtype=torch.float32, device=dev)
    t[:, :m] = torch.as_tensor(np.ascontiguousarray(a.T), device=dev)
    return ColMat(t, m, n)


def _relerr(got, ref):
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300))


@pytest.mark.parametrize("K,P,Q", [(20000, 300, 192), (8192, 128, 256), (50001, 77, 100),
                                   (31, 5, 16), (100000, 256, 64)])
def test_tn_tf32x3_matches_fp64(K, P, Q):
    ctx = get_ctx()
    dev = ctx.device
    rng = np.random.default_rng(K + P + Q)
    x = (rng.standard_normal((K, P)) * rng.uniform(0.1, 10, P)).astype(np.float32)
    y = rng.standard_normal((K, Q)).astype(np.float32)
    C = torch.zeros(P * Q, dtype=torch.float64, device=dev)
    ctx.tn_tf32x3(P, Q, 1.5, _colmat(x, dev), _colmat(y, dev), dptr(C), P)
    got = C.view(Q, P).cpu().numpy().T
    ref = 1.5 * (x.astype(np.float64).T @ y.astype(np.float64))
    assert _relerr(got, ref) <= TOL


def test_tn_tf32x3_gathered_gram_and_split_fp64():
    """The sampled Gram D^T D with D = A[:, idx] gathered in the loads (index
    -1 = zero column), and A^T U with an fp64 U pre-split into TF32 hi/lo."""
    ctx = get_ctx()
    dev = ctx.device
    rng = np.random.default_rng(3)
    K, n = 30000, 700
    a = rng.standard_normal((K, n)).astype(np.float32)
    A = _colmat(a, dev)
    idx = np.sort(rng.choice(n, 180, replace=False)).astype(np.int32)
    idx_pad = np.concatenate([idx, -np.ones(12, np.int32)])
    cols = torch.as_tensor(idx_pad, device=dev)
    g = idx_pad.size
    G = torch.zeros(g * g, dtype=torch.float64, device=dev)
    ctx.tn_tf32x3(g, g, 1.0, A, A, dptr(G), g, xcols=cols, ycols=cols)
    got = G.view(g, g).cpu().numpy().T
    d = np.zeros((K, g))
    d[:, :idx.size] = a[:, idx].astype(np.float64)
    assert _relerr(got, d.T @ d) <= TOL
    assert np.all(got[idx.size:, :] == 0) and np.all(got[:, idx.size:] == 0)
    # A^T U, U fp64 (m x r) split into TF32 (hi, lo)
    u = np.linalg.qr(rng.standard_normal((K, 96)))[0]
    U = ColMat(torch.as_tensor(np.ascontiguousarray(u.T), device=dev), K, 96)  # fp64
    hi = torch.empty(K * 96, dtype=torch.float32, device=dev)
    lo = torch.empty(K * 96, dtype=torch.float32, device=dev)
    ctx.split_tf32(U, 96, hi, lo)
    C = torch.zeros(n * 96, dtype=torch.float64, device=dev)
    ctx.tn_tf32x3(n, 96, 1.0, A, ColMat(hi.view(96, K), K, 96), dptr(C), n, Ylo=lo)
    got = C.view(96, n).cpu().numpy().T
    assert _relerr(got, a.astype(np.float64).T @ u) <= TOL


def test_mixed_precision_isma_config4_proxy():
    """precision="mixed" on a float32-stored config-4 proxy: finalize's A^T U
    on the tcgen05 tensor cores (3xTF32; the sampled Gram too with
    POD_TC_GRAM=1).  Against the
    fp64 oracle on the exact upcast: identical draws in every round (the
    norms and the draw are exact), sigma within 1e-4 relative and principal
    angles below 1e-3 rad (north_star's mixed-precision tolerances; measured
    errors are printed)."""
    import paper_1905_05107_b200 as pod
    from oracle import isma_oracle as orc
    from paper_1905_05107_b200 import engine, isma, workloads
    from parity_util import principal_angles_sin, sigma_relerr

    a32 = workloads.config4_torch(7, 256, 1200, device="cpu").numpy().T  # (65536, 1200) fp32
    cfg = pod.IsmaConfig(k=16, r=48, c=64, tau=1 - 1e-8, strategy="l2n", seed=3)
    engine.RECORD_DRAWS = True
    try:
        fm, trm = pod.isma_run(a32, cfg, precision="mixed")
        dm = isma.LAST_DRAWS
        fd, trd = pod.isma_run(a32, cfg)
        dd = isma.LAST_DRAWS
    finally:
        engine.RECORD_DRAWS = False
    o = orc.run(a32.astype(np.float64), 16, r=48, c=64, tau=1 - 1e-8, strategy="l2n", seed=3)
    assert len(dm) == len(dd) == len(o["trace"])
    for (gi, gc), (hi, hc), t in zip(dm, dd, o["trace"]):
        assert np.array_equal(gi, t["unique"]) and np.array_equal(hi, t["unique"])
    es = sigma_relerr(fm.sigma, o["sigma"])
    ea = principal_angles_sin(fm.u, o["u"]).max()
    print(f"mixed vs fp64 oracle: sigma rel err {es:.2e}, max angle {ea:.2e} rad; "
          f"fp64 path: {sigma_relerr(fd.sigma, o['sigma']):.2e}")
    assert es <= 1e-4 and ea <= 1e-3
