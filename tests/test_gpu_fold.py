"""Folded CholeskyQR2 of the merge (engine.FOLD_QR / EARLY_LEAK / TRI_APPLY):
block_merge with the fold on and off agrees to working precision and with the
CPU oracle, on the cases that drive every gated branch -- a plain update, an
update nearly inside span(U1) (the leak check of merge.py:72-73 fires and the
second projection materializes Q), an ill-conditioned residual (further
CholeskyQR passes materialize Q) and zero-padded updates -- at ranks on both
sides of the in-place NN width, the triangular-apply widths and the
speculative-core limit."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_1905_05107_b200 as pod

def cases(m, r):
    rng = np.random.default_rng(11)
    q = np.linalg.qr(rng.standard_normal((m, 2 * r)))[0]
    u1, fresh = q[:, :r], q[:, r:]
    s1 = np.linspace(9.0, 1.0, r)
    s2 = np.linspace(7.0, 0.5, r)
    out = []
    out.append((u1, s1, fresh, s2))                                   # plain
    # nearly inside span(U1): residual ~1e-9, leak amplified past 1e-8
    mix = np.linalg.qr(u1 @ rng.standard_normal((r, r)) + 1e-9 * fresh)[0]
    out.append((u1, s1, mix, s2))
    # ill-conditioned residual: directions fading over 12 decades
    fade = np.linalg.qr(u1 @ rng.standard_normal((r, r))
                        + fresh * np.logspace(0, -12, r))[0]
    out.append((u1, s1, fade, s2))
    # short update (zero-padded slots)
    k2 = max(1, r // 3)
    out.append((u1, s1, fresh[:, :k2], s2[:k2]))
    return out

res = []
for m, r in {shapes!r}:
    for u1, s1, u2, s2 in cases(m, r):
        f = pod.block_merge(pod.TruncatedFactor(u1, s1), pod.TruncatedFactor(u2, s2), r)
        res.append(np.array([float(f.nmodes)]))
        res.append(f.sigma)
        res.append(f.u.reshape(-1))
np.save({out!r}, np.concatenate(res))
"""

SHAPES = [(3000, 24), (4000, 130), (4096, 200)]


def _run(tmp_path, tag, **env):
    out = str(tmp_path / f"{tag}.npy")
    subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT, shapes=SHAPES, out=out)],
                   env=dict(os.environ, **env), check=True)
    return np.load(out)


def _split(flat):
    """-> list of (sigma, u, nmodes) per case, in the script's order."""
    out, pos = [], 0
    for m, r in SHAPES:
        for _ in range(4):
            nm = int(flat[pos])
            assert 1 <= nm <= r
            sig = flat[pos + 1:pos + 1 + nm]
            end = pos + 1 + nm + m * nm
            out.append((sig, flat[pos + 1 + nm:end].reshape(m, nm), nm))
            pos = end
    assert pos == flat.size
    return out


def test_fold_on_off_agree_and_match_oracle(tmp_path):
    from oracle import isma_oracle as orc
    from parity_util import principal_angles_sin, sigma_relerr

    on = _split(_run(tmp_path, "on"))
    off = _split(_run(tmp_path, "off", POD_FOLD_QR="0", POD_EARLY_LEAK="0", POD_TRI_APPLY="0"))
    assert len(on) == len(off) == 4 * len(SHAPES)
    for (s_on, u_on, n_on), (s_off, u_off, n_off) in zip(on, off):
        assert n_on == n_off
        assert sigma_relerr(s_on, s_off) <= 1e-12
        assert principal_angles_sin(u_on, u_off).max() <= 1e-10
        # the merged basis stays orthonormal to working precision
        assert np.abs(u_on.T @ u_on - np.eye(n_on)).max() <= 1e-12
    # and against the oracle's block_merge on the first shape's cases
    rng = np.random.default_rng(11)
    m, r = SHAPES[0]
    q = np.linalg.qr(rng.standard_normal((m, 2 * r)))[0]
    u1, fresh = q[:, :r], q[:, r:]
    s1, s2 = np.linspace(9.0, 1.0, r), np.linspace(7.0, 0.5, r)
    o = orc.merge(u1, s1, fresh, s2, r)
    assert sigma_relerr(on[0][0], o[1]) <= 1e-12
    assert principal_angles_sin(on[0][1], o[0]).max() <= 1e-10
