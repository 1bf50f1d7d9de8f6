"""Seeded synthetic inputs with the shapes of BASELINE.json's configs.

The reference's own datasets (ORL Faces, V2D snapshots, Yale Faces; see
``ref/PAPER.md:89-104``) are not available, so these generators stand in
for them with the shapes, spectra and noise levels BASELINE.json states.
Noise "N(0, x)" is read as variance x.

* ``config1`` -- A = U diag(exp(-i/10)) V^T + N(0, 1e-6), m=2000, n=500,
  U, V Haar (Q of QR of N(0,1)), numpy PCG64 from a seed; CPU-reproducible.
* ``config2`` -- snapshot-like Fourier field: column t is
  sum_{j=1..40} j^-2 cos(2 pi (kx_j x + ky_j y)/L + phi_{j,t}) on an L x L
  grid flattened (L=512 -> m=262144), n=2000, + N(0, 1e-4), rows mean-centred
  (``matcore.py:168-175`` semantics).  Built as A = B C with B the m x 80
  cos/sin basis, so it is a GEMM on the device; ``side`` shrinks the grid
  for proxies.

Data generation is outside every timed region.
"""

from __future__ import annotations

import math

import numpy as np

CFG1 = dict(m=2000, n=500, k=10, r=30, c=50, tol=1e-8)
CFG2 = dict(side=512, n=2000, k=20, r=60, c=100, tol=1e-8)


def config1(seed=0, m=2000, n=500, noise_var=1e-6):
    """BASELINE config 1 (CPU-runnable oracle case), float64 F-order."""
    rng = np.random.default_rng(seed)
    u = np.linalg.qr(rng.standard_normal((m, n)))[0]
    v = np.linalg.qr(rng.standard_normal((n, n)))[0]
    s = np.exp(-np.arange(n) / 10.0)
    a = (u * s) @ v.T + math.sqrt(noise_var) * rng.standard_normal((m, n))
    return np.asfortranarray(a)


def _fourier_modes(seed, nmodes=40, kmax=12):
    rng = np.random.default_rng(seed)
    ks = set()
    out = []
    while len(out) < nmodes:
        kx, ky = (int(v) for v in rng.integers(-kmax, kmax + 1, size=2))
        if (kx, ky) == (0, 0) or (kx, ky) in ks or (-kx, -ky) in ks:
            continue
        ks.add((kx, ky))
        out.append((kx, ky))
    return np.array(out, dtype=np.float64)


NOISE_CHUNK = 4096  # rows per independently seeded noise chunk (shard-invariant A)


def config2_torch(seed=0, side=512, n=2000, noise_var=1e-4, device="cpu", nmodes=40,
                  rows=None):
    """BASELINE config 2 snapshot matrix rows [r0, r1) (default: all m rows)
    as a column-major float64 torch tensor: storage (n, r1 - r0), i.e. the
    row block's transpose is contiguous.  The noise of global rows
    [c*4096, (c+1)*4096) comes from a generator seeded by (seed, c), so any
    row partition (one GPU or a row-sharded multi-GPU run) produces the same
    matrix.  Deterministic for a (seed, device type) pair."""
    import torch

    m = side * side
    r0, r1 = (0, m) if rows is None else (int(rows[0]), int(rows[1]))
    modes = _fourier_modes(seed, nmodes)
    dt = torch.float64
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed) * 7919 + 17)
    amp = torch.arange(1, nmodes + 1, dtype=dt, device=device) ** -2.0
    phi = 2.0 * math.pi * torch.rand((nmodes, n), generator=gen, dtype=dt, device=device)
    coef = torch.cat([amp[:, None] * torch.cos(phi), -amp[:, None] * torch.sin(phi)], dim=0)
    kx = torch.tensor(modes[:, 0], dtype=dt, device=device)
    ky = torch.tensor(modes[:, 1], dtype=dt, device=device)
    sd = math.sqrt(noise_var)
    at = torch.empty((n, r1 - r0), dtype=dt, device=device)
    # every quantity is computed per global 4096-row chunk (identical shapes
    # whatever the row partition), then the requested rows are sliced out
    for c in range(r0 // NOISE_CHUNK, (r1 + NOISE_CHUNK - 1) // NOISE_CHUNK):
        c0, c1 = c * NOISE_CHUNK, min(m, (c + 1) * NOISE_CHUNK)
        idx = torch.arange(c0, c1, dtype=torch.int64, device=device)
        x = (idx % side).to(dt)
        y = (idx // side).to(dt)
        theta = (2.0 * math.pi / side) * (x[:, None] * kx[None, :] + y[:, None] * ky[None, :])
        basis = torch.cat([torch.cos(theta), torch.sin(theta)], dim=1)  # chunk x 2J
        blk = (basis @ coef).T.contiguous()  # (n, chunk)
        g = torch.Generator(device=device)
        g.manual_seed((int(seed) * 1000003 + c * 7 + 3) % (2 ** 62))
        blk.add_(torch.randn((n, c1 - c0), generator=g, dtype=dt, device=device), alpha=sd)
        blk.sub_(blk.mean(dim=0, keepdim=True))  # subtract each row's mean
        lo, hi = max(c0, r0), min(c1, r1)
        at[:, lo - r0:hi - r0].copy_(blk[:, lo - c0:hi - c0])
    return at


def config2(seed=0, side=512, n=2000, noise_var=1e-4):
    """Host (numpy, F-order) copy of ``config2_torch`` generated on the CPU."""
    at = config2_torch(seed, side, n, noise_var, device="cpu")
    return np.asfortranarray(at.numpy().T)
