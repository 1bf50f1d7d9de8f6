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

* ``config4`` -- the config-2 generator at 1024 x 1024 (m = 1,048,576),
  n = 8192, stored float32 (the reference upcasts to float64 in as_dense;
  the kernels upcast exactly, so the fp64 oracle on the upcast is the
  parity reference).
* ``config5_host`` -- the out-of-core workload: rank-100 exp(-i/20) spectrum
  + N(0, 1e-5), stored float32 in page-locked host memory, generated block
  by block (4096-row chunks on the device, copied into the host block).
* ``config3`` -- power-law low-rank-plus-noise: A = U diag(i^-1.5) V^T +
  N(0, 1e-6), rank 200, m=1,000,000, n=20,000 (160 GB fp64), generated on
  the device.  U is Haar: G R^-1 with G ~ N(0,1) per 4096-row chunk and R the
  Cholesky factor of G^T G summed over all chunks in chunk order (= the R of
  a positive-diagonal QR), so every row partition yields the same matrix;
  V = Q of a (replicated) QR of an n x 200 Gaussian.  ``m``/``n`` shrink it
  for parity proxies.

Data generation is outside every timed region.
"""

from __future__ import annotations

import math

import numpy as np

CFG1 = dict(m=2000, n=500, k=10, r=30, c=50, tol=1e-8)
CFG2 = dict(side=512, n=2000, k=20, r=60, c=100, tol=1e-8)
CFG3 = dict(m=1_000_000, n=20_000, rank=200, k=50, r=150, c=200, tol=1e-8)
CFG4 = dict(side=1024, n=8192, k=64, r=192, c=256, tol=1e-8)


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
                  rows=None, dtype=None):
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
    at = torch.empty((n, r1 - r0), dtype=dt if dtype is None else dtype, device=device)
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


def config2(seed=0, side=512, n=2000, noise_var=1e-4, dtype=None):
    """Host (numpy, F-order) copy of ``config2_torch`` generated on the CPU."""
    at = config2_torch(seed, side, n, noise_var, device="cpu", dtype=dtype)
    return np.asfortranarray(at.numpy().T)


def config4_torch(seed=0, side=1024, n=8192, noise_var=1e-4, device="cpu", rows=None):
    """BASELINE config 4: the config-2 generator on a side x side grid
    (1024 -> m = 1,048,576), n = 8192, STORED float32 (each 4096-row chunk is
    generated in float64 and rounded once)."""
    import torch

    return config2_torch(seed, side, n, noise_var, device=device, rows=rows, dtype=torch.float32)


def config4(seed=0, side=64, n=300, noise_var=1e-4):
    """Host float32 (F-order) config-4 proxy made on the CPU."""
    return np.asfortranarray(config4_torch(seed, side, n, noise_var, device="cpu").numpy().T)


def _chunk_gen(device, seed, c, salt):
    import torch

    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1000003 + c * 7919 + salt) % (2 ** 62))
    return g


def config3_torch(seed=0, m=1_000_000, n=20_000, rank=200, noise_var=1e-6, device="cpu",
                  rows=None, chunk=NOISE_CHUNK):
    """BASELINE config 3 rows [r0, r1) as a column-major float64 torch tensor
    (storage (n, r1 - r0), like ``config2_torch``); identical for any row
    partition of the same (seed, m, n, device type)."""
    import torch

    dt = torch.float64
    r0, r1 = (0, m) if rows is None else (int(rows[0]), int(rows[1]))
    nchunk = (m + chunk - 1) // chunk
    # V: Haar n x rank (replicated on every rank)
    gv = _chunk_gen(device, seed, 0, 11)
    v = torch.linalg.qr(torch.randn((n, rank), generator=gv, dtype=dt, device=device))[0]
    sig = torch.arange(1, rank + 1, dtype=dt, device=device) ** -1.5
    vs = (v * sig).T.contiguous()  # rank x n: diag(sigma) V^T

    def gauss(c):
        c0, c1 = c * chunk, min(m, (c + 1) * chunk)
        return torch.randn((c1 - c0, rank), generator=_chunk_gen(device, seed, c, 5), dtype=dt,
                           device=device)

    # R of the positive-diagonal QR of G = [G_0; G_1; ...]: Cholesky of sum G_c^T G_c
    gram = torch.zeros((rank, rank), dtype=dt, device=device)
    for c in range(nchunk):
        gc = gauss(c)
        gram += gc.T @ gc
    rf = torch.linalg.cholesky(gram, upper=True)
    sd = math.sqrt(noise_var)
    at = torch.empty((n, r1 - r0), dtype=dt, device=device)
    for c in range(r0 // chunk, (r1 + chunk - 1) // chunk):
        c0, c1 = c * chunk, min(m, (c + 1) * chunk)
        uc = torch.linalg.solve_triangular(rf, gauss(c), upper=True, left=False)  # G_c R^-1
        blk = (uc @ vs).T.contiguous()  # n x chunk
        blk.add_(torch.randn((n, c1 - c0), generator=_chunk_gen(device, seed, c, 3), dtype=dt,
                             device=device), alpha=sd)
        lo, hi = max(c0, r0), min(c1, r1)
        at[:, lo - r0:hi - r0].copy_(blk[:, lo - c0:hi - c0])
        del blk, uc
    return at


CFG5 = dict(m=4_000_000, n=50_000, rank=100, k=32, r=96, c=128, tol=1e-8)


def config5_host(seed=0, m=4_000_000, n=50_000, rank=100, noise_var=1e-5, rows=None,
                 device="cuda", chunk=NOISE_CHUNK):
    """BASELINE config 5: A = U diag(exp(-i/20)) V^T + N(0, 1e-5), rank 100,
    STORED float32 in page-locked HOST memory (800 GB at full size; the
    out-of-core workload), rows [r0, r1) of it as a pinned torch tensor with
    storage (n, r1 - r0) -- column-major rows, like ``config2_torch``.
    Generated block by block from the seed: each 4096-row chunk is made on
    `device` (the same per-chunk construction as ``config3_torch``: Haar U
    = G R^-1 with R from the Gram summed over all chunks, Haar V replicated),
    rounded to float32 once and copied into the host block, so host memory
    never holds more than the result and any row partition yields the same
    matrix."""
    import torch

    dt = torch.float64
    r0, r1 = (0, m) if rows is None else (int(rows[0]), int(rows[1]))
    nchunk = (m + chunk - 1) // chunk
    gv = _chunk_gen(device, seed, 0, 11)
    v = torch.linalg.qr(torch.randn((n, rank), generator=gv, dtype=dt, device=device))[0]
    sig = torch.exp(-torch.arange(rank, dtype=dt, device=device) / 20.0)
    vs = (v * sig).T.contiguous()  # rank x n
    del v

    def gauss(c):
        c0, c1 = c * chunk, min(m, (c + 1) * chunk)
        return torch.randn((c1 - c0, rank), generator=_chunk_gen(device, seed, c, 5), dtype=dt,
                           device=device)

    gram = torch.zeros((rank, rank), dtype=dt, device=device)
    for c in range(nchunk):
        gc = gauss(c)
        gram += gc.T @ gc
    rf = torch.linalg.cholesky(gram, upper=True)
    sd = math.sqrt(noise_var)
    host = torch.empty((n, r1 - r0), dtype=torch.float32, pin_memory=True)
    for c in range(r0 // chunk, (r1 + chunk - 1) // chunk):
        c0, c1 = c * chunk, min(m, (c + 1) * chunk)
        uc = torch.linalg.solve_triangular(rf, gauss(c), upper=True, left=False)
        blk = (uc @ vs).T.contiguous()  # n x chunk
        blk.add_(torch.randn((n, c1 - c0), generator=_chunk_gen(device, seed, c, 3), dtype=dt,
                             device=device), alpha=sd)
        lo, hi = max(c0, r0), min(c1, r1)
        host[:, lo - r0:hi - r0].copy_(blk[:, lo - c0:hi - c0].to(torch.float32))
        del blk, uc
    if str(device).startswith("cuda"):
        torch.cuda.synchronize(device)
    return host


def config3(seed=0, m=20_000, n=2_000, rank=200, noise_var=1e-6):
    """Host (numpy, F-order) copy of a ``config3_torch`` proxy made on the CPU."""
    at = config3_torch(seed, m, n, rank, noise_var, device="cpu")
    return np.asfortranarray(at.numpy().T)
