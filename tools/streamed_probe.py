"""Multi-pass streamed ISMA (A in page-locked host memory, read over PCIe):
config 2, and config 3's generator at a host-sized m, vs device-resident.
    python tools/streamed_probe.py [m3]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads
dev = torch.device("cuda", 0)


def host_copy(at):
    h = torch.empty(tuple(at.shape), dtype=at.dtype, pin_memory=True)
    h.copy_(at)
    return h.T  # (m, n) column-major view of pinned memory


def timed(a, cfg, residency, reps=2):
    best = 1e9
    for _ in range(reps + 1):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        f, tr = pod.isma_run(a, cfg, residency=residency)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best, len(tr), f.sigma[0]


at = workloads.config2_torch(7, 512, 2000, device=dev)
a2 = host_copy(at)
del at
cfg2 = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7)
for res in ("device", "host"):
    t, nr, s0 = timed(a2, cfg2, res)
    print(f"config 2 ({a2.shape[0]}x{a2.shape[1]} fp64, 4.2 GB) residency={res}: {t:.3f} s (incl. H2D for device), {nr} rounds, sigma0 {s0:.6f}", flush=True)
del a2
m3 = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
n3 = 20_000
h = torch.empty((n3, m3), dtype=torch.float64, pin_memory=True)
chunk = 100_000
for r0 in range(0, m3, chunk):
    r1 = min(m3, r0 + chunk)
    h[:, r0:r1].copy_(workloads.config3_torch(0, m3, n3, device=dev, rows=(r0, r1)))
torch.cuda.synchronize()
cfg3 = pod.IsmaConfig(k=50, r=150, c=200, tau=1 - 1e-8, strategy="l2n", seed=7)
t, nr, s0 = timed(h.T, cfg3, "host", reps=1)
print(f"config-3 generator {m3}x{n3} fp64 ({m3 * n3 * 8 / 1e9:.0f} GB) host-resident streamed: {t:.3f} s, {nr} rounds, sigma0 {s0:.6f}", flush=True)
