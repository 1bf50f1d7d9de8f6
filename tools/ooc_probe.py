"""One-pass incremental POD over a PODM file of the config-2 matrix (4.2 GB,
t column blocks): prefetching stream vs serial (POD_OOC_SERIAL=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads
t = int(sys.argv[1]) if len(sys.argv) > 1 else 8
path = "/tmp/cfg2.podm"
if not os.path.exists(path):
    at = workloads.config2_torch(7, 512, 2000, device=torch.device("cuda", 0))
    a = np.asfortranarray(at.cpu().numpy().T)
    del at
    pod.write_matrix(path, a)
    del a
cfg = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with pod.BlockReader(path, t) as rd:
        f, tr = pod.incremental_pod(rd, cfg)
    torch.cuda.synchronize()
    print(f"run {i}: {time.perf_counter() - t0:.3f} s  blocks {t}  rounds {len(tr)}  sigma0 {f.sigma[0]:.6f}")
t0 = time.perf_counter()
with open(path, "rb") as fh:
    while fh.read(1 << 28):
        pass
print(f"plain file read of {os.path.getsize(path) / 1e9:.2f} GB: {time.perf_counter() - t0:.3f} s")
