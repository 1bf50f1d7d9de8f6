"""Where the config-2 e2e time goes: pinned H2D alone, the device-resident
run alone, the public call on the pinned host matrix, and its pieces."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_05107_b200 as pod  # noqa: E402
from paper_1905_05107_b200 import workloads  # noqa: E402
from paper_1905_05107_b200.device import to_device_colmajor  # noqa: E402

dev = torch.device("cuda", 0)
at = workloads.config2_torch(7, 512, 2000, device="cpu")  # (n, m) rows = columns
m = at.shape[1]
host = at.pin_memory()
a = host.numpy().T
cfg = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7)


def t(fn, reps=4):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
    return min(out[1:]), out


print("h2d to_device_colmajor", t(lambda: to_device_colmajor(a, dev)))
buf = torch.empty_like(host, device=dev)
print("h2d copy_ into fixed buffer", t(lambda: buf.copy_(host, non_blocking=True)))
A = to_device_colmajor(a, dev)
print("device-resident run", t(lambda: pod.isma_run(A, cfg)))
print("e2e public call", t(lambda: pod.isma_run(a, cfg)))
f, tr = pod.isma_run(a, cfg)
print("rounds", len(tr))
