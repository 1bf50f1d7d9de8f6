"""Phase split of the merge E-SVD (block Jacobi on a cluster) at config-2
size (E = 120 x 120) from the POD_BJ_TIMING build: clock64 deltas of CTA 0,
thread 0, summed over a block_merge call.  Usage (GPU box):

  nvcc ... -DPOD_BJ_TIMING -shared -o /tmp/libt.so csrc/*.cu
  POD_LIB=/tmp/libt.so python tools/bj_phase_probe.py
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_05107_b200 import _lib  # noqa: E402

if os.environ.get("POD_LIB"):
    _lib.LIB_PATH = os.environ["POD_LIB"]
import paper_1905_05107_b200 as pod  # noqa: E402
from paper_1905_05107_b200 import workloads  # noqa: E402

lib = _lib.load()
fn = lib.pod_debug_bj_phase
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 16)()

at = workloads.config2_torch(7, 128, 2000, device="cpu")  # m = 16384
a = at.numpy().T
u1, s1, _ = np.linalg.svd(a[:, :1000], full_matrices=False)
u2, s2, _ = np.linalg.svd(a[:, 1000:], full_matrices=False)
f1 = pod.TruncatedFactor(u1[:, :60], s1[:60])
f2 = pod.TruncatedFactor(u2[:, :60], s2[:60])
pod.block_merge(f1, f2, 60)
torch.cuda.synchronize()
fn(buf, 1)
reps = 20
t0 = time.perf_counter()
for _ in range(reps):
    pod.block_merge(f1, f2, 60)
torch.cuda.synchronize()
el = (time.perf_counter() - t0) / reps
fn(buf, 0)
names = ["-", "norms", "intra", "inter_step", "flag+fence+sync", "cluster_barrier",
         "bulk_issue", "mbar_wait", "sub:load+dot", "sub:shuffle", "sub:rot+apply", "sub:sync"]
tot = sum(buf[i] for i in range(1, 8))
print(f"block_merge wall {el * 1e3:.3f} ms per call (timing build)")
for i in range(1, 12):
    v = buf[i] / reps
    print(f"{names[i]:18s} {v:12.0f} cycles/call  {100.0 * buf[i] / max(tot, 1):5.1f}%")
