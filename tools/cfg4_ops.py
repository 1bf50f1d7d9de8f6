"""Per-op time of one config-4 run (1M x 8192 stored fp32, k=64, r=192,
c=256), eager with CUDA events around every launch (bench._profile_run),
for precision fp64 / mixed (argv[1])."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads
from paper_1905_05107_b200.device import ColMat
import bench

prec = sys.argv[1] if len(sys.argv) > 1 else "mixed"
dev = torch.device("cuda", 0)
w = workloads.CFG4
at = workloads.config4_torch(7, w["side"], w["n"], device=dev)
A = ColMat(at, w["side"] ** 2)
cfg = pod.IsmaConfig(k=w["k"], r=w["r"], c=w["c"], tau=1 - w["tol"], strategy="l2n", seed=7)
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    f, tr = pod.isma_run(A, cfg, precision=prec)
    torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"{prec}: run {t1 - t0:.3f} s, rounds {len(tr)}")
kern = bench._profile_run(pod, A, cfg, {"precision": prec})
tot = sum(v["ms"] for v in kern.values())
print(f"profiled (serialised) total {tot:.1f} ms")
for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["ms"])[:22]:
    tf = v["flops"] / (v["ms"] / 1e3) / 1e12 if v["flops"] else 0.0
    print(f"  {k:28s} {v['ms']:9.2f} ms  {v['calls']:5d} calls  {v['ms'] / v['calls']:8.3f} ms/call  {tf:6.1f} TF/s")
