"""BASELINE config 5 (out of core) proxy on one B200: the fp32 matrix lives in
page-locked host memory (generated block by block), isma_run streams it
(residency="host").  Reports the run time, the pinned H2D copy bandwidth
(cudaMemcpy of 1 GiB, the PCIe roofline of the streamed passes) and the
per-kernel breakdown of one profiled run.

    python tools/config5_probe.py [--m 4000000] [--n 5000]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_05107_b200 as pod  # noqa: E402
from paper_1905_05107_b200 import isma as isma_mod, workloads  # noqa: E402


def h2d_gbs(dev):
    h = torch.empty(1 << 28, dtype=torch.float32, pin_memory=True)
    d = torch.empty(1 << 28, dtype=torch.float32, device=dev)
    d.copy_(h)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return 5 * h.numel() * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4_000_000)
    ap.add_argument("--n", type=int, default=5000)
    ap.add_argument("--runs", type=int, default=2)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    out = {"m": args.m, "n": args.n, "h2d_pinned_gbs": h2d_gbs(dev)}
    t0 = time.perf_counter()
    host = workloads.config5_host(seed=0, m=args.m, n=args.n, device=dev)
    out["generation_s"] = time.perf_counter() - t0
    out["host_gb"] = host.numel() * 4 / 1e9
    w = workloads.CFG5
    cfg = pod.IsmaConfig(k=w["k"], r=w["r"], c=w["c"], tau=1 - w["tol"], strategy="l2n", seed=7)
    times = []
    for _ in range(args.runs):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        f, tr = pod.isma_run(host.T, cfg, residency="host")
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t1)
    out.update(run_s=times, rounds=len(tr), sigma_top3=[float(x) for x in f.sigma[:3]],
               remaining=tr[-1].remaining)
    # PCIe passes: norm pass + finalize read A once each, every round copies
    # its sampled columns: bytes over the bus per run
    gathered = sum(t.columns_sampled for t in tr) * args.m * 4
    out["pcie_bytes"] = 2 * out["host_gb"] * 1e9 + gathered
    out["pcie_gbs_effective"] = out["pcie_bytes"] / min(times) / 1e9
    from paper_1905_05107_b200.device import KernelProfile, get_ctx

    class NoRollback:
        def __init__(self, seed):
            self.g = np.random.default_rng(seed)

        def random(self, k):
            return self.g.random(k)

    ctx = get_ctx(dev)
    prof = KernelProfile()
    ctx.prof = prof
    pod.isma_run(host.T, cfg, rng=NoRollback(7), residency="host")
    ctx.prof = None
    kern = prof.summary()
    out["kernels"] = {k: {"ms": v["ms"], "calls": v["calls"],
                          "gbs": v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["bytes"] else None}
                      for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["ms"])[:12]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
