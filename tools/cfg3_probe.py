"""Full-size BASELINE config 3 (1M x 20k fp64, 160 GB) or config 4 (config-2
generator at 1024^2 x 8192, stored fp32, 34 GB) on one B200: device
generation, timed isma_run, per-kernel breakdown.

    python tools/cfg3_probe.py [--config 3|4] [--m 1000000] [--n 20000] [--criterion modes]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_05107_b200 as pod  # noqa: E402
from paper_1905_05107_b200 import isma as isma_mod, workloads  # noqa: E402
from paper_1905_05107_b200.device import ColMat  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3, choices=[3, 4])
    ap.add_argument("--m", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--criterion", default="modes")
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--precision", default="fp64", choices=["fp64", "mixed"])
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    free, total = torch.cuda.mem_get_info(dev)
    print(f"mem free {free / 2**30:.1f} GiB of {total / 2**30:.1f} GiB", flush=True)
    t = time.perf_counter()
    if args.config == 3:
        args.m = args.m or 1_000_000
        args.n = args.n or 20_000
        at = workloads.config3_torch(0, args.m, args.n, device=dev)
        kw = dict(k=50, r=150, c=200)
    else:
        side = int(round((args.m or 1 << 20) ** 0.5))
        args.m, args.n = side * side, args.n or 8192
        at = workloads.config4_torch(7, side, args.n, device=dev)
        kw = dict(k=64, r=192, c=256)
    torch.cuda.synchronize()
    print(f"generated {args.m}x{args.n} {at.dtype} in {time.perf_counter() - t:.1f} s", flush=True)
    A = ColMat(at, args.m)
    cfg = pod.IsmaConfig(tau=1 - args.tol, strategy="l2n", criterion=args.criterion, seed=7, **kw)
    out = {}
    for i in range(args.runs):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f, tr = pod.isma_run(A, cfg, precision=args.precision)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        st = isma_mod.LAST_STATS
        print(f"run {i}: {ms / 1e3:.3f} s, rounds {len(tr)}, cols {sum(x.columns_sampled for x in tr)}"
              f", remaining {tr[-1].remaining}, sigma0 {f.sigma[0]:.6f}, "
              f"eigh sweeps {st.get('eigh_sweeps', [])[:3]}, merge sweeps "
              f"{st.get('merge_sweeps', [])[:3]}", flush=True)
        out = dict(seconds=ms / 1e3, rounds=len(tr), sigma=f.sigma[:10].tolist(),
                   min_cos=[float(np.min(x.cosines)) for x in tr[1:]][-5:])
    # one profiled eager (unpipelined) pass: per-kernel breakdown
    from paper_1905_05107_b200.device import KernelProfile, get_ctx

    class NoRollback:
        def __init__(self, seed):
            self.g = np.random.default_rng(seed)

        def random(self, k):
            return self.g.random(k)

    ctx = get_ctx(dev)
    prof = KernelProfile()
    ctx.prof = prof
    pod.isma_run(A, cfg, rng=NoRollback(7), precision=args.precision)
    if args.precision == "mixed":  # the same run in fp64: the mixed path's errors
        from parity_util import principal_angles_sin, sigma_relerr
        fm = f
        fd, _ = pod.isma_run(A, cfg)
        out["mixed_vs_fp64"] = {"sigma_rel_err": sigma_relerr(fm.sigma, fd.sigma),
                                "max_angle_rad": float(principal_angles_sin(fm.u, fd.u).max())}
    ctx.prof = None
    kern = prof.summary()
    print(json.dumps(out))
    tot = sum(v["ms"] for v in kern.values())
    print(f"profiled eager total {tot / 1e3:.3f} s")
    for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["ms"])[:25]:
        tf = v["flops"] / (v["ms"] / 1e3) / 1e12 if v["flops"] else 0.0
        gb = v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["bytes"] else 0.0
        print(f"{k:28s} calls {v['calls']:5d} ms {v['ms']:9.2f} ({100 * v['ms'] / tot:5.1f}%) "
              f"TF/s {tf:6.2f} GB/s {gb:7.0f}")
    print(f"mem peak {torch.cuda.max_memory_allocated(dev) / 2**30:.1f} GiB")


if __name__ == "__main__":
    main()
