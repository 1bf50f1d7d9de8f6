"""Fused one-pass Wedin residuals vs the two-pass NN + TN path at config-2 /
config-3-like shapes: device time (CUDA events) and achieved rates."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_05107_b200 import quality  # noqa: E402
from paper_1905_05107_b200.device import ColMat, get_ctx  # noqa: E402


def run(m, n, k, dtype, reps=5):
    ctx = get_ctx()
    dev = ctx.device
    g = torch.Generator(device=dev).manual_seed(1)
    at = torch.randn((n, m), dtype=dtype, device=dev, generator=g)
    A = ColMat(at, m)
    U = ColMat(torch.randn((k, m), dtype=torch.float64, device=dev, generator=g), m)
    V = ColMat(torch.randn((k, n), dtype=torch.float64, device=dev, generator=g), n)
    s = torch.linspace(5.0, 1.0, k, dtype=torch.float64, device=dev)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    import numpy as np
    sk = s.cpu().numpy()

    def fused():
        ctx.wedin(A, U, V, s, k, out)

    def two():
        quality._wedin_two_pass(ctx, A, U, V, sk, m, n, k)

    res = {}
    for name, fn in (("fused", fused), ("two_pass", two)):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        flops = 4.0 * m * n * k
        res[name] = {"ms": ms, "tflops": flops / ms / 1e9,
                     "a_gbs": at.element_size() * m * n / ms / 1e6}
    res["shape"] = {"m": m, "n": n, "k": k, "dtype": str(dtype)}
    print(json.dumps(res))
    del at


if __name__ == "__main__":
    run(262144, 2000, 20, torch.float64)
    run(262144, 2000, 50, torch.float64)
    run(1000000, 4000, 50, torch.float64)
    run(1048576, 8192, 64, torch.float32)
