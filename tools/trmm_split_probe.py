"""Triangular apply Q = W R^-1 (R^-1 upper triangular): one m x l x l NN GEMM
against column-split calls that skip the zero part of R^-1 (columns [c0, c1)
need only K rows [0, c1)).  argv: m l [splits...] (default config-3/4 shapes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1905_05107_b200.device import ColMat, dptr, get_ctx

ctx = get_ctx(); dev = ctx.device


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(m, l, splits_list):
    W = ColMat(torch.randn((l, m), dtype=torch.float64, device=dev), m)
    Q = ColMat.zeros(m, l, dev)
    Q2 = ColMat.zeros(m, l, dev)
    T = torch.triu(torch.randn((l, l), dtype=torch.float64, device=dev).t()).t().contiguous()
    # col-major l x l upper triangular: element (i, j) at j * l + i, zero for i > j
    Tc = torch.triu(torch.randn((l, l), dtype=torch.float64, device=dev))  # row-major (i, j)
    T = Tc.t().contiguous().reshape(-1)  # col-major storage
    full = timeit(lambda: ctx.nn(l, l, 1.0, W, dptr(T), l, Q))
    print(f"m={m} l={l}: full {full:.3f} ms")
    for splits in splits_list:
        bounds = [0] + list(splits) + [l]

        def split():
            for c0, c1 in zip(bounds[:-1], bounds[1:]):
                ctx.nn(c1, c1 - c0, 1.0, W.cols(0, c1), dptr(T, c0 * l), l, Q2.cols(c0, c1))
        t = timeit(split)
        err = (Q2.t - Q.t).abs().max().item()
        print(f"  split {splits}: {t:.3f} ms  max|diff| {err:.2e}")


if __name__ == "__main__":
    if len(sys.argv) > 2:
        m, l = int(sys.argv[1]), int(sys.argv[2])
        run(m, l, [tuple(int(x) for x in s.split(",")) for s in sys.argv[3:]])
    else:
        run(1000000, 150, [(80,), (72,), (64,), (48, 96), (40, 80, 120)])
        run(1048576, 192, [(96,), (80,), (64, 128), (80, 160), (48, 96, 144)])
        run(262144, 60, [(32,), (24,), (16, 32, 48)])
