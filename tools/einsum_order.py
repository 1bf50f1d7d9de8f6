"""Pin numpy's einsum("ij,ij->j") and ndarray.sum() summation orders.

Restates the two orders exact_sums.cu reproduces (SSE2 2-lane einsum with
separate mul/add roundings; pairwise sum with 8 accumulators per <=128 block)
in plain Python and checks them bit-for-bit against numpy on random inputs.
Prints "ok" or the first mismatch.  (CPU only; part of the test suite via
tests/test_cpu_exact_order.py.)
"""

import sys

import numpy as np


def einsum_order_col(x):
    a0 = a1 = 0.0
    m = len(x)
    m8 = m - m % 8
    for i in range(0, m8, 8):
        a0 = x[i + 6] * x[i + 6] + a0
        a1 = x[i + 7] * x[i + 7] + a1
        a0 = x[i + 4] * x[i + 4] + a0
        a1 = x[i + 5] * x[i + 5] + a1
        a0 = x[i + 2] * x[i + 2] + a0
        a1 = x[i + 3] * x[i + 3] + a1
        a0 = x[i] * x[i] + a0
        a1 = x[i + 1] * x[i + 1] + a1
    for i in range(m8, m, 2):
        a0 = x[i] * x[i] + a0
        a1 = (x[i + 1] * x[i + 1] if i + 1 < m else 0.0) + a1
    return a0 + a1


def main():
    rng = np.random.default_rng(11)
    for m in [1, 3, 7, 8, 9, 31, 100, 1001, 4099, 8192, 20000]:
        a = np.asfortranarray(rng.standard_normal((m, 3)) * rng.uniform(0.1, 10, 3))
        ref = np.einsum("ij,ij->j", a, a)
        got = [einsum_order_col([float(v) for v in a[:, j]]) for j in range(3)]
        if list(ref) != got:
            print("mismatch", m, ref, got)
            return 1
    print("ok")
    return 0


if __name__ == "__main__":
    sys.exit(main())
