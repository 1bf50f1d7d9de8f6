"""CPU pins of the summation orders the GPU draw reproduces (exact_sums.cu):
numpy's einsum("ij,ij->j") lane order (also chained across 8-aligned row
segments, as the row-sharded norm pass hands it from rank to rank) and the
pairwise order of ndarray.sum().  The GPU kernels are checked against numpy
itself in tests/test_gpu_exact_draw.py; these pin the restatement they follow."""

import numpy as np
import pytest

from oracle import isma_oracle as orc
from paper_1905_05107_b200.parallel import ROW_ALIGN, shard_rows


@pytest.mark.parametrize("m", [1, 7, 8, 9, 63, 64, 65, 1000, 4097, 20003])
def test_einsum_lane_order_is_numpys(m):
    rng = np.random.default_rng(m)
    a = np.asfortranarray(rng.standard_normal((m, 5)) * rng.uniform(0.01, 100.0, 5))
    m8 = m - m % 8
    st = orc.einsum_lane_state(a[:m8])
    got = orc.einsum_lane_finish(a[m8:], st)
    assert np.array_equal(got, np.einsum("ij,ij->j", a, a))


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_chained_segments_equal_one_pass(world):
    """Shard boundaries from shard_rows are 8-aligned, and handing the lane
    state through the shards reproduces numpy's norms bit for bit."""
    rng = np.random.default_rng(world)
    m = 10007
    a = np.asfortranarray(rng.standard_normal((m, 7)))
    st = None
    for r in range(world):
        r0, r1 = shard_rows(m, world, r)
        if r < world - 1:
            assert r1 % ROW_ALIGN == 0 and (r1 - r0) % 8 == 0
            st = orc.einsum_lane_state(a[r0:r1], st)
        else:
            seg = a[r0:r1]
            body = seg.shape[0] - seg.shape[0] % 8
            st = orc.einsum_lane_state(seg[:body], st)
            got = orc.einsum_lane_finish(seg[body:], st)
    assert np.array_equal(got, np.einsum("ij,ij->j", a, a))


@pytest.mark.parametrize("n", list(range(1, 140)) + [255, 256, 257, 1000, 2000, 8191, 20000])
def test_pairwise_sum_is_numpys(n):
    rng = np.random.default_rng(n)
    x = rng.random(n) * rng.uniform(1e-3, 1e3)
    assert orc.pairwise_sum(x) == x.sum()


def test_shard_rows_cover_and_align():
    for m in (1, 7, 100, 262144, 1000003):
        for world in (1, 2, 3, 8):
            b = [shard_rows(m, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == m
            for (x0, x1), (y0, _) in zip(b, b[1:]):
                assert x1 == y0 and x1 % ROW_ALIGN == 0
