"""BlockReader / PODM host logic (reference tests/test_ooc.py:29-129 semantics)."""

import io
import struct

import numpy as np
import pytest

import paper_1905_05107_b200 as pod
from paper_1905_05107_b200.podio import HEADER_BYTES


def _write(tmp_path, a, name="a.podm"):
    p = tmp_path / name
    pod.write_matrix(str(p), a)
    return str(p)


def test_ten_columns_in_four_blocks(tmp_path, rng):
    a = rng.standard_normal((5, 10))
    with pod.BlockReader(_write(tmp_path, a), 4) as rd:
        assert [rd.block_bounds(i) for i in range(4)] == [(0, 2), (2, 5), (5, 7), (7, 10)]


@pytest.mark.parametrize("n,t", [(7, 1), (7, 7), (100, 3), (13, 5)])
def test_blocks_partition_and_are_bit_exact(tmp_path, rng, n, t):
    a = rng.standard_normal((9, n))
    with pod.BlockReader(_write(tmp_path, a), t) as rd:
        parts = list(rd)
        assert rd.blocks_read == t
    np.testing.assert_array_equal(np.hstack(parts), a)


def test_block_index_and_count_checked(tmp_path, rng):
    p = _write(tmp_path, rng.standard_normal((4, 6)))
    with pod.BlockReader(p, 2) as rd:
        with pytest.raises(pod.ParameterError):
            rd.block_bounds(2)
        with pytest.raises(pod.ParameterError):
            rd.block_bounds(-1)
    for bad in (0, 7):
        with pytest.raises(pod.ParameterError):
            pod.BlockReader(p, bad)


def test_bad_magic_names_the_header_offset(tmp_path):
    p = tmp_path / "bad.podm"
    p.write_bytes(b"XXXX" + bytes(20))
    with pytest.raises(pod.FormatError, match="byte offset 0"):
        pod.BlockReader(str(p), 1)


def test_zero_row_header_rejected(tmp_path):
    p = tmp_path / "z.podm"
    p.write_bytes(struct.pack("<4sIQQ", b"PODM", 1, 0, 3))
    with pytest.raises(pod.FormatError, match="zero rows or columns"):
        pod.BlockReader(str(p), 1)


def test_truncated_payload_reports_byte_offset(tmp_path, rng):
    a = rng.standard_normal((6, 4))
    buf = io.BytesIO()
    pod.write_matrix(buf, a)
    raw = buf.getvalue()[:HEADER_BYTES + 6 * 8 * 3 + 5]
    rd = pod.BlockReader(io.BytesIO(raw), 4)
    for _ in range(3):
        rd.read_block()
    with pytest.raises(pod.FormatError, match="byte offset"):
        rd.read_block()


def test_borrowed_file_stays_open(tmp_path, rng):
    p = _write(tmp_path, rng.standard_normal((3, 3)))
    with open(p, "rb") as f:
        with pod.BlockReader(f, 1) as rd:
            rd.read_block()
        assert not f.closed


def test_pass_count():
    assert pod.pass_count("incremental", False, 9) == 1
    assert pod.pass_count("full", False, 4) == 5
    assert pod.pass_count("full", True, 4) == 13
    with pytest.raises(pod.ParameterError):
        pod.pass_count("full", False, -1)
    with pytest.raises(pod.ParameterError):
        pod.pass_count("bogus", False, 1)
