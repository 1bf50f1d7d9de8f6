"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares; host-side parameter validation mirrors the reference; the
product path refuses to run without a GPU (no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "podsketch_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(pod_\w+)\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    # and the Python binding declares a signature for each
    assert set(syms) <= set(_lib.SIGNATURES)


def test_abi_queries_without_gpu():
    lib = _lib.load()
    assert lib.pod_abi_version() == 1
    assert lib.pod_gemm_tn_ws_bytes(262144, 100, 100) > 0
    assert lib.pod_draw_ws_bytes(2000) >= 2000 * 12
    assert lib.pod_small_ws_bytes(384) >= 384 * 384 * 8


def test_sass_is_sm100a_with_dmma():
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "DMMA.8x8x4" in sass


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pod.DeviceError):
        pod.isma_run(np.eye(4), pod.IsmaConfig(k=1))


# --- reference test_isma.py:39-87 (config validation is host logic) -------
def test_config_defaults():
    cfg = pod.IsmaConfig(k=4)
    assert cfg.r == 12 and cfg.tau == 0.99 and cfg.strategy == "unf"
    assert cfg.criterion == "modes" and cfg.rows is False and cfg.finalize is True


@pytest.mark.parametrize("kwargs", [
    {"k": 0}, {"k": 3, "r": 2}, {"k": 2, "epsilon": 0.0}, {"k": 2, "delta": 1.0},
    {"k": 2, "tau": -0.1}, {"k": 2, "tau": 1.5}, {"k": 2, "strategy": "foo"},
    {"k": 2, "criterion": "bar"}, {"k": 2, "strategy": "ls", "rows": False},
    {"k": 2, "strategy": "l2n", "rows": True}, {"k": 2, "c": 0}, {"k": 2, "w": 0}])
def test_config_rejects_bad_parameters(kwargs):
    with pytest.raises(pod.ParameterError):
        pod.IsmaConfig(**kwargs)


def test_budgets():
    assert pod.ltsvd_sample_count(10, 0.7, 0.6) == 746
    cfg = pod.IsmaConfig(k=4, c=17)
    assert cfg.column_budget() == 17


def test_distribution_invariants():
    d = pod.Distribution(np.array([7, 3, 9]), np.array([0.3, 0.2, 0.5]))
    np.testing.assert_array_equal(d.indices, [3, 7, 9])
    np.testing.assert_allclose(d.weights, [0.2, 0.3, 0.5])
    with pytest.raises(pod.DegenerateDistributionError):
        pod.Distribution.from_weights([0, 1], [0.0, 0.0])
    with pytest.raises(pod.ParameterError):
        pod.Distribution(np.array([0, 0]), np.array([0.5, 0.5]))


def test_truncated_factor_invariants():
    with pytest.raises(pod.ParameterError):
        pod.TruncatedFactor(np.eye(3)[:, :2], np.array([1.0, 2.0]))
    f = pod.TruncatedFactor(np.eye(3)[:, :2], np.array([2.0, 1.0]))
    assert f.truncate(1).nmodes == 1
