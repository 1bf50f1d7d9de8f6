"""ctypes binding of the C ABI (include/podsketch_b200.h).

The library is built in-tree (``paper_1905_05107_b200/libpodsketch_b200.so``,
see ``__graft_entry__.build``).  There is no fallback: if the library or a
CUDA device is missing, every entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (
    DegenerateDistributionError,
    DeviceError,
    FormatError,
    ParameterError,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
# POD_LIB_PATH: an alternative build of the same library (A/B measurements only)
LIB_PATH = os.environ.get("POD_LIB_PATH") or os.path.join(_HERE, "libpodsketch_b200.so")

POD_OK, POD_EPARAM, POD_EFORMAT, POD_EDEGENERATE, POD_ENOCONVERGE, POD_ECUDA, POD_ENCCL = (
    0, 2, 3, 4, 5, 6, 7)

_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_f64 = ctypes.c_double
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t

# name -> (restype, argtypes)
SIGNATURES = {
    "pod_abi_version": (_i32, []),
    "pod_last_error": (ctypes.c_char_p, []),
    "pod_colnorms2_f64": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "pod_colnorms2": (_i32, [_i32, _vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "pod_colnorms2_chain": (_i32, [_i32, _vp, _i64, _i64, _i64, _vp, _vp, _i32, _vp, _vp, _vp]),
    "pod_tc_tn_ws_bytes": (_sz, [_i64, _i64, _i64]),
    "pod_gemm_tn_tf32x3": (_i32, [_i64, _i64, _i64, _f64, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp,
                                  _vp, _i64, _vp, _sz, _vp]),
    "pod_split_tf32": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "pod_draw_ws_bytes": (_sz, [_i64]),
    "pod_draw_exact_ws_bytes": (_sz, [_i64]),
    "pod_draw_exact": (_i32, [_i32, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _sz, _vp,
                              _f64, _vp, _vp]),
    "pod_draw": (_i32, [_i32, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _sz, _vp, _f64,
                        _vp, _vp]),
    "pod_rownorms2": (_i32, [_i32, _vp, _i64, _i64, _i64, _vp, _f64, _vp, _vp, _vp]),
    "pod_gather_scale_rows": (_i32, [_i32, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _f64, _i64, _vp,
                                     _vp, _i64, _vp]),
    "pod_resid_ws_bytes": (_sz, [_i64, _i64]),
    "pod_resid_colnorms2": (_i32, [_i32, _i64, _i64, _vp, _i64, _vp, _vp, _i64, _i64, _vp, _i64,
                                   _vp, _vp, _sz, _vp]),
    "pod_wedin_ws_bytes": (_sz, [_i64, _i64, _i64]),
    "pod_wedin_residuals": (_i32, [_i32, _vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp,
                                   _i64, _vp, _vp, _sz, _vp]),
    "pod_gemm_nn_dots_ws_bytes": (_sz, [_i64]),
    "pod_gemm_nn_dots": (_i32, [_i64, _i64, _i64, _f64, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _vp,
                                _vp, _sz, _vp, _vp]),
    "pod_gemm_nn_gram_ok": (_i32, [_i64, _i64]),
    "pod_gemm_nn_gram_ws_bytes": (_sz, [_i64, _i64]),
    "pod_gemm_nn_gram": (_i32, [_i64, _i64, _i64, _f64, _vp, _i64, _vp, _i64, _f64, _vp, _i64,
                                _vp, _i64, _vp, _i64, _vp, _sz, _vp, _vp]),
    "pod_gemm_tn_ws_bytes": (_sz, [_i64, _i64, _i64]),
    "pod_gemm_tn_f64": (_i32, [_i64, _i64, _i64, _f64, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _i64,
                               _vp, _sz, _vp, _vp]),
    "pod_gemm_nn_f64": (_i32, [_i64, _i64, _i64, _f64, _vp, _i64, _vp, _vp, _i64, _f64, _vp, _i64,
                               _vp, _i64, _vp, _vp]),
    "pod_gemm_tn": (_i32, [_i32, _i32, _i64, _i64, _i64, _f64, _vp, _i64, _vp, _vp, _i64, _vp, _vp,
                           _i64, _vp, _sz, _vp, _vp]),
    "pod_gemm_nn": (_i32, [_i32, _i64, _i64, _i64, _f64, _vp, _i64, _vp, _vp, _i64, _f64, _vp,
                           _i64, _vp, _i64, _vp, _vp]),
    "pod_set_grid_cap": (_i32, [_i32]),
    "pod_gather_cols": (_i32, [_i32, _vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp]),
    "pod_gather_scale_cols": (_i32, [_i32, _vp, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _vp]),
    "pod_host_register": (_i32, [_vp, _sz]),
    "pod_host_unregister": (_i32, [_vp]),
    "pod_small_ws_bytes": (_sz, [_i64]),
    "pod_svd_small_ws_bytes": (_sz, [_i64, _i64, _i32]),
    "pod_gram_eigh_max_g": (_i64, []),
    "pod_gram_eigh": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "pod_cholqr_factor": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _sz, _vp,
                                 _vp, _i32, _vp]),
    "pod_cholqr_factor2": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp,
                                  _vp, _sz, _vp, _vp, _i32, _vp]),
    "pod_merge_core": (_i32, [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _vp, _i64,
                              _i64, _vp, _vp, _vp, _sz, _vp]),
    "pod_merge_core_gatable": (_i32, [_i64, _i64]),
    "pod_merge_core_gated": (_i32, [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _vp,
                                    _i64, _i64, _vp, _vp, _vp, _vp]),
    "pod_svd_small": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "pod_small_gemm": (_i32, [_i64, _i64, _i64, _f64, _vp, _i64, _i32, _vp, _i64, _f64, _vp, _i64,
                              _vp, _vp]),
    "pod_small_copy": (_i32, [_i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp]),
    "pod_maxabs": (_i32, [_vp, _i64, _i64, _i64, _f64, _vp, _vp, _vp]),
    "pod_colwise_ws_bytes": (_sz, [_i64, _i64]),
    "pod_fix_signs": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _vp, _sz, _vp]),
    "pod_colargmax": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _sz, _vp]),
    "pod_scale_cols": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp]),
    "pod_coldots": (_i32, [_vp, _i64, _vp, _i64, _i64, _i64, _i64, _i32, _vp, _vp, _sz, _vp]),
}

_LIB = None


def load():
    """Load the in-tree library (once) and declare every ABI signature."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"CUDA library not built: {LIB_PATH} missing (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


_EXC = {
    POD_EPARAM: ParameterError,
    POD_EFORMAT: FormatError,
    POD_EDEGENERATE: DegenerateDistributionError,
}


def check(status, what=""):
    if status == POD_OK:
        return
    msg = (_LIB.pod_last_error() or b"").decode(errors="replace") if _LIB else ""
    exc = _EXC.get(status)
    if exc is not None:
        raise exc(msg or what)
    if status == POD_ENOCONVERGE:
        import scipy.linalg as sla

        raise sla.LinAlgError(msg or what)
    raise DeviceError(f"{what}: {msg} (status {status})")


def call(name, *args):
    lib = load()
    check(getattr(lib, name)(*args), name)
