"""Per-phase cycle breakdown of one cluster-Jacobi step (timing build)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_05107_b200 import _lib
_lib.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpod_timing.so")
import numpy as np, torch
from paper_1905_05107_b200.device import get_ctx, dptr
ctx = get_ctx(); dev = ctx.device
lib = _lib.load()
buf = (ctypes.c_ulonglong * 8)()
for n in (60, 120):
    E = torch.as_tensor((np.random.default_rng(0).standard_normal((n, n)) * np.exp(-np.arange(n) / 8.0)).reshape(-1), device=dev)
    s = torch.empty(n, dtype=torch.float64, device=dev)
    ctx.svd_small(dptr(E), n, n, n, None, 1, s, None, 1); torch.cuda.synchronize()
    lib.pod_debug_cj_phase(buf, 1)
    ctx.svd_small(dptr(E), n, n, n, None, 1, s, None, 1); torch.cuda.synchronize()
    sweeps = ctx.read_info(1)[0]
    lib.pod_debug_cj_phase(buf, 1)
    steps = sweeps * (n - 1)
    names = ["-", "dots+st.async", "mbar wait", "sum+params+rotate", "nrm/flags", "syncthreads"]
    print(f"n={n} sweeps={sweeps} steps={steps}: " + ", ".join(f"{names[i]}={buf[i]/steps:.0f}" for i in range(1, 6)))
