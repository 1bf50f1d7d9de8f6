"""Per-phase cycle breakdown of the block-Jacobi solver (timing build)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_05107_b200 import _lib
_lib.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpod_timing.so")
import numpy as np, torch
from paper_1905_05107_b200.device import get_ctx, dptr
ctx = get_ctx(); dev = ctx.device
lib = _lib.load()
buf = (ctypes.c_ulonglong * 16)()
for n in (120, 300):
    E = torch.as_tensor((np.random.default_rng(0).standard_normal((n, n)) * np.exp(-np.arange(n) / 8.0)).reshape(-1), device=dev)
    s = torch.empty(n, dtype=torch.float64, device=dev)
    ctx.svd_small(dptr(E), n, n, n, None, 1, s, None, 1); torch.cuda.synchronize()
    lib.pod_debug_bj_phase(buf, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.svd_small(dptr(E), n, n, n, None, 1, s, None, 1)
    e1.record(); torch.cuda.synchronize()
    sweeps = ctx.read_info(1)[0]
    lib.pod_debug_bj_phase(buf, 1)
    names = ["-", "norms", "intra", "inter", "flags+sync", "cluster barrier", "issue copies", "mbar wait"]
    tot = sum(buf[i] for i in range(1, 8))
    print(f"n={n} sweeps={sweeps} {e0.elapsed_time(e1)*1e3:.0f} us total cycles {tot}: " + ", ".join(f"{names[i]}={buf[i]/sweeps:.0f}" for i in range(1, 8)) + "  (per sweep)")
    sub = sweeps * (2 * 8 - 1) * ((n + 15) // 16)
    print("   per inter sub-round (CTA 0, thread 0): " + ", ".join(f"{nm}={buf[i]/sub:.0f}" for i, nm in ((8, "loads+dot"), (9, "shuffles"), (10, "rotate"), (11, "syncthreads"))))
