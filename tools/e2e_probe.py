"""Where the end-to-end (host buffers) time of a cfg2 run goes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads, engine, device
dev = torch.device("cuda", 0)
at = workloads.config2_torch(7, 512, 2000, device=dev)
n, m = at.shape
host = torch.empty((n, m), dtype=torch.float64).pin_memory()
host.copy_(at)
a_host = host.numpy().T
del at
torch.cuda.empty_cache()
cfg = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7)
marks = {}
def wrap(mod, name):
    orig = getattr(mod, name)
    def w(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out = orig(*a, **k)
        torch.cuda.synchronize(); marks[name] = marks.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
        return out
    setattr(mod, name, w)
import paper_1905_05107_b200.isma as im
wrap(device, "to_device_colmajor")
wrap(engine, "get_engine")
wrap(engine.IsmaEngine, "run")
wrap(engine.IsmaEngine, "result")
n_eng = [0]
orig_init = engine.IsmaEngine.__init__
def cnt(self, *a, **k):
    n_eng[0] += 1
    orig_init(self, *a, **k)
engine.IsmaEngine.__init__ = cnt
for i in range(int(os.environ.get("E2E_CALLS", "3"))):
    marks.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    f, tr = pod.isma_run(a_host, cfg)
    torch.cuda.synchronize()
    print(f"call {i}: {1e3*(time.perf_counter()-t0):.1f} ms  engines created so far {n_eng[0]}  " + str({k: round(v, 1) for k, v in marks.items()}))
