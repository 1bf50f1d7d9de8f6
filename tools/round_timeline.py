"""Per-round GPU time vs host gaps of a graph-mode cfg2 run (CUDA events
around every round's graph replay)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads, engine
from paper_1905_05107_b200.device import ColMat
dev = torch.device("cuda", 0)
side = int(sys.argv[1]) if len(sys.argv) > 1 else 512
at = workloads.config2_torch(7, side, 2000, device=dev)
A = ColMat(at, side * side)
cfg = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7)
orig = engine.IsmaEngine.launch_round
ev = []
def timed(self, *a, **k):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    orig(self, *a, **k)
    e1.record()
    ev.append((e0, e1, t0, time.perf_counter()))
engine.IsmaEngine.launch_round = timed
for it in range(3):
    ev.clear()
    torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
    s0.record(); t0 = time.perf_counter()
    f, tr = pod.isma_run(A, cfg)
    s1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
total = s0.elapsed_time(s1)
gpu = [a.elapsed_time(b) for a, b, _, _ in ev]
first = s0.elapsed_time(ev[0][0])
last = ev[-1][1].elapsed_time(s1)
gaps = [ev[i][1].elapsed_time(ev[i + 1][0]) for i in range(len(ev) - 1)]
host = [(c - b) * 1e3 for _, _, b, c in ev]
print(f"total {total:.2f} ms wall {1e3*(t1-t0):.2f}; rounds {len(ev)}; before first round {first:.2f} ms; after last {last:.2f} ms")
print(f"round gpu ms: mean {np.mean(gpu):.3f} min {np.min(gpu):.3f} max {np.max(gpu):.3f}; gaps between rounds mean {np.mean(gaps):.3f} ms; host launch ms mean {np.mean(host):.3f}")

# tail breakdown: finalize / fix_signs / result / factor construction
import paper_1905_05107_b200.isma as im
from paper_1905_05107_b200 import matcore
marks = {}
def wrap(cls, name):
    orig_fn = getattr(cls, name)
    def w(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out = orig_fn(*a, **k)
        torch.cuda.synchronize(); marks[name] = marks.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
        return out
    setattr(cls, name, w)
wrap(engine.IsmaEngine, "finalize")
wrap(engine.IsmaEngine, "result")
wrap(engine.IsmaEngine, "norm_pass")
wrap(matcore.TruncatedFactor, "__init__")
f, tr = pod.isma_run(A, cfg)
print("tail ms:", {k: round(v, 2) for k, v in marks.items()})
