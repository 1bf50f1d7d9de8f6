"""Speculative merge core (engine.SPEC_CORE): how often the leak gate
(merge.py:73) fires, and the run time with the core speculative vs after the
leak check.  python tools/spec_probe.py [2|3|4] (config; env POD_SPEC_CORE)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads, engine
from paper_1905_05107_b200.device import ColMat
dev = torch.device("cuda", 0)
which = int(sys.argv[1]) if len(sys.argv) > 1 else 2
if which == 2:
    at, m, kw = workloads.config2_torch(7, 512, 2000, device=dev), 512 * 512, dict(k=20, r=60, c=100)
elif which == 3:
    at, m, kw = workloads.config3_torch(0, 1_000_000, 20_000, device=dev), 1_000_000, dict(k=50, r=150, c=200)
else:
    at, m, kw = workloads.config4_torch(7, 1024, 8192, device=dev), 1 << 20, dict(k=64, r=192, c=256)
A = ColMat(at, m)
cfg = pod.IsmaConfig(tau=1 - 1e-8, strategy="l2n", seed=7, **kw)
orig = engine.IsmaEngine.launch_round
fired, leaks = [], []
def probe(self, *a, **k):
    orig(self, *a, **k)
    if COUNT:
        torch.cuda.synchronize()
        fired.append(int(self.gates[engine.G_LEAK].item()))
        leaks.append(float(self.leak.item()))
engine.IsmaEngine.launch_round = probe
COUNT = True
f0, _ = pod.isma_run(A, cfg)
print(f"config {which} SPEC_CORE={engine.SPEC_CORE}: leak gate fired in {sum(fired)}/{len(fired)} "
      f"rounds: {''.join(map(str, fired))}")
print("  max|U1^T Q| per round:", " ".join(f"{x:.1e}" for x in leaks))
print("  sigma[:4]:", f0.sigma[:4].tolist())
COUNT = False
ts = []
for it in range(3):
    torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
    s0.record(); pod.isma_run(A, cfg); s1.record(); torch.cuda.synchronize()
    ts.append(s0.elapsed_time(s1))
print(f"  runs ms: {' '.join(f'{t:.2f}' for t in ts)}")
