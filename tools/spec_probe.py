"""Speculative merge core (engine.SPEC_CORE): how often the leak gate
(merge.py:73) fires at config 2, and the per-round GPU time with the core
speculative vs after the leak check (run once per POD_SPEC_CORE setting)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads, engine
from paper_1905_05107_b200.device import ColMat
dev = torch.device("cuda", 0)
at = workloads.config2_torch(7, 512, 2000, device=dev)
A = ColMat(at, 512 * 512)
cfg = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7)
orig = engine.IsmaEngine.launch_round
fired, ev = [], []
def probe(self, *a, **k):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); orig(self, *a, **k); e1.record()
    ev.append((e0, e1))
    if COUNT:
        torch.cuda.synchronize()
        fired.append(int(self.gates[engine.G_LEAK].item()))
engine.IsmaEngine.launch_round = probe
COUNT = True
pod.isma_run(A, cfg)
print(f"SPEC_CORE={engine.SPEC_CORE}: leak gate fired in {sum(fired)}/{len(fired)} rounds")
COUNT = False
for it in range(4):
    ev.clear()
    torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
    s0.record(); pod.isma_run(A, cfg); s1.record(); torch.cuda.synchronize()
gpu = [a.elapsed_time(b) for a, b in ev]
print(f"run {s0.elapsed_time(s1):.2f} ms; {len(gpu)} rounds, round gpu ms mean {np.mean(gpu):.3f} "
      f"median {np.median(gpu):.3f}")
