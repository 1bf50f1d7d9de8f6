import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads
from paper_1905_05107_b200.device import ColMat, Ctx
dev = torch.device("cuda", 0)
at = workloads.config2_torch(7, 512, 2000, device=dev)
A = ColMat(at, 512 * 512)
cfg = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7)
orig = Ctx.cholqr_factor
log = []
def wrapped(self, G, ldg, l, nrows, Rinv, ldri, R, ldr, gate_in=None, gate_out=None, first_pass=0):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    orig(self, G, ldg, l, nrows, Rinv, ldri, R, ldr, gate_in=gate_in, gate_out=gate_out, first_pass=first_pass)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e6
    ran = gate_in is None or int(gate_in.item()) != 0
    if ran:
        log.append((first_pass, l, [float(x) for x in self.dinfo[:4].cpu()], dt))
Ctx.cholqr_factor = wrapped
class NoRollback:
    def __init__(self, seed): self.g = np.random.default_rng(seed)
    def random(self, k): return self.g.random(k)
pod.isma_run(A, cfg, rng=NoRollback(7), use_graphs=False)
for e in log[:24]:
    print(e)
att = [e[2][1] for e in log]
print("calls", len(log), "attempts histogram", np.unique(att, return_counts=True))
