"""Per-kernel device time of one eager (unpipelined, CUDA events around every
launch) config-2 run, plus the graph-mode total for comparison."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_05107_b200 as pod  # noqa: E402
from paper_1905_05107_b200 import isma as isma_mod, workloads  # noqa: E402
from paper_1905_05107_b200.device import ColMat, KernelProfile, get_ctx  # noqa: E402

dev = torch.device("cuda", 0)
at = workloads.config2_torch(7, 512, 2000, device=dev)
A = ColMat(at, 512 * 512)
cfg = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7)
for _ in range(2):
    f, tr = pod.isma_run(A, cfg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
f, tr = pod.isma_run(A, cfg)
e1.record()
torch.cuda.synchronize()
print(f"graph-mode run {e0.elapsed_time(e1):.2f} ms, rounds {len(tr)}")
st = isma_mod.LAST_STATS
print("eigh sweeps", st.get("eigh_sweeps", [])[:25])
print("merge sweeps", st.get("merge_sweeps", [])[:25])


class NoRollback:
    def __init__(self, seed):
        self.g = np.random.default_rng(seed)

    def random(self, k):
        return self.g.random(k)


ctx = get_ctx(dev)
prof = KernelProfile()
ctx.prof = prof
pod.isma_run(A, cfg, rng=NoRollback(7))
ctx.prof = None
kern = prof.summary()
tot = sum(v["ms"] for v in kern.values())
print(f"eager profiled total {tot:.2f} ms")
for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["ms"])[:20]:
    print(f"{k:28s} calls {v['calls']:5d} ms {v['ms']:8.3f} ({100 * v['ms'] / tot:5.1f}%) "
          f"per call {1e3 * v['ms'] / v['calls']:8.1f} us")
