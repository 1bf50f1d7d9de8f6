"""Segment times inside each replayed round graph of a config-2 run:
external CUDA events recorded (and captured) around merge GEMMs, E-SVD,
rotation and the side-stream update."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads, engine, device
from paper_1905_05107_b200.device import ColMat
dev = torch.device("cuda", 0)
at = workloads.config2_torch(7, 512, 2000, device=dev)
A = ColMat(at, 512 * 512)
cfg = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7)

cur_events = {}
def mark(name):
    e = torch.cuda.Event(enable_timing=True, external=True)
    e.record(torch.cuda.current_stream(dev))
    cur_events[name] = e

orig_merge_core = device.Ctx.merge_core
def merge_core(self, *a, **k):
    mark("core_start"); orig_merge_core(self, *a, **k); mark("core_end")
device.Ctx.merge_core = merge_core
orig_update_ops = engine.IsmaEngine.update_ops
def update_ops(self, *a, **k):
    mark("upd_start"); orig_update_ops(self, *a, **k); mark("upd_end")
engine.IsmaEngine.update_ops = update_ops
orig_round_ops = engine.IsmaEngine.round_ops
def round_ops(self, *a, **k):
    mark("round_start"); orig_round_ops(self, *a, **k); mark("round_end")
engine.IsmaEngine.round_ops = round_ops
graph_events = {}
orig_launch = engine.IsmaEngine.launch_round
rows = []
def launch_round(self, mode, cur, ub, pipelined, rowsrc=None):
    key = (self.A.ptr.value, self.A.code, mode, cur, ub, pipelined, rowsrc)
    had = key in self.graphs
    cur_events.clear()
    orig_launch(self, mode, cur, ub, pipelined, rowsrc)
    if not had:
        graph_events[key] = dict(cur_events)  # the events captured into this graph
    ev = graph_events.get(key)
    torch.cuda.synchronize()
    if ev and had:
        t = lambda a, b: ev[a].elapsed_time(ev[b])
        rows.append((t("round_start", "core_start"), t("core_start", "core_end"),
                     t("core_end", "round_end"), t("upd_start", "upd_end"),
                     t("round_start", "upd_start"), t("round_start", "round_end")))
engine.IsmaEngine.launch_round = launch_round
for i in range(3):
    rows.clear()
    f, tr = pod.isma_run(A, cfg)
r = np.array(rows)
print("rounds traced", len(r))
names = ["merge GEMM phase", "E-SVD", "rotate+cosines(+join)", "update (side)", "update fork offset", "round"]
for j, n in enumerate(names):
    print(f"{n:24s} mean {r[:, j].mean():.3f} ms  min {r[:, j].min():.3f}  max {r[:, j].max():.3f}")
