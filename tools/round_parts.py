"""GPU time of a config-2 round's parts, each captured alone in a CUDA graph:
merge chain only, update only (both on one stream), and the pipelined round."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_05107_b200 as pod
from paper_1905_05107_b200 import workloads, engine
from paper_1905_05107_b200.device import ColMat, get_ctx
dev = torch.device("cuda", 0)
at = workloads.config2_torch(7, 512, 2000, device=dev)
A = ColMat(at, 512 * 512)
cfg = pod.IsmaConfig(k=20, r=60, c=100, tau=1 - 1e-8, strategy="l2n", seed=7)
f, tr, eng = pod.isma_run(A, cfg, return_device=True)
ctx = get_ctx(dev)
eng.A = A
rng = np.random.default_rng(0)
for b in (0, 1):
    eng._stage_uniforms(rng, b)
eng.live.fill_(1)


def timed(fn, reps=20):
    st = torch.cuda.Stream(dev)
    st.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(st):
        fn()
    torch.cuda.current_stream(dev).wait_stream(st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay(); torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        eng.live.fill_(1)
        g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms_merge = timed(lambda: (eng.merge_ops(0, 1), eng.cosines_ops(0, 1)))
ms_update = timed(lambda: eng.update_ops(engine.MODE_L2N, 1, eng.Uupd_b[1].cols(0, eng.r)))
ms_round = timed(lambda: eng.round_ops(engine.MODE_L2N, 0, 1, True))
ms_serial = timed(lambda: eng.round_ops(engine.MODE_L2N, 0, 1, False))
print(f"merge chain {ms_merge:.3f} ms, update {ms_update:.3f} ms, pipelined round {ms_round:.3f} ms, serial round {ms_serial:.3f} ms")
