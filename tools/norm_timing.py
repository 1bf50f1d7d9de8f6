"""CUDA-event timing of the einsum-order norm pass and the exact draw."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1905_05107_b200 import _lib
from paper_1905_05107_b200.device import ColMat, _ptr, get_ctx

ctx = get_ctx()
dev = ctx.device
out = {}
for (m, n, dt) in [(262144, 2000, torch.float64), (1000000, 2000, torch.float64),
                   (1048576, 8192, torch.float32), (1000000, 20000, torch.float64)]:
    try:
        t = torch.empty((n, m), dtype=dt, device=dev)
        t.normal_()
    except torch.OutOfMemoryError:
        continue
    A = ColMat(t, m, n)
    nrm = torch.empty(n, dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    for _ in range(2):
        ctx.colnorms2(A, nrm, flag)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ctx.colnorms2(A, nrm, flag)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    gb = m * n * t.element_size() / 1e9
    out[f"norms {m}x{n} {dt}"] = {"ms": ms, "GBps": gb / ms * 1e3}
    del t, A
    torch.cuda.empty_cache()
lib = _lib.load()
for n in (2000, 8192, 20000, 50000):
    raw = torch.rand(n, dtype=torch.float64, device=dev)
    live = torch.ones(n, dtype=torch.uint8, device=dev)
    uni = torch.rand(256, dtype=torch.float64, device=dev)
    ws = torch.zeros(int(lib.pod_draw_ws_bytes(n)), dtype=torch.uint8, device=dev)
    idx = torch.empty(256, dtype=torch.int32, device=dev)
    cnt = torch.empty(256, dtype=torch.int64, device=dev)
    info = torch.zeros(4, dtype=torch.int64, device=dev)
    for mode in (0, 1):
        def go():
            live.fill_(1)
            _lib.call("pod_draw", mode, _ptr(raw), _ptr(live), n, _ptr(uni), 256, _ptr(idx),
                      _ptr(cnt), 256, _ptr(ws), ws.numel(), _ptr(info), 0.0, None, ctx.stream)
        go(); go()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            go()
        e1.record()
        torch.cuda.synchronize()
        out[f"draw n={n} mode={mode}"] = {"ms": e0.elapsed_time(e1) / 5}
print(json.dumps(out, indent=1))
