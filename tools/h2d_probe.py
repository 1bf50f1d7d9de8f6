"""H2D bandwidth of the public-API input path (pinned vs pageable, chunked)."""
import time, torch, numpy as np
dev = torch.device("cuda", 0)
n, m = 2000, 262144
host = torch.empty((n, m), dtype=torch.float64).pin_memory()
host.fill_(1.0)
d = torch.empty((n, m), dtype=torch.float64, device=dev)
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
gb = n * m * 8 / 1e9
print("pinned tensor copy_      %.1f GB/s" % (gb / t(lambda: d.copy_(host, non_blocking=True))))
a = host.numpy()
ft = torch.from_numpy(a)
print("from_numpy(pinned) copy_ %.1f GB/s  is_pinned=%s" % (gb / t(lambda: d.copy_(ft, non_blocking=True)), ft.is_pinned()))
print("from_numpy .to(dev)      %.1f GB/s" % (gb / t(lambda: ft.to(dev))))
pg = np.ones((n, m))
pt = torch.from_numpy(pg)
print("pageable copy_           %.1f GB/s" % (gb / t(lambda: d.copy_(pt, non_blocking=True))))
# chunked on two streams
s = [torch.cuda.Stream(dev) for _ in range(2)]
def chunked(src):
    nch = 16
    step = n // nch
    for i in range(nch):
        with torch.cuda.stream(s[i % 2]):
            d[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)
    for st in s: torch.cuda.current_stream().wait_stream(st)
print("pinned chunked 2 streams %.1f GB/s" % (gb / t(lambda: chunked(host))))
