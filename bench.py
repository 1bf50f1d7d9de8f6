#!/usr/bin/env python
"""Benchmark: time to converged k POD modes on B200 (BASELINE.json metric).

Headline workload (BASELINE.json configs[1], the config the metric is quoted
on for one GPU, and the one the CPU reference can run in full): the config-2
snapshot matrix, m = 262144 (512 x 512 field) x n = 2000, fp64, k = 20,
r = 3k = 60, c = 100 draws per round, strategy l2n, criterion "modes",
tau = 1 - tol with tol = 1e-8, seed 7, finalize on.  The
matrix comes from ``workloads.config2_torch`` on the HOST CPU (seeded,
device-independent), so the GPU arm, its e2e leg and the CPU reference arm
all run on the same bits.  A step = one full ``isma_run`` (norm pass,
bootstrap, every update round, finalize) over the matrix; A is 4.2 GB >> the
126 MB L2, so no flush is needed between steps.

North-star workload, reported in the same line under "north_star": config 3
(1M x 20k fp64 = 160 GB, rank-200 power-law spectrum + N(0, 1e-6), generated
ON THE DEVICE from a seed as BASELINE.json states; k = 50, r = 150, c = 200,
l2n, modes, tau = 1 - 1e-8) with its own value, roofline and e2e (the e2e of a
device-generated input = the public call from the seed: generation + run +
result copy-back).  Row-sharded over the ranks when N > 1.

Arms:
  default           our CUDA path (value = device-resident run, e2e = the
                    public API on a pinned host matrix incl. its H2D copy)
  --impl reference  the reference algorithm on the host CPU: the oracle port
                    (numpy / LAPACK, oracle/isma_oracle.py) of isma_run, the
                    FULL run on the same matrix each step, at the better of
                    1 thread and all physical cores (both reported)
  --dry-run         CPU-only (gloo) rehearsal of the N-rank launch and the
                    sharded host protocol (chained norm pass + redundant
                    draws): every rank must agree bit for bit

``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks (127.0.0.1).  One JSON line on stdout
(rank 0).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time to converged k POD modes (s) & achieved HBM GB/s, 1/2/4/8 B200 vs CPU ref"
CFG2 = dict(side=512, n=2000, k=20, r=60, c=100, tol=1e-8, strategy="l2n", criterion="modes",
            seed=7, data_seed=0)
CFG3 = dict(m=1_000_000, n=20_000, rank=200, k=50, r=150, c=200, tol=1e-8, strategy="l2n",
            criterion="modes", seed=7, data_seed=0)
FP64_DMMA_TFLOPS = 37.17  # tools/fp64_peak.cu on this pool's B200 (profiles/fp64_peak.txt)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) during the timed region."""

    def __init__(self, index=0, period=0.1):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._th = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover
            self.nv = None
        self.period = period

    def _run(self):
        nv = self.nv
        names = {
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown",
                                               0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._th:
            self._th.join()

    def result(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ncu `--set full` DRAM traffic per call of the hot kernels (committed
# summary of tools/profile_targets.py): "name | dram_rd [unit] | dram_wr [unit]"
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "r02c_ncu_traffic.txt")


def _profiled_traffic():
    try:
        lines = [ln for ln in open(PROFILE_SUMMARY) if ln.strip() and not ln.startswith("#")]
    except OSError:
        return {}
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = {}
    for ln in lines[1:]:
        parts = [p.strip() for p in ln.split("|")]
        if len(parts) < 5:
            continue
        name, rd, rdu, wr, wru = parts[:5]
        try:
            out[name] = float(rd) * scale.get(rdu, 1.0) + float(wr) * scale.get(wru, 1.0)
        except ValueError:
            pass
    return out


def _kernel_roofline(name, v, w, peaks, traffic, stats):
    per_launch_s = v["ms"] / 1e3 / v["calls"]
    if v["flops"] > 0 and name[:3] in ("tn_", "nn_"):
        ach = v["flops"] / v["calls"] / per_launch_s / 1e12
        roof = {"kernel": name, "bound": "tensor", "achieved": ach, "peak": FP64_DMMA_TFLOPS,
                "unit": "TFLOP/s", "frac": ach / FP64_DMMA_TFLOPS,
                "peak_source": "measured FP64 DMMA.8x8x4 peak (tools/fp64_peak.cu)",
                "algorithmic": f"{v['flops'] / v['calls']:.4g} flop per call (DESIGN.md 4)"}
    elif name in ("merge_core", "gram_eigh"):
        # block Jacobi: the flops actually done (sweeps x n(n-1)/2 pairs x 6n)
        key = "merge_sweeps" if name == "merge_core" else "eigh_sweeps"
        nn_ = 2 * w["r"] if name == "merge_core" else min(w["c"], w["n"])
        sw = stats.get(key, [0])
        sweeps = sum(sw) / max(len(sw), 1)
        flops = sweeps * nn_ * (nn_ - 1) / 2 * 6 * nn_
        ach = flops / per_launch_s / 1e12
        roof = {"kernel": name, "bound": "tensor", "achieved": ach, "peak": FP64_DMMA_TFLOPS,
                "unit": "TFLOP/s", "frac": ach / FP64_DMMA_TFLOPS,
                "peak_source": "measured FP64 DMMA.8x8x4 peak (tools/fp64_peak.cu); "
                               "latency-bound Jacobi (sequential depth), DESIGN.md 4",
                "algorithmic": f"{sweeps:.2f} sweeps x {nn_}({nn_}-1)/2 pairs x 6*{nn_} flop"}
    else:
        ach = v["bytes"] / v["calls"] / per_launch_s / 1e9
        pk = peaks.get("hbm_gbs", 6650.0)
        roof = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": pk, "unit": "GB/s",
                "frac": ach / pk,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks
                else "fallback 6650 GB/s",
                "algorithmic": f"{v['bytes'] / v['calls']:.4g} bytes per call"}
    roof["avg_launch_ms"] = per_launch_s * 1e3
    roof["traffic"] = traffic.get(name)
    if roof["traffic"] is not None:
        roof["traffic_source"] = f"{os.path.relpath(PROFILE_SUMMARY, ROOT)} (dram rd+wr per call)"
    return roof


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _physical_cores():
    try:
        import psutil

        return psutil.cpu_count(logical=False) or os.cpu_count()
    except Exception:
        return os.cpu_count()


def _host_desc():
    """CPU model and the BLAS / numpy / scipy versions behind the CPU arm."""
    model = "unknown CPU"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        import scipy
        from threadpoolctl import threadpool_info

        blas = ", ".join(sorted({f"{d.get('internal_api')} {d.get('version')}"
                                 for d in threadpool_info()}))
        return f"{model}; numpy {np.__version__}, scipy {scipy.__version__}, {blas}"
    except Exception:
        return f"{model}; numpy {np.__version__}"


def config2_host(rows=None):
    """The headline matrix on the host: (torch (n, rows) storage, F-order view)."""
    from paper_1905_05107_b200 import workloads

    w = CFG2
    at = workloads.config2_torch(w["data_seed"], w["side"], w["n"], device="cpu", rows=rows)
    return at, at.numpy().T


def _config2_dict(n_rounds=None):
    w = CFG2
    d = {"workload": "config2 snapshot field 512x512 -> m=262144, n=2000, fp64; k=20, r=60, "
                     "c=100, l2n, modes, tau=1-1e-8, finalize",
         "m": w["side"] ** 2, "n": w["n"], "k": w["k"], "r": w["r"], "c": w["c"],
         "tau": 1 - w["tol"], "strategy": w["strategy"], "criterion": w["criterion"],
         "seed": w["seed"], "data": "seeded host generator (workloads.config2_torch, CPU)",
         "l2_policy": "A is 4.2 GB >> 126 MB L2 (no flush needed)"}
    if n_rounds is not None:
        d["rounds"] = n_rounds
    return d


# ------------------------------------------------------------ CPU arm ------
def cpu_isma_once(a_host, threads):
    """One FULL isma_run of the oracle port (norms, every round, finalize) on
    `threads` BLAS threads; returns (seconds, rounds)."""
    from threadpoolctl import threadpool_limits

    from oracle import isma_oracle as orc

    w = CFG2
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        out = orc.run(a_host, w["k"], r=w["r"], c=w["c"], tau=1 - w["tol"],
                      strategy=w["strategy"], criterion=w["criterion"], seed=w["seed"])
        dt = time.perf_counter() - t0
    return dt, len(out["trace"])


def cpu_baseline_pair(a_host):
    """Full runs at 1 thread and at all physical cores; the better is the baseline."""
    cores = _physical_cores()
    t1, rounds = cpu_isma_once(a_host, 1)
    tn, _ = cpu_isma_once(a_host, cores)
    best_threads, best = (1, t1) if t1 <= tn else (cores, tn)
    return {"value": best, "unit": "s", "cores": best_threads, "kind": "port",
            "threads_1_s": t1, f"threads_{cores}_s": tn, "physical_cores": cores,
            "host": _host_desc(), "rounds": rounds,
            "sample": "oracle port (numpy/LAPACK) of podsketch isma_run: ONE full run (norm "
                      "pass, all rounds, finalize) on the same config-2 matrix, at 1 thread and "
                      f"at {cores} threads; value = the better"}


def run_reference_arm(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return 0
    _, a_host = config2_host()
    cores = _physical_cores()
    # warm-up: one run at 1 thread and the rest at all cores decide the arm's
    # thread count (the better of the two); then K timed runs
    t1, n_rounds = cpu_isma_once(a_host, 1)
    tn = [cpu_isma_once(a_host, cores)[0] for _ in range(max(args.warmup - 1, 1))]
    threads = 1 if t1 <= statistics.median(tn) else cores
    times = [cpu_isma_once(a_host, threads)[0] for _ in range(args.steps)]
    value = statistics.mean(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config2_dict(n_rounds),
        "cpu_baseline": {"value": value, "unit": "s", "cores": threads, "kind": "port",
                         "threads_1_s": t1, f"threads_{cores}_s": statistics.median(tn),
                         "physical_cores": cores, "host": _host_desc(),
                         "median_s": statistics.median(times),
                         "sample": f"oracle port of podsketch isma_run: the FULL run (norm pass, "
                                   f"all {n_rounds} rounds, finalize) on the config-2 matrix every "
                                   f"step, at {threads} BLAS thread(s) (the better of 1 and "
                                   f"{cores}, decided in the warm-up)"},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------- launcher -----
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(argv, nproc):
    """Re-exec this script under torch.distributed.run with nproc ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def dry_run(args):
    """CPU rehearsal of the sharded protocol (gloo): each rank holds its row
    shard of a config-2 proxy, runs the chained einsum-order norm pass (the
    oracle's lane restatement stands in for pod_colnorms2_chain), and draws
    every round's index set redundantly; rank 0 checks that all ranks agree
    and equal the single-process numpy result."""
    import torch
    import torch.distributed as dist

    from oracle import isma_oracle as orc
    from paper_1905_05107_b200 import workloads
    from paper_1905_05107_b200.parallel import Comm, shard_rows

    ws, rank, _ = _dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    comm = Comm()
    side, n, c = 64, 300, 40
    m = side * side
    r0, r1 = shard_rows(m, comm.world, comm.rank)
    seg = workloads.config2_torch(1, side, n, device="cpu", rows=(r0, r1)).numpy().T
    st = None
    if comm.rank > 0:
        st = comm.recv(torch.empty(2 * n, dtype=torch.float64), comm.rank - 1).numpy()
        st = st.reshape(2, n)
    last = comm.rank == comm.world - 1
    body = seg.shape[0] - (seg.shape[0] % 8 if last else 0)
    st = orc.einsum_lane_state(seg[:body], st)
    norms = torch.zeros(n, dtype=torch.float64)
    if last:
        norms = torch.as_tensor(orc.einsum_lane_finish(seg[body:], st))
    else:
        comm.send(torch.as_tensor(st.reshape(-1).copy()), comm.rank + 1)
    comm.broadcast_(norms, comm.world - 1)
    nr = norms.numpy()
    rng = np.random.default_rng(CFG2["seed"])
    s = np.arange(n)
    draws = []
    while s.size:
        idx, _ = orc.cdf_draw(s, orc.normalized_weights(nr[s]), rng.random(c))
        draws.append(idx)
        s = np.setdiff1d(s, idx, assume_unique=True)
    h = hashlib.sha256(nr.tobytes() + b"".join(d.tobytes() for d in draws)).hexdigest()
    digests = [None] * comm.world
    if comm.world > 1:
        dist.all_gather_object(digests, h)
    else:
        digests = [h]
    if rank == 0:
        full = workloads.config2_torch(1, side, n, device="cpu").numpy().T
        ref = np.einsum("ij,ij->j", full, full)
        ok = all(d == digests[0] for d in digests) and np.array_equal(nr, ref)
        print(json.dumps({"dry_run": True, "n_ranks": comm.world, "rounds": len(draws),
                          "agree": ok, "digest": digests[0][:16],
                          "norms_equal_numpy": bool(np.array_equal(nr, ref))}), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------- GPU arm -----
def _profile_run(pod, A, cfg, kw):
    """The same run launched eagerly with CUDA events around every kernel on
    the launching stream (unpipelined: no concurrent side stream)."""
    from paper_1905_05107_b200.device import KernelProfile, get_ctx

    class NoRollback:  # a generator without a rollback-able state: unpipelined rounds
        def __init__(self, seed):
            self.g = np.random.default_rng(seed)

        def random(self, k):
            return self.g.random(k)

    ctx = get_ctx()
    prof = KernelProfile()
    ctx.prof = prof
    pod.isma_run(A, cfg, rng=NoRollback(cfg.seed), **kw)
    ctx.prof = None
    return prof.summary()


def _roofline_from(kern, w, stats):
    peaks = _peaks()
    traffic = _profiled_traffic()
    ranked = sorted(((k, v) for k, v in kern.items() if "[gated]" not in k),
                    key=lambda kv: -kv[1]["ms"])
    roofs = [_kernel_roofline(k, v, w, peaks, traffic, stats) for k, v in ranked[:6]]
    breakdown = {k: {"ms_per_step": v["ms"], "calls_per_step": v["calls"],
                     "tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["flops"] else None,
                     "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["bytes"] else None}
                 for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["ms"])}
    return roofs, breakdown


def _stats_summary(st):
    return {k: (v if not isinstance(v, list) else
                {"mean": sum(v) / max(len(v), 1), "max": max(v) if v else 0})
            for k, v in st.items()}


def _timed_runs(fn, steps, stream, torch):
    times = []
    for _ in range(steps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    return times


def _max_over_ranks(x, comm, torch, dev):
    if comm is None:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    comm.allreduce_max_(t)
    return float(t.item())


def north_star_block(args, pod, torch, dev, comm, ws, rank):
    """Config 3 (1M x 20k fp64, device-generated), row-sharded over the ranks."""
    from paper_1905_05107_b200 import engine as eng_mod, isma as isma_mod, workloads
    from paper_1905_05107_b200.device import ColMat, get_ctx
    from paper_1905_05107_b200.parallel import shard_rows

    w = CFG3
    eng_mod._ENGINE_CACHE.clear()
    torch.cuda.empty_cache()
    rows = (0, w["m"]) if ws == 1 else shard_rows(w["m"], ws, rank)
    t0 = time.perf_counter()
    at = workloads.config3_torch(w["data_seed"], w["m"], w["n"], w["rank"], device=dev, rows=rows)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    A = ColMat(at, rows[1] - rows[0])
    cfg = pod.IsmaConfig(k=w["k"], r=w["r"], c=w["c"], tau=1 - w["tol"], strategy=w["strategy"],
                         criterion=w["criterion"], seed=w["seed"])
    kw = {} if comm is None else dict(comm=comm, m_total=w["m"])
    stream = torch.cuda.current_stream(dev)
    ctx = get_ctx()
    res = {}

    def run():
        res["f"], res["tr"] = pod.isma_run(A, cfg, **kw)

    for _ in range(args.warmup):
        run()
    if comm is not None:
        comm.dist.barrier()
    l0 = ctx.launches
    steps = max(1, min(args.steps, args.ns_steps))
    times = _timed_runs(run, steps, stream, torch)
    launches = (ctx.launches - l0) // steps
    value = _max_over_ranks(statistics.mean(times), comm, torch, dev)
    stats = dict(isma_mod.LAST_STATS)
    kern = _profile_run(pod, A, cfg, kw)
    roofs, breakdown = _roofline_from(kern, dict(w, n=w["n"]), stats)
    out = {
        "workload": "config3 power-law 1M x 20k fp64 (160 GB), rank 200, sigma_i = i^-1.5, "
                    "N(0,1e-6), generated on the device from a seed; k=50, r=150, c=200, l2n, "
                    "modes, tau=1-1e-8, finalize",
        "value": value, "unit": "s", "steps": steps, "warmup": args.warmup,
        "rounds": len(res["tr"]), "columns_sampled": int(sum(t.columns_sampled for t in res["tr"])),
        "sigma_top3": [float(x) for x in res["f"].sigma[:3]],
        "roofline": dict(roofs[0]), "roofline_top": roofs, "kernels": breakdown,
        "gpu_launches_per_step": launches, "generation_s": gen_s,
        "engine_stats": _stats_summary(stats),
        "peak_mem_gib": torch.cuda.max_memory_allocated(dev) / 2 ** 30,
    }
    # e2e: the public call from the seed -- device generation + run + the
    # result's D2H (the input is defined as device-generated, BASELINE config 3)
    del A, at
    eng_mod._ENGINE_CACHE.clear()
    torch.cuda.empty_cache()
    e2e = []
    for _ in range(max(1, min(args.steps, args.ns_e2e_steps))):
        torch.cuda.synchronize()
        if comm is not None:
            comm.dist.barrier()
        t1 = time.perf_counter()
        at = workloads.config3_torch(w["data_seed"], w["m"], w["n"], w["rank"], device=dev,
                                     rows=rows)
        f, tr = pod.isma_run(ColMat(at, rows[1] - rows[0]), cfg, **kw)
        torch.cuda.synchronize()
        e2e.append(time.perf_counter() - t1)
        del at
    out["e2e"] = {"value": _max_over_ranks(statistics.mean(e2e), comm, torch, dev), "unit": "s",
                  "h2d_bytes_per_step": len(tr) * w["c"] * 8,
                  "d2h_bytes_per_step": (f.u.size + f.sigma.size
                                         + (f.v.size if f.v is not None else 0)) * 8,
                  "includes": "device generation of A from the seed + isma_run + factor D2H"}
    eng_mod._ENGINE_CACHE.clear()
    torch.cuda.empty_cache()
    return out


def config4_block(args, pod, torch, dev):
    """Config 4 (the config-2 generator at 1024^2 x 8192, STORED float32, 34 GB;
    k = 64, r = 192, c = 256): precision="mixed" -- finalize's A^T U on the
    tcgen05 tensor cores (3xTF32, TMEM accumulators) -- against the fp64
    path on the same matrix: both times, the mixed path's sigma / angle errors
    against the fp64 run, and the tcgen05 kernel's throughput."""
    from paper_1905_05107_b200 import engine as eng_mod, workloads
    from paper_1905_05107_b200.device import ColMat, get_ctx

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from parity_util import principal_angles_sin, sigma_relerr

    eng_mod._ENGINE_CACHE.clear()
    torch.cuda.empty_cache()
    w = workloads.CFG4
    at = workloads.config4_torch(7, w["side"], w["n"], device=dev)
    m = w["side"] ** 2
    A = ColMat(at, m)
    cfg = pod.IsmaConfig(k=w["k"], r=w["r"], c=w["c"], tau=1 - w["tol"], strategy="l2n", seed=7)
    stream = torch.cuda.current_stream(dev)
    out = {"workload": "config4 snapshot field 1024x1024 -> m=1048576, n=8192, stored fp32 "
                       "(34 GB); k=64, r=192, c=256, l2n, modes, tau=1-1e-8, finalize"}
    res = {}
    steps = max(1, min(args.steps, args.ns_steps))
    for prec in ("mixed", "fp64"):
        def run(prec=prec):
            res[prec] = pod.isma_run(A, cfg, precision=prec)
        for _ in range(args.warmup):
            run()
        t = _timed_runs(run, steps, stream, torch)
        out[f"{prec}_s"] = statistics.mean(t)
        out[f"{prec}_runs_s"] = t
    fm, fd = res["mixed"][0], res["fp64"][0]
    out["mixed_vs_fp64"] = {"sigma_rel_err": sigma_relerr(fm.sigma, fd.sigma),
                            "max_angle_rad": float(principal_angles_sin(fm.u, fd.u).max()),
                            "tolerance": "north_star mixed precision: sigma 1e-4, angles 1e-3"}
    kern = _profile_run(pod, A, cfg, {"precision": "mixed"})
    tc = kern.get("tc_finalize_AtU")
    if tc:
        peaks = _peaks()
        pk = 0.5 * peaks.get("bf16_tflops", 2250.0)
        ach = tc["flops"] / (tc["ms"] / 1e3) / tc["calls"] / 1e12
        out["tc_kernel"] = {
            "kernel": "tc_finalize_AtU (tcgen05.mma kind::tf32, 3 MMAs per product)",
            "ms": tc["ms"] / tc["calls"], "algorithmic_tflops": ach,
            "mma_tflops": 3 * ach, "peak_tf32_tflops": pk,
            "frac_of_tf32_peak": 3 * ach / pk,
            "peak_source": "0.5 x MEASURED_PEAKS.json bf16_tflops (dense TF32 = half of BF16)"}
        fd64 = kern.get("tn_finalize_AtU")
        if fd64:
            out["tc_kernel"]["fp64_dmma_ms"] = fd64["ms"] / fd64["calls"]
    del A, at
    eng_mod._ENGINE_CACHE.clear()
    torch.cuda.empty_cache()
    return out


def gpu_arm(args):
    import torch

    import paper_1905_05107_b200 as pod
    from paper_1905_05107_b200 import isma as isma_mod
    from paper_1905_05107_b200.device import get_ctx, to_device_colmajor

    ws, rank, local = _dist_env()
    comm = None
    if ws > 1:
        torch.cuda.set_device(local % torch.cuda.device_count())
        import torch.distributed as dist

        dist.init_process_group(os.environ.get("POD_DIST_BACKEND", "nccl"))
        from paper_1905_05107_b200.parallel import Comm

        comm = Comm()
    from paper_1905_05107_b200.parallel import shard_rows

    w = CFG2
    ctx = get_ctx()
    dev = ctx.device
    m_total = w["side"] ** 2
    rows = (0, m_total) if ws == 1 else shard_rows(m_total, ws, rank)
    at_host, a_host = config2_host(rows=rows)
    m, n = a_host.shape
    A = to_device_colmajor(a_host, dev)
    cfg = pod.IsmaConfig(k=w["k"], r=w["r"], c=w["c"], tau=1 - w["tol"], strategy=w["strategy"],
                         criterion=w["criterion"], seed=w["seed"])
    kw = {} if comm is None else dict(comm=comm, m_total=m_total)
    stream = torch.cuda.current_stream(dev)
    res = {}

    def one_run():
        res["f"], res["tr"] = pod.isma_run(A, cfg, **kw)

    for _ in range(args.warmup):
        one_run()
    torch.cuda.synchronize()
    if comm is not None:
        comm.dist.barrier()
    launches0 = ctx.launches
    with ClockSampler(index=torch.cuda.current_device()) as clk:
        times = _timed_runs(one_run, args.steps, stream, torch)
    launches = ctx.launches - launches0
    step_s = _max_over_ranks(statistics.mean(times), comm, torch, dev)
    stats = dict(isma_mod.LAST_STATS)
    kern = _profile_run(pod, A, cfg, kw)
    roofs, breakdown = _roofline_from(kern, w, stats)
    norm = kern.get("colnorms2")
    n_rounds = len(res["tr"])
    line = {
        "metric": METRIC, "value": step_s, "unit": "s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded config-2 Fourier snapshot generator on the host; the CPU "
                "reference arm uses the same bits)",
        "parallelism": f"row-sharded dp{ws}" if ws > 1 else "single GPU",
        "config": _config2_dict(n_rounds),
        "hbm_gbs_norm_pass": ((norm["bytes"] / (norm["ms"] / 1e3)) / 1e9) if norm else None,
        "roofline": dict(roofs[0]),
        "roofline_top": roofs,
        "kernels": breakdown,
        "gpu_launches": launches,
        "clocks": clk.result(),
        "sigma_top3": [float(x) for x in res["f"].sigma[:3]],
        "engine_stats": _stats_summary(stats),
        "timed_runs_s": times,
    }
    del A
    # e2e: the public API on a page-locked HOST matrix (H2D of A and D2H of the
    # factor inside the timed region), steady state
    if not args.no_e2e:
        host = at_host.pin_memory()
        a_pinned = host.numpy().T
        e2e = []
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            if comm is not None:
                comm.dist.barrier()
            t0 = time.perf_counter()
            f_h, tr_h = pod.isma_run(a_pinned, cfg, **kw)
            torch.cuda.synchronize()
            if i >= args.warmup:
                e2e.append(time.perf_counter() - t0)
        h2d = m * n * 8 + len(tr_h) * w["c"] * 8
        d2h = (f_h.u.size + f_h.sigma.size + (f_h.v.size if f_h.v is not None else 0)) * 8
        # this box's pinned H2D rate for the same bytes (the e2e floor's main term)
        dst = torch.empty_like(host, device=dev)
        h2d_t = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dst.copy_(host, non_blocking=True)
            torch.cuda.synchronize()
            h2d_t.append(time.perf_counter() - t0)
        del dst
        line["e2e"] = {"value": _max_over_ranks(statistics.mean(e2e), comm, torch, dev),
                       "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "runs_s": e2e, "h2d_matrix_s": min(h2d_t),
                       "h2d_gbs": m * n * 8 / min(h2d_t) / 1e9}
        del host, a_pinned
    if not args.no_north_star:
        line["north_star"] = north_star_block(args, pod, torch, dev, comm, ws, rank)
    if ws == 1 and not args.no_config4:
        line["config4_mixed"] = config4_block(args, pod, torch, dev)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_pair(a_host)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dry-run", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-north-star", action="store_true")
    ap.add_argument("--no-config4", action="store_true")
    ap.add_argument("--ns-steps", type=int, default=5, help="timed config-3 runs (<= --steps)")
    ap.add_argument("--ns-e2e-steps", type=int, default=2)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, _, _ = _dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(sys.argv[1:], args.gpus)
    if args.dry_run:
        return dry_run(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    return gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
