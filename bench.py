#!/usr/bin/env python
"""Benchmark: time to converged k POD modes on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], the largest config quoted for 1 GPU):
the config-2 snapshot matrix, m = 262144 (512 x 512 field) x n = 2000,
fp64, k = 20, r = 3k = 60, c = 100 draws per round, strategy l2n,
criterion "modes", tau = 1 - tol with tol = 1e-8, seed 7,
finalize on.  Synthetic data from ``workloads.config2_torch`` generated on
the device (outside the timed region).  A step = one full ``isma_run``
(norm pass, bootstrap, every update round, finalize) over the resident
matrix; A is 4.2 GB >> 126 MB L2, so no L2 flush is needed between steps.

Arms:
  default           our CUDA path (value = device-resident run, e2e = the
                    public API on pinned host memory incl. H2D of A)
  --impl reference  the reference algorithm on the host CPU (the numpy /
                    LAPACK oracle port, oracle/isma_oracle.py, all cores),
                    each step a bounded sample extrapolated to the run.

One JSON line on stdout (rank 0).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time to converged k POD modes (s) & achieved HBM GB/s, 1/2/4/8 B200 vs CPU ref"
WORKLOAD = dict(side=512, n=2000, k=20, r=60, c=100, tol=1e-8, strategy="l2n",
                criterion="modes", seed=7, data_seed=0)
CPU_SAMPLE_ROUNDS = 3


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


FP64_DMMA_TFLOPS = 37.17  # tools/fp64_peak.cu on this pool's B200 (profiles/fp64_peak.txt)


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


# ncu `--set full` capture of every hot kernel (tools/profile_targets.py,
# committed summary): launch order -> the bench's kernel tags
PROFILE_SUMMARY = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                               "r01_ncu_full_summary.txt")
PROFILE_TAGS = ["colnorms2", "colnorms2", "tn_gram_gather", "tn_gram_gather", "tn_merge_proj",
                "tn_merge_proj", "tn_cholqr_gram", "tn_cholqr_gram", "nn_lift_gather",
                "nn_lift_gather", "nn_merge_resid", "nn_merge_resid", "nn_merge_rotate",
                "nn_merge_rotate", "gram_eigh", "gram_eigh", "gram_eigh", "gram_eigh",
                "merge_core", "merge_core", "cholqr_factor", "cholqr_factor"]


def _profiled_traffic():
    """DRAM bytes (read + write) per call of each tagged kernel from the
    committed ncu capture (second, warm call of each op; pivoted Cholesky and
    Jacobi summed for gram_eigh), or {} when the summary is absent."""
    try:
        lines = [ln for ln in open(PROFILE_SUMMARY) if not ln.startswith("#")]
    except OSError:
        return {}
    hdr = [h.strip() for h in lines[0].split("|")]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    cols = {}
    for i, h in enumerate(hdr):
        for key in ("dram_rd", "dram_wr"):
            if h.startswith(key):
                cols[key] = (i, scale.get(h[h.find("[") + 1:h.find("]")], 1.0))
    rows = [[c.strip() for c in ln.split("|")] for ln in lines[1:] if "|" in ln]
    per_call = {}
    seen = {}
    for tag, r in zip(PROFILE_TAGS, rows):
        b = sum(float(r[i]) * sc for i, sc in cols.values())
        seen[tag] = seen.get(tag, 0) + 1
        per_call.setdefault(tag, []).append(b)
    out = {}
    for tag, vals in per_call.items():
        k = 2 if tag == "gram_eigh" else 1  # launches per call
        calls = [sum(vals[i:i + k]) for i in range(0, len(vals), k)]
        out[tag] = calls[-1]  # the warm call
    return out


def _kernel_roofline(name, v, w, peaks, traffic):
    per_launch_s = v["ms"] / 1e3 / v["calls"]
    if v["flops"] > 0 and name[:3] in ("tn_", "nn_"):
        ach = v["flops"] / v["calls"] / per_launch_s / 1e12
        roof = {"kernel": name, "bound": "tensor", "achieved": ach, "peak": FP64_DMMA_TFLOPS,
                "unit": "TFLOP/s", "frac": ach / FP64_DMMA_TFLOPS,
                "peak_source": "measured FP64 DMMA.8x8x4 peak (tools/fp64_peak.cu)"}
    elif name in ("merge_core", "gram_eigh"):
        # cluster block-Jacobi: the flops actually done (sweeps x n(n-1)/2
        # pairs x 6 n) on 8 SMs; the solver is bound by its sequential depth
        # (n - 1 dependent sub-rounds per sweep), see DESIGN.md section 3
        import paper_1905_05107_b200.isma as _isma
        st = _isma.LAST_STATS
        key = "merge_sweeps" if name == "merge_core" else "eigh_sweeps"
        nn_ = 2 * w["r"] if name == "merge_core" else min(w["c"], w["n"])
        sweeps = sum(st.get(key, [0])) / max(len(st.get(key, [1])), 1)
        flops = sweeps * nn_ * (nn_ - 1) / 2 * 6 * nn_
        ach = flops / per_launch_s / 1e12
        roof = {"kernel": name, "bound": "tensor", "achieved": ach, "peak": FP64_DMMA_TFLOPS,
                "unit": "TFLOP/s", "frac": ach / FP64_DMMA_TFLOPS,
                "peak_source": "measured FP64 DMMA.8x8x4 peak (tools/fp64_peak.cu); "
                               "latency-bound cluster Jacobi, see DESIGN.md"}
    else:
        ach = v["bytes"] / v["calls"] / per_launch_s / 1e9
        pk = peaks.get("hbm_gbs", 6650.0)
        roof = {"kernel": name, "bound": "hbm", "achieved": ach, "peak": pk, "unit": "GB/s",
                "frac": ach / pk,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks
                else "fallback 6650 GB/s"}
    roof["traffic"] = traffic.get(name)
    if roof["traffic"] is not None:
        roof["traffic_source"] = "profiles/r01_ncu_full_summary.txt dram__bytes_read+write per call"
    return roof


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference_sample(a_host, steps, warmup, n_rounds_full):
    """The reference algorithm (oracle port) on the host: bootstrap + the
    first CPU_SAMPLE_ROUNDS update rounds + finalize on the full matrix,
    extrapolated to the full round count with the mean sampled round."""
    from oracle import isma_oracle as orc

    w = WORKLOAD
    est = []
    for i in range(warmup + steps):
        out = orc.run(a_host, w["k"], r=w["r"], c=w["c"], tau=1 - w["tol"],
                      strategy=w["strategy"], criterion=w["criterion"], seed=w["seed"],
                      max_rounds=CPU_SAMPLE_ROUNDS)
        tr = out["trace"]
        t_boot = tr[0]["wall_time"]
        rounds = [t["wall_time"] for t in tr[1:]]
        per_round = sum(rounds) / max(len(rounds), 1)
        full = (out["timings"]["norms"] + t_boot + per_round * (n_rounds_full - 1)
                + out["timings"]["finalize"])
        if i >= warmup:
            est.append(full)
    try:
        from threadpoolctl import threadpool_info

        threads = max([d.get("num_threads", 1) for d in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    return statistics.mean(est), threads


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


def run_reference_arm(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return 0
    import torch

    from paper_1905_05107_b200 import workloads

    w = WORKLOAD
    at = workloads.config2_torch(w["data_seed"], w["side"], w["n"], device="cpu")
    a_host = at.numpy().T  # F-order view
    # full round count: the l2n index stream does not depend on the factor,
    # so replay the draws alone (cheap) to learn it
    from oracle import isma_oracle as orc

    norms2 = orc.column_norms2(a_host)
    rng = np.random.default_rng(w["seed"])
    s = np.arange(w["n"])
    n_rounds = 0
    while s.size:
        idx, _ = orc.cdf_draw(s, orc.normalized_weights(norms2[s]), rng.random(w["c"]))
        s = np.setdiff1d(s, idx, assume_unique=True)
        n_rounds += 1
    value, threads = cpu_reference_sample(a_host, args.steps, args.warmup, n_rounds)
    del torch
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_dict(n_rounds),
        "cpu_baseline": {"value": value, "unit": "s", "cores": threads, "kind": "port",
                         "host": _host_desc(),
                         "sample": f"oracle port of podsketch isma_run on the full config-2 "
                                   f"matrix: norm pass + bootstrap + {CPU_SAMPLE_ROUNDS} update "
                                   f"rounds + finalize, extrapolated to {n_rounds} rounds"},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _config_dict(n_rounds=None):
    w = WORKLOAD
    d = {"workload": "config2 snapshot field 512x512 -> m=262144, n=2000, fp64; k=20, r=60, "
                     "c=100, l2n, modes, tau=1-1e-8, finalize",
         "m": w["side"] ** 2, "n": w["n"], "k": w["k"], "r": w["r"], "c": w["c"],
         "tau": 1 - w["tol"], "strategy": w["strategy"], "criterion": w["criterion"],
         "seed": w["seed"], "l2_policy": "A is 4.2 GB >> 126 MB L2 (no flush needed)"}
    if n_rounds is not None:
        d["rounds"] = n_rounds
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch

    import paper_1905_05107_b200 as pod
    from paper_1905_05107_b200 import workloads
    from paper_1905_05107_b200.device import KernelProfile, get_ctx, to_device_colmajor

    ws, rank, local = _dist_env()
    comm = None
    if ws > 1:
        torch.cuda.set_device(local % torch.cuda.device_count())
        import torch.distributed as dist

        dist.init_process_group(os.environ.get("POD_DIST_BACKEND", "nccl"))
        from paper_1905_05107_b200.parallel import Comm, shard_rows

        comm = Comm()
    w = WORKLOAD
    ctx = get_ctx()
    dev = ctx.device
    m_total = w["side"] ** 2
    rows = (0, m_total) if ws == 1 else shard_rows(m_total, ws, rank)  # row-sharded A
    at = workloads.config2_torch(w["data_seed"], w["side"], w["n"], device=dev, rows=rows)
    m, n = at.shape[1], at.shape[0]
    A = to_device_colmajor(at.T, dev)
    cfg = pod.IsmaConfig(k=w["k"], r=w["r"], c=w["c"], tau=1 - w["tol"], strategy=w["strategy"],
                         criterion=w["criterion"], seed=w["seed"])
    stream = torch.cuda.current_stream(dev)

    def one_run():
        if comm is None:
            return pod.isma_run(A, cfg)
        return pod.isma_run(A, cfg, comm=comm, m_total=m_total)

    for _ in range(args.warmup):
        factor, traces = one_run()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    launches0 = ctx.launches
    times = []
    with ClockSampler(index=torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            factor, traces = one_run()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    launches = ctx.launches - launches0
    step_s = statistics.mean(times)
    if ws > 1:
        t = torch.tensor([step_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_s = float(t.item())
    # instrumented pass: the same run launched eagerly with CUDA events around
    # every kernel (graph replay hides individual launches)
    class _NoRollback:  # a generator without a rollback-able state: unpipelined rounds,
        def __init__(self, seed):  # so every kernel is timed without a concurrent stream
            self.g = np.random.default_rng(seed)

        def random(self, k):
            return self.g.random(k)

    prof = KernelProfile()
    ctx.prof = prof
    if comm is None:
        pod.isma_run(A, cfg, rng=_NoRollback(w["seed"]))
    else:
        pod.isma_run(A, cfg, rng=_NoRollback(w["seed"]), comm=comm, m_total=m_total)
    ctx.prof = None
    kern = prof.summary()
    n_rounds = len(traces)

    # roofline of the dominant kernel (by total device time; gated launches,
    # whose work is decided on the device, are excluded from the flop count),
    # and of the next five for context
    peaks = _peaks()
    traffic = _profiled_traffic()
    ranked = sorted(((k, v) for k, v in kern.items() if "[gated]" not in k),
                    key=lambda kv: -kv[1]["ms"])
    roofs = [_kernel_roofline(k, v, w, peaks, traffic) for k, v in ranked[:6]]
    roof = dict(roofs[0])
    norm = kern.get("colnorms2")
    hbm_norm = (norm["bytes"] / (norm["ms"] / 1e3)) / 1e9 if norm else None
    breakdown = {k: {"ms_per_step": v["ms"], "calls_per_step": v["calls"],
                     "tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["flops"] else None,
                     "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["bytes"] else None}
                 for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["ms"])}

    line = {
        "metric": METRIC, "value": step_s, "unit": "s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded config-2 Fourier snapshot generator, on device)",
        "parallelism": f"row-sharded dp{ws}" if ws > 1 else "single GPU",
        "config": _config_dict(n_rounds),
        "hbm_gbs_norm_pass": hbm_norm,
        "roofline": roof,
        "roofline_top": roofs,
        "kernels": breakdown,
        "gpu_launches": launches,
        "clocks": clk.result(),
        "sigma_top3": [float(x) for x in factor.sigma[:3]],
        "engine_stats": {k: (v if not isinstance(v, list) else
                             {"mean": sum(v) / max(len(v), 1), "max": max(v) if v else 0})
                         for k, v in __import__("paper_1905_05107_b200.isma", fromlist=["x"])
                         .LAST_STATS.items()},
    }

    if rank == 0 and ws == 1 and not args.no_e2e:
        # public API with HOST buffers: H2D of A and D2H of the factor inside the timed region
        host = torch.empty((n, m), dtype=torch.float64).pin_memory()
        host.copy_(at)
        a_host = host.numpy().T  # F-order numpy view of pinned memory
        del at
        torch.cuda.empty_cache()
        e2e = []
        # same warm-up / timed split as the device-resident measurement: the
        # steady state reuses the cached device buffers, captured graphs and
        # page-locked result blocks (a caller's previous result stays alive)
        for i in range(max(args.warmup, 3) + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f_h, tr_h = pod.isma_run(a_host, cfg)
            torch.cuda.synchronize()
            if i >= max(args.warmup, 3):
                e2e.append(time.perf_counter() - t0)
        h2d = m * n * 8 + len(tr_h) * w["c"] * 8
        d2h = (f_h.u.size + f_h.sigma.size + (f_h.v.size if f_h.v is not None else 0)) * 8
        line["e2e"] = {"value": statistics.mean(e2e), "unit": "s", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h}
        if not args.no_cpu_baseline:
            cpu_s, threads = cpu_reference_sample(a_host, 1, 0, n_rounds)
            line["cpu_baseline"] = {
                "value": cpu_s, "unit": "s", "cores": threads, "kind": "port",
                "host": _host_desc(),
                "sample": f"oracle port (numpy/LAPACK) of podsketch isma_run, full config-2 "
                          f"matrix: norm pass + bootstrap + {CPU_SAMPLE_ROUNDS} update rounds + "
                          f"finalize, extrapolated to {n_rounds} rounds"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
