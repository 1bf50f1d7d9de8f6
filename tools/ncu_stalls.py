"""Warp-stall reasons (pc sampling) and pipe utilisation per profiled kernel
of an ncu --set full report:  python tools/ncu_stalls.py report.ncu-rep"""
import csv, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki = hdr.index("Kernel Name")
KEEP = [("gpu__time_duration.sum", "dur"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem%"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("lts__t_sector_hit_rate.pct", "l2hit%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]
for r in rows[2:]:
    name = r[ki].split("(")[0][-56:]
    vals = [f"{lab} {r[hdr.index(m)]}" for m, lab in KEEP if m in hdr]
    st = []
    for i, h in enumerate(hdr):
        if "pcsamp_warps_issue_stalled" in h and "not_issued" not in h:
            try:
                st.append((float(r[i].replace(",", "")), h.split("stalled_")[1]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1.0
    top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:6])
    print(name + " | " + " | ".join(vals))
    print("    stalls: " + top)
