"""One line per profiled kernel of an ncu report (--set full): duration,
DRAM bytes, DRAM/tensor/SM utilisation, occupancy, registers.
    python tools/ncu_summary.py report.ncu-rep"""
import csv, subprocess, sys

METRICS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
ki = hdr.index("Kernel Name")
idx = [(hdr.index(m), lab, units[hdr.index(m)]) for m, lab in METRICS if m in hdr]
print("kernel | " + " | ".join(f"{lab} [{u}]" for _, lab, u in idx))
for r in rows[2:]:
    name = r[ki].split("(")[0][-48:]
    print(name + " | " + " | ".join(r[i] for i, _, _ in idx))
