"""profiles/r02_ncu_traffic.txt from an ncu --set full report of
tools/profile_targets.py: DRAM bytes read / written per call of each op
(the second, warm call; multi-kernel ops summed), matched to the op order.
    python tools/ncu_traffic.py report.ncu-rep > profiles/r02_ncu_traffic.txt"""
import csv, subprocess, sys

# kernels per call of each op, in tools/profile_targets.py order
OPS = [("colnorms2", 1), ("draw", 1), ("tn_gram_gather", 2), ("tn_merge_proj", 2),
       ("tn_cholqr_gram", 2), ("nn_lift_gather", 1), ("nn_merge_resid", 1),
       ("nn_merge_rotate", 1), ("gram_eigh", 2), ("merge_core", 1), ("cholqr_factor", 1),
       ("nn_merge_resid+gram", 2), ("wedin_k20", 3)]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
it = hdr.index("gpu__time_duration.sum")
ki = hdr.index("Kernel Name")
data = rows[2:]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
print("# ncu --set full --clock-control none, tools/profile_targets.py on one B200 (round 2, session 2):")
print("# DRAM traffic per call of each hot op (its second, warm call), config-2 shapes")
print(f"op | dram_rd | unit | dram_wr | unit | dur [{units[it]}] | kernels")
pos = 0
for name, nk in OPS:
    calls = []
    for _ in range(2):
        ks = data[pos:pos + nk]
        pos += nk
        rd = sum(float(r[ir]) * scale.get(units[ir], 1) for r in ks)
        wr = sum(float(r[iw]) * scale.get(units[iw], 1) for r in ks)
        dt = sum(float(r[it]) for r in ks)
        calls.append((rd, wr, dt, "+".join(r[ki].split("(")[0][-40:] for r in ks)))
    rd, wr, dt, kn = calls[-1]
    print(f"{name} | {rd / 1e6:.3f} | Mbyte | {wr / 1e6:.3f} | Mbyte | {dt:.4g} | {kn}")
