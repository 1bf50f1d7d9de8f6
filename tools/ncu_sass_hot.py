"""Aggregate ncu --page source --csv (SASS) warp-stall samples by opcode and
list the hottest instructions:  python tools/ncu_sass_hot.py report.ncu-rep [kernel-substr]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
lines = out.splitlines()
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]; blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
want = sys.argv[2] if len(sys.argv) > 2 else ""
for b in blocks:
    name = next(csv.reader([b[0]]))[1]
    if want not in name:
        continue
    rows = list(csv.reader(b[1:]))
    hdr = rows[0]
    si, ss = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    ops = collections.Counter(); tot = 0; hot = []
    for r in rows[1:]:
        try:
            n = int(r[ss])
        except ValueError:
            continue
        op = r[si].strip().split()[0] if r[si].strip() else "?"
        if op.startswith("@"):
            op = r[si].strip().split()[1]
        ops[op.split(".")[0]] += n; tot += n
        hot.append((n, r[si].strip()))
    print(name[:100], "total samples", tot)
    for op, n in ops.most_common(12):
        print(f"  {op:10s} {n:8d} {100 * n / tot:5.1f}%")
    for n, s in sorted(hot, reverse=True)[:15]:
        print(f"  {n:7d}  {s[:90]}")
