"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch
list:  python tools/launch_summary.py launches.csv"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr = rows[hi]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = collections.Counter(), collections.Counter()
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = re.sub(r"\(.*", "", r[ki])
    name = re.sub(r"^void ", "", name)[:64]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    cnt[name] += 1
T = sum(tot.values())
print(f"launches {sum(cnt.values())}, summed device time {T:.2f} ms (serialised, cold-cache ncu replay)")
print(f"{'kernel':64s} {'launches':>8s} {'ms':>9s} {'share':>6s}")
for k, v in tot.most_common(30):
    print(f"{k:64s} {cnt[k]:8d} {v:9.2f} {100 * v / T:5.1f}%")
