for i in 1 2 3; do
for v in "" "POD_LIB_PATH=/root/repo/abuild/nozp/libpodsketch_b200.so"; do
  env $v python bench.py --no-cpu-baseline --no-e2e --no-north-star --no-config4 --steps 10 2>/dev/null | python -c '
import sys, json
for l in sys.stdin:
    if l.startswith("{"):
        d = json.loads(l); print(sys.argv[1] or "prefetch", round(d["value"]*1e3, 3))
' "$v"
done; done
