#!/bin/bash
# Config-2 A/B of an alternative library build (tools/ab_build.sh NAME ... ->
# abuild/NAME/libpodsketch_b200.so) against the in-tree one: three
# alternations of `bench.py` (config 2 only, 10 timed runs), ms per run.
# usage: tools/cfg2_ab.sh [abuild/NAME/libpodsketch_b200.so]
ALT=${1:-/root/repo/abuild/nozp/libpodsketch_b200.so}
for i in 1 2 3; do
for v in "" "POD_LIB_PATH=$ALT"; do
  env $v python bench.py --no-cpu-baseline --no-e2e --no-north-star --no-config4 --steps 10 2>/dev/null | python -c '
import sys, json
for l in sys.stdin:
    if l.startswith("{"):
        d = json.loads(l); print(sys.argv[1] or "in-tree", round(d["value"]*1e3, 3))
' "$v"
done; done
