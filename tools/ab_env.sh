#!/bin/bash
# A/B of engine environment switches on the bench workloads (configs 2, 3, 4):
#   tools/ab_env.sh "POD_X=1" "POD_X=1 POD_Y=1" ...
# prints value / north_star / config4 times per variant ("" = defaults).
for v in "$@"; do
  echo "== ${v:-defaults}"
  env $v python bench.py --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | python -c '
import sys, json
for l in sys.stdin:
    if l.startswith("{"):
        d = json.loads(l)
        print("cfg2", round(d["value"], 5), "cfg3", round(d["north_star"]["value"], 4),
              "cfg4 mixed/fp64", round(d["config4_mixed"]["mixed_s"], 4),
              round(d["config4_mixed"]["fp64_s"], 4))
'
done
