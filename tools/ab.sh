#!/usr/bin/env bash
# A/B timing of two builds of libzen_b200.so on the same box, alternating:
#   tools/ab.sh <tag> <libA> <libB> [rounds] [extra bench args]
set -u
TAG=$1; A=$2; B=$3; R=${4:-3}; shift 4 || true
O=gpurun_out/$TAG; mkdir -p $O
for r in $(seq 1 $R); do
  for v in A B; do
    L=$A; [ $v = B ] && L=$B
    ZEN_B200_LIB=$L timeout 300 python bench.py --no-cpu --no-e2e --no-extras "$@" > $O/$v.$r.json 2>/dev/null
  done
done
python - "$O" <<'PY'
import json, glob, sys, statistics, os
o = sys.argv[1]
for v in "AB":
    vals = []
    for f in sorted(glob.glob(os.path.join(o, f"{v}.*.json"))):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            vals.append(d["value"])
        except Exception:
            pass
    print(v, [round(x, 4) for x in vals], "median", round(statistics.median(vals), 4) if vals else None)
PY
