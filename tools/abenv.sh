#!/usr/bin/env bash
# A/B of environment settings with one build, interleaved (N=1 bench):
#   tools/abenv.sh <tag> <rounds> "<envA>" "<envB>" [extra bench args]
set -u
TAG=$1; R=$2; A=$3; B=$4; shift 4
O=gpurun_out/$TAG; mkdir -p $O
for r in $(seq 1 $R); do
  for v in A B; do
    E=$A; [ $v = B ] && E=$B
    env $E timeout 300 python bench.py --no-cpu --no-e2e --no-extras "$@" > $O/$v.$r.json 2>/dev/null
  done
done
python - "$O" <<'PY'
import json, glob, sys, os, statistics
o = sys.argv[1]
for v in "AB":
    vals, st = [], None
    for f in sorted(glob.glob(os.path.join(o, f"{v}.*.json"))):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1]); vals.append(d["value"]); st = d["stage_ms"]
        except Exception:
            pass
    print(v, vals, "median", statistics.median(vals) if vals else None, st)
PY
