#!/usr/bin/env bash
# A/B/... timing of several builds of libzen_b200.so on the same box, interleaved:
#   tools/abn.sh <tag> <rounds> <lib1> <lib2> ... [-- extra bench args]
set -u
TAG=$1; R=$2; shift 2
LIBS=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do LIBS+=("$1"); shift; done
[ $# -gt 0 ] && shift
O=gpurun_out/$TAG; mkdir -p $O
for r in $(seq 1 $R); do
  for i in "${!LIBS[@]}"; do
    ZEN_B200_LIB=${LIBS[$i]} timeout 300 python bench.py --no-cpu --no-e2e --no-extras "$@" > $O/$i.$r.json 2>/dev/null
  done
done
python - "$O" "${LIBS[@]}" <<'PY'
import json, glob, sys, statistics, os
o, libs = sys.argv[1], sys.argv[2:]
for i, lib in enumerate(libs):
    vals, st = [], None
    for f in sorted(glob.glob(os.path.join(o, f"{i}.*.json"))):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            vals.append(d["value"]); st = d.get("stage_ms")
        except Exception:
            pass
    print(os.path.basename(lib), [round(x, 4) for x in vals],
          "median", round(statistics.median(vals), 4) if vals else None, st)
PY
