#!/usr/bin/env bash
# A/B of environment settings with one build at N GPUs, interleaved:
#   tools/abenv_n.sh <tag> <N> <rounds> "<envA>" "<envB>"
set -u
TAG=$1; N=$2; R=$3; A=$4; B=$5
O=gpurun_out/$TAG; mkdir -p $O
for r in $(seq 1 $R); do
  for v in A B; do
    E=$A; [ $v = B ] && E=$B
    env $E timeout 300 python -m torch.distributed.run --standalone --nnodes=1 --nproc-per-node $N \
      bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e --no-extras > $O/$v.$r.json 2>/dev/null
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
