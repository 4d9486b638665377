#!/usr/bin/env bash
# A/B of two source trees (each with its own bench.py + library) at N GPUs:
#   tools/ab_tree.sh <tag> <N> <rounds> <treeA> <treeB>
set -u
TAG=$1; N=$2; R=$3; A=$4; B=$5
O=$PWD/gpurun_out/$TAG; mkdir -p $O
for r in $(seq 1 $R); do
  for v in A B; do
    T=$A; [ $v = B ] && T=$B
    (cd $T && timeout 300 python -m torch.distributed.run --standalone --nnodes=1 --nproc-per-node $N \
      bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e --no-extras > $O/$v.$r.json 2>/dev/null)
  done
done
python - "$O" <<'PY'
import json, glob, sys, os, statistics
o = sys.argv[1]
for v in "AB":
    vals, pr = [], []
    for f in sorted(glob.glob(os.path.join(o, f"{v}.*.json"))):
        try:
            d = json.loads(open(f).read().strip().splitlines()[-1])
            vals.append(d["value"]); pr.append([r["ms"] for r in d.get("per_rank") or []])
        except Exception:
            pass
    print(v, vals, statistics.median(vals) if vals else None, pr)
PY
