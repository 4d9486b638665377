#!/usr/bin/env bash
# N-GPU A/B of library builds on one box, interleaved:
#   tools/abmg_n.sh <tag> <N> <rounds> <lib1> <lib2> ...
set -u
TAG=$1; N=$2; R=$3; shift 3
O=gpurun_out/$TAG; mkdir -p $O
for r in $(seq 1 $R); do
  i=0
  for L in "$@"; do
    ZEN_B200_LIB=$L timeout 300 python -m torch.distributed.run --standalone --nnodes=1 \
      --nproc-per-node $N bench.py --gpus $N --steps 30 --warmup 5 --no-cpu --no-e2e --no-extras \
      > $O/$i.$r.json 2>/dev/null
    i=$((i+1))
  done
done
python - "$O" "$@" <<'PY'
import json, glob, sys, os, statistics
o, libs = sys.argv[1], sys.argv[2:]
for i, lib in enumerate(libs):
    vals = []
    for f in sorted(glob.glob(os.path.join(o, f"{i}.*.json"))):
        try:
            vals.append(json.loads(open(f).read().strip().splitlines()[-1])["value"])
        except Exception:
            pass
    print(os.path.basename(lib), vals, statistics.median(vals) if vals else None)
PY
