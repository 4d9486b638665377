#!/usr/bin/env bash
# Multi-GPU A/B of library builds (alternating, same box):
#   tools/abmg.sh <tag> <N> <rounds> <libA> <libB> [<libC> ...]
set -u
TAG=$1; N=$2; R=$3; shift 3
O=gpurun_out/$TAG; mkdir -p $O; : > $O/status
for r in $(seq 1 $R); do
  i=0
  for L in "$@"; do
    i=$((i+1))
    ZEN_B200_LIB=$L timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29700 + r * 10 + i)) bench.py --gpus $N --no-cpu \
      --no-e2e --no-extras --steps 100 > $O/x.json 2>/dev/null
    python -c "
import json; d=json.loads(open('$O/x.json').read().strip().splitlines()[-1]); print('lib$i', d['value'], {k: round(v*1000,1) for k,v in d['stage_ms'].items()})" >> $O/status
  done
done
cat $O/status
