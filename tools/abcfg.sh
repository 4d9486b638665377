#!/usr/bin/env bash
# A/B of two library builds over several configs on one box:
#   tools/abcfg.sh <tag> <libA> <libB> ["bench args" ...]
set -u
TAG=$1; A=$2; B=$3; shift 3
O=gpurun_out/$TAG; mkdir -p $O; : > $O/status
for cfg in "$@"; do
 for v in A B; do
  L=$A; [ $v = B ] && L=$B
  ZEN_B200_LIB=$L timeout 300 python bench.py --no-cpu --no-e2e --no-extras --steps 50 $cfg > $O/x.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$O/x.json').read().strip().splitlines()[-1]); print('$v', '$cfg', d['value'], {k: round(v*1000,1) for k,v in d['stage_ms'].items()})" >> $O/status
 done
done
cat $O/status
