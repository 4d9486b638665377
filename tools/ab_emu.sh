# A/B: 8 workers emulated on one GPU (local mode), side-path width
mkdir -p gpurun_out/$1
for r in 1 2; do
 for c in default 3 6 8; do
  if [ $c = default ]; then unset ZEN_SIDE_CTAS; else export ZEN_SIDE_CTAS=$c; fi
  timeout 300 python bench.py --emulate 8 --steps 30 --warmup 5 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['emulated_local']; print('side=$c n1', d['value'], 'emu8', e['ms_per_sync_one_gpu'], e['stage_ms'])" >> gpurun_out/$1/ab.txt
 done
done
unset ZEN_SIDE_CTAS
python tools/timeline.py --syncs 2 --workers 8 --out gpurun_out/$1/tl_n8.txt > /dev/null 2>&1
