# A/B: value-fold unroll (ZEN_AGG_UNROLL) and the extraction variants, 3 interleaved runs each, N=1
mkdir -p gpurun_out/$1
for r in 1 2 3; do
 for u in 1 0; do
  ZEN_AGG_UNROLL=$u timeout 200 python bench.py --steps 100 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('unroll=$u', d['value'], d['stage_ms'], 'extract_part_ms', d['roofline']['launch_ms'])" >> gpurun_out/$1/ab.txt
 done
 ZEN_DIAG_EXTRACT_PLAIN=1 timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('extract_plain_ms', d['roofline']['launch_ms'])" >> gpurun_out/$1/ab.txt
done
python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_1pct.txt > /dev/null 2>&1
