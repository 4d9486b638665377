# A/B: side-path width (CTAs per SM of the hash-memory kernels), N=1 at 1 % and 10 %
mkdir -p gpurun_out/$1
for r in 1 2; do
 for c in 1 2 3 4 6; do
  for d in 0.01 0.1; do
   ZEN_SIDE_CTAS=$c timeout 200 python bench.py --density $d --steps 60 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('side=$c dens=$d', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
  done
 done
done
