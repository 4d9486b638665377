# A/B of an environment switch on one library: $2 = "VAR=value" (the B arm), N=1 at 1 % / 10 % and 8 emulated workers, interleaved
mkdir -p gpurun_out/$1
for r in 1 2; do
 for arm in base "$2"; do
  for d in 0.01 0.1; do
   env $([ "$arm" = base ] || echo "$arm") timeout 200 python bench.py --density $d --steps 60 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$arm dens=$d', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
  done
  env $([ "$arm" = base ] || echo "$arm") timeout 300 python bench.py --emulate 8 --steps 40 --warmup 5 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['emulated_local']; print('$arm emu8', e['ms_per_sync_one_gpu'], e['stage_ms'])" >> gpurun_out/$1/ab.txt
 done
done
