# A/B of two builds of the library (ZEN_B200_LIB): N=1 and 8 emulated workers, interleaved
mkdir -p gpurun_out/$1
for r in 1 2 3; do
 for L in base ab; do
  if [ $L = ab ]; then export ZEN_B200_LIB=$PWD/paper_2309_13254_b200/lib/libzen_b200_ab.so; else unset ZEN_B200_LIB; fi
  timeout 300 python bench.py --emulate 8 --steps 60 --warmup 5 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['emulated_local']; print('$L n1', d['value'], d['stage_ms'], 'emu8', e['ms_per_sync_one_gpu'], e['stage_ms'])" >> gpurun_out/$1/ab.txt
 done
done
unset ZEN_B200_LIB
