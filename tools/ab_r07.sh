# r07 A/B: library variant (_ab) vs HEAD build + diagnostic timelines
mkdir -p gpurun_out/$1
export ZEN_B200_LIB=$PWD/paper_2309_13254_b200/lib/libzen_b200_ab.so
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/$1/pytest_ab.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest_ab.log
python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_ab.txt > /dev/null 2>&1
ZEN_DIAG_NO_SIDE=1 python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_ab_noside.txt > /dev/null 2>&1
ZEN_DIAG_NO_SIDE=1 python tools/timeline.py --syncs 2 --density 0.1 --out gpurun_out/$1/tl_ab_noside_10.txt > /dev/null 2>&1
python tools/timeline.py --syncs 2 --density 0.1 --out gpurun_out/$1/tl_ab_10.txt > /dev/null 2>&1
for r in 1 2; do
  ZEN_DIAG_NO_SIDE=1 timeout 200 python bench.py --steps 60 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('noside n1', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
done
unset ZEN_B200_LIB
bash tools/ab_lib.sh $1
