mkdir -p gpurun_out/$1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/$1/pytest.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest.log
for r in 1 2; do
 timeout 200 python bench.py --density 0.1 --steps 40 --warmup 5 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('10%', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
 timeout 300 python bench.py --emulate 8 --steps 40 --warmup 5 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['emulated_local']; print('n1', d['value'], 'emu8', e['ms_per_sync_one_gpu'])" >> gpurun_out/$1/ab.txt
done
python tools/timeline.py --syncs 2 --density 0.1 --out gpurun_out/$1/tl_10pct.txt > /dev/null 2>&1
