mkdir -p gpurun_out/$1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/$1/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest_gpu.log
timeout 600 ./build/compat_test > gpurun_out/$1/compat_test.log 2>&1; echo rc=$? >> gpurun_out/$1/compat_test.log
for r in 1 2; do for d in 0.01 0.1; do
 timeout 200 python bench.py --density $d --steps 60 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('dens=$d', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
done
 timeout 300 python bench.py --emulate 8 --steps 40 --warmup 5 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['emulated_local']; print('emu8', e['ms_per_sync_one_gpu'])" >> gpurun_out/$1/ab.txt
done
