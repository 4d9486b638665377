mkdir -p gpurun_out/$1
timeout 900 python -m pytest tests/test_gpu_parity.py -k "aggregate_paths or single_worker" -q > gpurun_out/$1/pytest.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest.log
ZEN_AGG_FUSED=1 python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_1pct_fused.txt > /dev/null 2>&1
for r in 1 2 3; do for F in 0 1; do
 ZEN_AGG_FUSED=$F timeout 200 python bench.py --steps 60 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fused=$F', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
done; done
