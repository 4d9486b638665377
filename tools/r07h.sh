mkdir -p gpurun_out/$1
python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_1pct.txt > gpurun_out/$1/tl.err 2>&1
python tools/timeline.py --syncs 2 --density 0.1 --out gpurun_out/$1/tl_10pct.txt >> gpurun_out/$1/tl.err 2>&1
SHORT="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras"
timeout 600 $SHORT > gpurun_out/$1/short.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_agg_fused' -s 3 -c 1 -o gpurun_out/$1/fused1 $SHORT > gpurun_out/$1/ncu.log 2>&1
for d in 0.01 0.1; do for r in 1 2; do
timeout 200 python bench.py --density $d --steps 60 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('dens=$d', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
done; done
