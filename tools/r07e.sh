mkdir -p gpurun_out/$1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_buckets.py -x -q > gpurun_out/$1/pytest.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest.log
python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_1pct.txt > gpurun_out/$1/tl.err 2>&1
python tools/timeline.py --syncs 2 --density 0.1 --out gpurun_out/$1/tl_10pct.txt >> gpurun_out/$1/tl.err 2>&1
bash tools/ab_env.sh $1 ZEN_AGG_FUSED=0
SHORT="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras"
timeout 600 $SHORT > gpurun_out/$1/short.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_agg_fused' -s 3 -c 1 -o gpurun_out/$1/fused1 $SHORT > gpurun_out/$1/ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_agg_fused' -s 3 -c 1 -o gpurun_out/$1/fused10 python bench.py --density 0.1 --steps 3 --warmup 3 --no-e2e --no-cpu --no-extras >> gpurun_out/$1/ncu.log 2>&1
