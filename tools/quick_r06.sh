# quick check after a kernel change: parity + full-size tests, bench, extraction A/B, timeline
mkdir -p gpurun_out/$1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_buckets.py -x -q > gpurun_out/$1/pytest.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu --no-extras > gpurun_out/$1/bench.json 2>&1
ZEN_DIAG_EXTRACT_PLAIN=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-extras > gpurun_out/$1/extract_plain.json 2>&1
python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_1pct.txt > /dev/null 2>&1
python tools/timeline.py --syncs 2 --density 0.1 --out gpurun_out/$1/tl_10pct.txt > /dev/null 2>&1
