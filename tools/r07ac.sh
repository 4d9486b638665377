mkdir -p gpurun_out/$1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/$1/pytest.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest.log
python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_1pct.txt > /dev/null 2>&1
python tools/timeline.py --syncs 2 --density 0.1 --out gpurun_out/$1/tl_10pct.txt > /dev/null 2>&1
bash tools/ab_env.sh $1 ZEN_HIST_INLINE=0
