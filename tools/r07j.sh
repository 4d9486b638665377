mkdir -p gpurun_out/$1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/$1/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest_gpu.log
timeout 600 python bench.py --emulate 8 > gpurun_out/$1/bench.json 2> gpurun_out/$1/bench.err
python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_1pct.txt > /dev/null 2>&1
python tools/timeline.py --syncs 2 --density 0.1 --out gpurun_out/$1/tl_10pct.txt > /dev/null 2>&1
python tools/timeline.py --syncs 2 --workers 8 --out gpurun_out/$1/tl_emu8.txt > /dev/null 2>&1
