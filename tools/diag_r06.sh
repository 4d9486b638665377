# r06 diagnosis: GPU suite + warm timelines (CUPTI) at 1 % and 10 % + a short bench
mkdir -p gpurun_out/$1
timeout 1200 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/$1/pytest.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest.log
python tools/timeline.py --syncs 2 --out gpurun_out/$1/tl_1pct.txt > /dev/null 2>&1
python tools/timeline.py --syncs 2 --density 0.1 --out gpurun_out/$1/tl_10pct.txt > /dev/null 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --no-extras > gpurun_out/$1/bench.json 2> gpurun_out/$1/bench.err
