mkdir -p gpurun_out/$1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/$1/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest_gpu.log
timeout 600 ./build/compat_test > gpurun_out/$1/compat_test.log 2>&1; echo rc=$? >> gpurun_out/$1/compat_test.log
timeout 300 python bench.py --steps 60 --warmup 10 --no-cpu --no-extras --no-e2e > gpurun_out/$1/bench.json 2>&1
