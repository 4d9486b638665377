set -u
mkdir -p gpurun_out/r30
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r30/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r30/status
timeout 300 ./build/compat_test > gpurun_out/r30/compat.log 2>&1; echo "compat rc=$?" >> gpurun_out/r30/status
ZEN_PDL=0 timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/r30/nopdl.json 2>gpurun_out/r30/nopdl.err
timeout 300 python bench.py --no-e2e --no-cpu --emulate 8 > gpurun_out/r30/pdl.json 2>gpurun_out/r30/pdl.err
tail -3 gpurun_out/r30/pytest.log
