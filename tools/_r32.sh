set -u
O=gpurun_out/${TAG:-r32}; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status
timeout 300 ./build/compat_test > $O/compat.log 2>&1; echo "compat rc=$?" >> $O/status
timeout 300 python bench.py --no-e2e --no-cpu --emulate 8 > $O/bench.json 2>$O/bench.err; echo "bench rc=$?" >> $O/status
timeout 300 python tools/timeline.py --out $O/tl_n1.txt > /dev/null 2>&1
tail -3 $O/pytest.log
