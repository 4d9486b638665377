set -u
O=gpurun_out/${TAG:-all}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/status
timeout 300 ./build/compat_test > $O/compat.log 2>&1; echo "compat rc=$?" >> $O/status
timeout 300 python bench.py --no-e2e --no-cpu --emulate 8 > $O/bench_n1.json 2>$O/bench_n1.err; echo "bench1 rc=$?" >> $O/status
NG=$(nvidia-smi -L | wc -l)
for N in 2 4; do
  [ "$N" -le "$NG" ] || continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
     --master-port $((29500 + N)) bench.py --gpus "$N" --no-cpu --no-e2e > "$O/bench_n$N.json" 2> "$O/bench_n$N.err"
  echo "bench n=$N rc=$?" >> "$O/status"
done
tail -2 $O/pytest.log
