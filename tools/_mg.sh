set -u
O=gpurun_out/${TAG:-mg}; mkdir -p $O
NG=$(nvidia-smi -L | wc -l)
for N in 2 4; do
  [ "$N" -le "$NG" ] || continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
     --master-port $((29500 + N)) bench.py --gpus "$N" --no-cpu > "$O/bench_n$N.json" 2> "$O/bench_n$N.err"
  echo "bench n=$N rc=$?" >> "$O/status"
done
timeout 600 python -m pytest tests/test_multi_gpu.py -m gpu -q > $O/pytest_mgpu.log 2>&1; echo "pytest rc=$?" >> $O/status
