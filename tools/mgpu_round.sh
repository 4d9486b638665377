#!/usr/bin/env bash
# Multi-GPU pass: parity under torchrun + bench at N = 2..#GPUs.
#   gpurun --gpus 4 --timeout 1800 -- 'bash tools/mgpu_round.sh r01_n4'
set -u
TAG=${1:-mgpu}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
NG=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > "$OUT/topo.txt" 2>&1
timeout 900 python -m pytest tests/test_multi_gpu.py -m gpu -q > "$OUT/pytest_mgpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/status"
for N in 2 4 8; do
  [ "$N" -le "$NG" ] || continue
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
     --master-port $((29500 + N)) bench.py --gpus "$N" > "$OUT/bench_n$N.json" 2> "$OUT/bench_n$N.err"
  echo "bench n=$N rc=$?" >> "$OUT/status"
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
     --master-port $((29600 + N)) bench.py --gpus "$N" --impl reference > "$OUT/bench_ref_n$N.json" 2> "$OUT/bench_ref_n$N.err"
  echo "ref n=$N rc=$?" >> "$OUT/status"
done
