# 4 GPUs: fused aggregate in rank mode (tests + N=2/N=4 A/B), new dense-path tests
mkdir -p gpurun_out/$1
timeout 900 python -m pytest tests/test_multi_gpu.py tests/test_gpu_parity.py -k "multi_gpu or aggregate_paths or dense_pipeline or single_worker" -q > gpurun_out/$1/pytest.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest.log
for r in 1 2; do for N in 2 4; do for F in 0 1; do
 ZEN_AGG_FUSED=$F timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 296$N$F bench.py --gpus $N --steps 100 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | grep -v NCCL | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('N=$N fused=$F', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
done; done; done
