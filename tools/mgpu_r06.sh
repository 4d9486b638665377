# 4 GPUs: rank-mode tests, N=2/N=4 benches (arrival gate vs wait kernels), exchange kernel rates
mkdir -p gpurun_out/$1
timeout 600 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/$1/pytest_mgpu.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest_mgpu.log
for N in 2 4; do
 for wk in 0 1; do
  ZEN_WAIT_KERNEL=$wk timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --steps 100 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N wait_kernel=$wk', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
 done
done
for N in 2 4; do
 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --steps 50 --warmup 5 > gpurun_out/$1/bench_n$N.json 2> gpurun_out/$1/bench_n$N.err
 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N tools/nvlink_profile.py --out gpurun_out/$1/exchange_kernels_n$N.json > gpurun_out/$1/nvl_n$N.log 2>&1
done
