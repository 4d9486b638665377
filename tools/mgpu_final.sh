# 4 GPUs, final: rank-mode tests, N=2/N=4 bench lines, exchange kernel rates
mkdir -p gpurun_out/$1
timeout 600 python -m pytest tests/test_multi_gpu.py tests/test_gpu_buckets.py -q > gpurun_out/$1/pytest_mgpu.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest_mgpu.log
for N in 2 4; do
 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --steps 100 --warmup 10 > gpurun_out/$1/bench_n$N.json 2> gpurun_out/$1/bench_n$N.err
 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N tools/nvlink_profile.py --out gpurun_out/$1/exchange_kernels_n$N.json > gpurun_out/$1/nvl_n$N.log 2>&1
 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N bench.py --impl reference --gpus $N --steps 5 --warmup 1 > gpurun_out/$1/bench_ref_n$N.json 2>&1
done
