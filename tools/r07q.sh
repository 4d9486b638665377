# 4 GPUs: single-store signals (ab) vs HEAD (base) at N=2 / N=4, multi-GPU tests on ab
mkdir -p gpurun_out/$1
export ZEN_B200_LIB=$PWD/paper_2309_13254_b200/lib/libzen_b200_ab.so
timeout 900 python -m pytest tests/test_multi_gpu.py -q > gpurun_out/$1/pytest_mgpu_ab.log 2>&1; echo rc=$? >> gpurun_out/$1/pytest_mgpu_ab.log
for r in 1 2; do for N in 2 4; do for L in base ab; do
 if [ $L = ab ]; then export ZEN_B200_LIB=$PWD/paper_2309_13254_b200/lib/libzen_b200_ab.so; else unset ZEN_B200_LIB; fi
 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 298$r$N bench.py --gpus $N --steps 100 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | grep -v NCCL | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L N=$N', d['value'], d['stage_ms'], 'hc', d.get('schemes',{}).get('hc'))" >> gpurun_out/$1/ab.txt
done; done; done
unset ZEN_B200_LIB
