mkdir -p gpurun_out/$1
for r in 1 2; do for N in 2 4; do for P in 0 1; do
 ZEN_HIST_INLINE=$P timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29$r$N$P bench.py --gpus $N --steps 100 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | grep -v NCCL | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('hist_inline=$P N=$N', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
done; done; done
