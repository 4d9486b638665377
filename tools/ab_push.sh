# A/B of the push scatter's peer-store regrouping and the fused push signal, N=2 and N=4
mkdir -p gpurun_out/$1
for N in 2 4; do
 for cfg in "1 0" "0 0" "1 1" "0 1"; do
  set -- $1 $cfg
  ZEN_PUSH_REORDER=$2 ZEN_PUSH_SIGNAL_FUSED=$((1 - $3)) timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --steps 100 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N reorder=$2 sigkernel=$3', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
 done
done
