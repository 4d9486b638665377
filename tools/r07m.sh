mkdir -p gpurun_out/$1
bash tools/ab_lib.sh $1
for r in 1 2; do for L in base ab; do
 if [ $L = ab ]; then export ZEN_B200_LIB=$PWD/paper_2309_13254_b200/lib/libzen_b200_ab.so; else unset ZEN_B200_LIB; fi
 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2970$r bench.py --gpus 2 --steps 100 --warmup 10 --no-cpu --no-extras --no-e2e 2>/dev/null | grep -v NCCL | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L N=2', d['value'], d['stage_ms'])" >> gpurun_out/$1/ab.txt
done; done
unset ZEN_B200_LIB
